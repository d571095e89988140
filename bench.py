#!/usr/bin/env python
"""Benchmark: Gpoints/s hierarchized (fp64) on B200, with the HBM roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload C5|C2|C3|C4] [--impl sgh|reference]

Default workload C5 = BASELINE.json configs[4]: the full combination-grid set
d=4, n=22 (|l|_1 in {22,21,20,19}), 4,255 grids, 5,143,278,175 points
(41.1 GB fp64), uniform [-1,1) seeded -- the set BASELINE.json's metric is
quoted on for 1/2/4/8 GPUs.  A step = one batched hierarchization of every
grid (all d axis rounds; Alg. 1) through the C ABI.  With N ranks
(torchrun) the grids are LPT-balanced by point count over the ranks (strong
scaling: the set is fixed), no data-path collective; the elapsed time is the
max over ranks.  Inputs (41 GB) are far larger than L2, so no flush is needed.

Single-grid workloads C2/C3/C4 run the same way with one grid (replicated per
rank; C4 with N > 1 runs the sharded path: by default the halo + coarse-lattice
exchange -- one all-gather of a row per rank -- or, with --sharded a2a, the NCCL
all-to-all re-shard).

--impl reference times the CPU oracle (oracle/, the plain Alg. 1) on this box's
host cores on a bounded sample of the same workload (the paper has no GPU
code and no shipped implementation).

Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Gpoints/s hierarchized (fp64) and achieved HBM GB/s vs B200 roofline, 1/2/4/8 GPU"
UNIT = "Gpoints/s"
FALLBACK_HBM = 6650.0


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy read+write)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ workload
def workload(name):
    import sgh_inputs as si
    if name in ("C5", "C5cycle"):
        cfg = si.CONFIGS["C5"]
        members = si.combination_set(cfg.d, cfg.n)
        desc = (f"C5: combination set d={cfg.d} n={cfg.n}, |l|_1 in {{{cfg.n},{cfg.n-1},{cfg.n-2},{cfg.n-3}}}, "
                f"{len(members)} grids")
        return members, list(range(len(members))), desc
    lv = (si.CONFIGS.get(name) or si.SWEEPS[name]).levels
    return [tuple(lv)], [0], f"{name}: single grid level {tuple(lv)}"


def d_eff(levels):
    return sum(1 for l in levels if l > 1)


def c5_partition(sgh, members, nparts, inverse=False):
    """Grids over ranks: LPT by the planner's estimated time per grid
    (sgh_plan_cost: bytes per pass over each kernel's measured rate), not by
    points -- grids of equal size differ in passes and kernels (a one-GPU
    projection of N = 8, scripts/scale_projection.py, had rank times 3.87 to
    4.17 ms with points balanced to 4e-5)."""
    import sgh_inputs as si
    return si.lpt_partition([sgh.plan_cost(lv, inverse=inverse) for lv in members], nparts)


def plan_passes(sgh, members, inverse, fuse):
    """HBM round trips per point of the library's plans (sgh_plan_describe:
    points each phase writes, summed over the phases, / grid points)."""
    import re

    import sgh_inputs as si
    pts = tot = 0
    for lv in members:
        tot += si.num_points(lv)
        for m in re.finditer(r"points=(\d+)", sgh.plan_describe(lv, inverse=inverse, fuse=fuse)):
            pts += int(m.group(1))
    return pts / tot if tot else None


# ------------------------------------------------------------------ clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu_index = gpu_index
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu_index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------ cpu baseline
def oracle_rate(members, ids, target_cpu_s=12.0, max_points=400_000_000, threads=None, steps=1, warmup=0,
                seed=13090392):
    """Time the CPU oracle (plain Alg. 1, one grid per thread; a single-grid
    workload: its poles split over the threads) on a bounded, deterministic
    sample of the workload.  Returns (Gpoints/s, sample desc, cores, per-step times)."""
    from concurrent.futures import ThreadPoolExecutor

    import oracle
    import sgh_inputs as si
    threads = threads or os.cpu_count() or 1
    sizes = [si.num_points(l) for l in members]
    if len(members) == 1:
        # single-grid workloads (C2-C4, S1, S10): the whole grid, each axis
        # pass's poles split over the host threads (SURVEY 8(c) "--threads T
        # splits poles"; same arithmetic, bitwise equal)
        g = oracle.fill_uniform(sizes[0], seed, ids[0])
        times = []
        for s in range(warmup + steps):
            t0 = time.perf_counter()
            oracle.transform_threads(g, members[0], threads)
            dt = time.perf_counter() - t0
            if s >= warmup:
                times.append(dt)
        desc = (f"the whole grid {tuple(members[0])} ({sizes[0]:,} points), plain Alg. 1 oracle, poles of "
                f"each axis pass split over {threads} threads")
        return sizes[0] / (sum(times) / len(times)) / 1e9, desc, threads, times, sizes[0]
    # calibrate single-thread rate on a mid-sized member
    order = sorted(range(len(members)), key=lambda i: sizes[i])
    probe = order[len(order) // 2]
    g = oracle.fill_uniform(sizes[probe], seed, ids[probe])
    t0 = time.perf_counter()
    oracle.hierarchize(g, members[probe])
    rate1 = sizes[probe] / max(time.perf_counter() - t0, 1e-6)
    budget_pts = min(max_points, int(rate1 * target_cpu_s))
    # deterministic stride sample over the member list
    if sum(sizes) <= budget_pts:
        pick = list(range(len(members)))
    else:
        stride = max(1, int(sum(sizes) / budget_pts))
        pick, tot = [], 0
        for i in range(0, len(members), stride):
            if tot + sizes[i] > budget_pts and pick:
                break
            pick.append(i)
            tot += sizes[i]
        if not pick:
            pick = [order[0]]
    grids = [oracle.fill_uniform(sizes[i], seed, ids[i]) for i in pick]
    npts = sum(sizes[i] for i in pick)

    def run_one(j):
        oracle.hierarchize(grids[j], members[pick[j]])

    times = []
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for s in range(warmup + steps):
            t0 = time.perf_counter()
            list(ex.map(run_one, sorted(range(len(pick)), key=lambda j: -sizes[pick[j]])))
            dt = time.perf_counter() - t0
            if s >= warmup:
                times.append(dt)
    desc = (f"{len(pick)} of {len(members)} grids ({npts:,} points, every {max(1, len(members)//max(len(pick),1))}th "
            f"member), plain Alg. 1 oracle, {threads} threads (one grid per thread)")
    return npts / (sum(times) / len(times)) / 1e9, desc, threads, times, npts


# ------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="C5", choices=["C5", "C2", "C3", "C4", "S1", "S10", "C5cycle"],
                    help="BASELINE.json configs C2..C5 (default C5, the metric's config); S1 / S10 are the "
                         "paper's 1-D l=27 and 10-D (9,2,..,2) sweep tops; C5cycle is the whole combination "
                         "cycle on the C5 set: hierarchize, gather, scatter, dehierarchize (SURVEY 8(f))")
    ap.add_argument("--impl", default="sgh", choices=["sgh", "reference"])
    ap.add_argument("--gather-bfs", action="store_true",
                    help="C5cycle ablation: permute the grids' x_1 rows to BFS order into a scratch copy and gather "
                         "from it (SGH_FLAG_X1_BFS)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--inverse", action="store_true",
                    help="time dehierarchization (P:77) instead (reported under a 'dehierarchized' metric)")
    ap.add_argument("--per-axis", action="store_true",
                    help="one HBM round trip per axis (disable the multi-axis FUSED kernel)")
    ap.add_argument("--sharded", default="halo", choices=["halo", "a2a", "lsa"],
                    help="C4 with N > 1 ranks: halo + coarse-lattice exchange (one all-gather of a row per rank, "
                         "SURVEY 8(f) 1; default) or the all-to-all re-shard (SURVEY 8(a) a7)")
    ap.add_argument("--dump-launch-keys", default=None,
                    help="write the kernel keys of one timed step's launches (in order) to this JSON file "
                         "(pairs the launches of an ncu launch list with the bench's kernel keys: "
                         "scripts/ncu_traffic.py)")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU work: every rank prints its RANK / WORLD_SIZE / LOCAL_RANK and the path it would "
                         "time (CPU test of the multi-rank launch)")
    args = ap.parse_args()

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        return self_launch(args.gpus)
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}: launch one rank per GPU "
            "(torchrun --nproc-per-node N, or bench.py --gpus N without WORLD_SIZE)")
        return 2
    if args.dry_run:
        return dry_run(args, rank, world, local_rank)
    if args.impl == "reference":
        return reference_arm(args, rank, world)
    return sgh_arm(args, rank, world, local_rank)


def self_launch(n):
    """--gpus N without a torchrun environment: start N ranks of this script
    (one per GPU, rendezvous on 127.0.0.1); rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dry_run(args, rank, world, local_rank):
    """The rank layout and the path each rank would time, without a GPU."""
    import sgh_inputs as si
    members, ids, desc = workload(args.workload)
    sizes = [si.num_points(l) for l in members]
    info = {"dry_run": True, "rank": rank, "world_size": world, "local_rank": local_rank,
            "impl": args.impl, "workload": args.workload}
    if args.impl == "reference":
        info["path"] = "oracle on host cores (rank 0 only)" if rank == 0 else "idle (rank > 0)"
    elif args.workload == "C5" and world > 1:
        import paper_1309_0392_b200 as sgh
        part = c5_partition(sgh, members, world, args.inverse)[rank]
        info.update(path="C5 grids LPT-balanced by planned time, batched transform, no data-path collective",
                    grids=len(part), points=sum(sizes[i] for i in part),
                    planned_ns=sum(sgh.plan_cost(members[i], inverse=args.inverse) for i in part))
    elif args.workload == "C4" and world > 1:
        import paper_1309_0392_b200 as sgh
        b, e = sgh.shard_rows(members[0], world, rank)
        info.update(path=("C4 sharded along x_d: " + ("halo + coarse-lattice all-gather" if args.sharded == "halo"
                                                       else "NCCL device-API (LSA) re-shard in kernels"
                                                       if args.sharded == "lsa" else "NCCL all-to-all re-shard")),
                    rows=[b, e])
    else:
        info.update(path="replica of the single-grid workload" if world > 1 else "single GPU",
                    grids=len(members), points=sum(sizes))
    # one write(2) per rank: the ranks share stdout, and a single short write
    # to a pipe is atomic (print may split the line from its newline)
    sys.stdout.flush()
    os.write(1, (json.dumps(info) + "\n").encode())
    return 0


def reference_arm(args, rank, world):
    if rank != 0:
        return 0
    import sgh_inputs as si
    members, ids, desc = workload(args.workload)
    total = sum(si.num_points(l) for l in members)
    rate, sample, cores, times, npts = oracle_rate(members, ids, target_cpu_s=4.0, max_points=200_000_000,
                                                   steps=args.steps, warmup=args.warmup)
    ms = 1e3 * sum(times) / len(times)
    out = {"impl": "reference", "metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           # the sgh arm's config keys (the same workload), plus the bounded sample timed per step
           "config": {"workload": desc, "points": total, "bytes": 8 * total,
                      "l2": "host memory (oracle on host cores)",
                      "parallelism": (f"oracle, one grid per host thread ({cores} threads), rank 0 only" if len(members) > 1
                                      else f"oracle, poles split over {cores} host threads, rank 0 only"),
                      "seed": si.SEED, "sample_points_per_step": npts},
           "cpu_baseline": {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
           "note": "the paper's comparison codes (SGpp, Buse et al.) and its own CPU code are not available; "
                   "the reference arm is this repo's plain C oracle of Alg. 1 on host cores"}
    print(json.dumps(out), flush=True)
    return 0


def sgh_arm(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    import paper_1309_0392_b200 as sgh
    import sgh_inputs as si

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        import datetime
        # communicator lines (rank / nranks) in the log, and no indefinite hang
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        dist.init_process_group("nccl", device_id=dev, timeout=datetime.timedelta(seconds=600))
    members, ids, desc = workload(args.workload)
    sizes = [si.num_points(l) for l in members]
    sharded = args.workload == "C4" and world > 1
    gather_desc = None
    if args.workload == "C5" and world > 1:
        part = c5_partition(sgh, members, world, args.inverse)[rank]
        my_members, my_ids = [members[i] for i in part], [ids[i] for i in part]
    elif args.workload == "C5cycle" and world > 1:   # the gather chain needs contiguous grid blocks
        b0, b1 = si.contiguous_partition(sizes, world)[rank]
        my_members, my_ids = members[b0:b1], ids[b0:b1]
    else:
        my_members, my_ids = members, ids
    total_points = sum(sizes) if (args.workload in ("C5", "C5cycle") or sharded) else sum(sizes) * world

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])

    stream = torch.cuda.current_stream()
    if sharded:
        levels = members[0]
        b, e = sgh.shard_rows(levels, world, rank)
        C = sizes[0] // ((1 << levels[-1]) - 1)
        comm = sgh.ShardComm()
        if args.sharded == "halo":
            buf = torch.empty((e - b + 1) * C, dtype=torch.float64, device=dev)   # + the halo slot
            shard = buf[:(e - b) * C]
            ws = torch.empty(sgh.sharded_halo_workspace_bytes(levels, world) // 8 + 1, dtype=torch.float64,
                             device=dev)
            step = lambda: comm.transform_halo(buf, levels, ws, inverse=args.inverse)  # noqa: E731
        elif args.sharded == "lsa":     # the re-shard in kernels over NVLink peer memory (NCCL device API)
            shard = torch.empty((e - b) * C, dtype=torch.float64, device=dev)
            comm.enable_lsa(sgh.sharded_lsa_window_bytes(levels, world))
            step = lambda: comm.transform_lsa(shard, levels, inverse=args.inverse)  # noqa: E731
        else:
            shard = torch.empty((e - b) * C, dtype=torch.float64, device=dev)
            ws = torch.empty(sgh.sharded_workspace_bytes(levels, world) // 8 + 1, dtype=torch.float64, device=dev)
            step = lambda: comm.transform(shard, levels, ws, inverse=args.inverse)  # noqa: E731
        sgh.fill_uniform(shard, si.SEED, 0, b * C)
        my_points = shard.numel()
        deff_pts = d_eff(levels) * my_points
    else:
        batch = sgh.GridBatch(my_members, device=dev, grid_ids=my_ids)
        batch.fill_uniform(si.SEED)
        fuse = not args.per_axis
        step = lambda: batch.transform(args.inverse, fuse=fuse)  # noqa: E731
        if args.workload == "C5cycle":
            cfg = si.CONFIGS["C5"]
            coeffs = [float(si.combination_coefficient(cfg.d, cfg.n, lv)) for lv in my_members]
            sparse = torch.empty(sgh.sparse_num_points(cfg.d, cfg.n), dtype=torch.float64, device=dev)
            # --gather-bfs (ablation, one GPU): gather from a scratch copy whose
            # x_1 rows are in BFS order (sgh_permute_x1_bfs + SGH_FLAG_X1_BFS:
            # same sums; measured slower overall, DESIGN section 1 f3)
            bfs_views = None
            if args.gather_bfs and world == 1 and torch.cuda.mem_get_info(dev)[0] > 8 * batch.total_points + (8 << 30):
                scratch = torch.empty(batch.total_points, dtype=torch.float64, device=dev)
                bfs_views, off = [], 0
                for v in batch.views:
                    bfs_views.append(scratch[off:off + v.numel()])
                    off += v.numel()
            gather_desc = ("x_1 rows permuted to BFS order into a scratch copy, then gathered (contiguous reads)"
                           if bfs_views is not None else "row-major pull")

            def step():
                batch.hierarchize(fuse=fuse)
                if world > 1:   # ranks continue each other's sums in grid order, then broadcast
                    sgh.gather_chain(batch.views, my_members, coeffs, cfg.n, sparse)
                elif bfs_views is not None:
                    sgh.permute_x1_bfs(batch.views, bfs_views, my_members)
                    sgh.gather(bfs_views, my_members, coeffs, cfg.n, sparse, x1_bfs=True)
                else:
                    sgh.gather(batch.views, my_members, coeffs, cfg.n, sparse)
                sgh.scatter(sparse, batch.views, my_members, cfg.n)
                batch.dehierarchize(fuse=fuse)
        my_points = batch.total_points
        deff_pts = sum(d_eff(l) * si.num_points(l) for l in my_members)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # working sets below 1 GB (C2, C3, S10) would otherwise keep part of the
    # grid in the 126 MB L2 between the in-place steps: flush it by writing a
    # 256 MB scratch buffer before every step and time each step alone
    flush_l2 = 8 * my_points < 1e9
    scratch = torch.empty((256 << 20) // 8, dtype=torch.float64, device=dev) if flush_l2 else None

    def timed(k):
        """k steps bracketed by a barrier + synchronize; device ms (events on the work stream)."""
        barrier()
        torch.cuda.synchronize()
        if flush_l2:
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(k)]
            for i in range(k):
                scratch.fill_(float(i))
                evs[i][0].record(stream)
                step()
                evs[i][1].record(stream)
        else:
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            for _ in range(k):
                step()
            ev1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return sum(a.elapsed_time(b) for a, b in evs) if flush_l2 else ev0.elapsed_time(ev1)

    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    n0 = sgh.launch_count()
    ms = timed(args.steps)                       # the headline: no per-launch events inside
    launches = sgh.launch_count() - n0
    clk = clocks.stop()
    # the roofline pass: the same K steps again, every launch bracketed by
    # events on its stream (kernel durations and shares of the step)
    sgh.profile_enable(True)
    ms_prof = timed(args.steps)
    recs = sgh.profile_read()
    sgh.profile_enable(False)
    if args.dump_launch_keys and rank == 0:
        per_step = len(recs) // max(1, args.steps)
        with open(args.dump_launch_keys, "w") as f:
            json.dump({"workload": args.workload, "inverse": bool(args.inverse), "launches_per_step": per_step,
                       "warmup": args.warmup, "keys": [r["kernel"] for r in recs[:per_step]],
                       "algorithmic_bytes": [r["bytes"] for r in recs[:per_step]]}, f)
    if world > 1:
        t = torch.tensor([ms, ms_prof], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ms_prof = float(t[0].item()), float(t[1].item())
    ms_step = ms / args.steps
    value = total_points / (ms_step * 1e-3) / 1e9

    # roofline of the dominant kernel (live events on the launching stream)
    peak, peak_src = peak_hbm()
    per = {}
    for r in recs:
        k = r["kernel"]
        a = per.setdefault(k, {"ms": 0.0, "bytes": 0.0, "launches": 0})
        a["ms"] += r["ms"]
        a["bytes"] += r["bytes"]
        a["launches"] += 1
    kern_tab = {k: {"launches_per_step": v["launches"] / args.steps,
                    "share_of_step": v["ms"] / ms_prof if ms_prof else None,
                    "GBps": v["bytes"] / (v["ms"] * 1e-3) / 1e9 if v["ms"] > 0 else None}
                for k, v in per.items()}
    roof = None
    if per:
        dom = max(per, key=lambda k: per[k]["ms"])
        a = per[dom]
        achieved = a["bytes"] / (a["ms"] * 1e-3) / 1e9
        traffic = None
        tf = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        tkey = args.workload + ("_dehier" if args.inverse else "") + ("_per_axis" if args.per_axis else "")
        if os.path.exists(tf) and not sharded:
            try:   # ncu DRAM bytes of this kernel key, captured for this workload AND direction
                t = json.load(open(tf)).get(tkey, {}).get(dom)
                traffic = t["traffic_bytes_per_launch"] if isinstance(t, dict) else t
            except Exception:
                traffic = None
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "algorithmic_bytes_per_launch": a["bytes"] / a["launches"],
                "avg_launch_ms": a["ms"] / a["launches"], "peak_source": peak_src,
                "timing": "per-launch CUDA events on the launching stream over a second timed pass of the "
                          "same K steps (the headline pass has no per-launch events)",
                "traffic_source": f"profiles/ncu_traffic.json[{tkey}] (ncu dram__bytes_read+write per launch)"}
    step_s = ms_step * 1e-3
    ppp = None if sharded else plan_passes(sgh, my_members, args.inverse, not args.per_axis)
    model = {"per_axis_GBps": 16.0 * deff_pts / step_s / 1e9 if not sharded else None,
             "fused_GBps": 16.0 * my_points / step_s / 1e9,
             "per_axis_frac": (16.0 * deff_pts / step_s / 1e9) / peak if not sharded else None,
             "fused_floor_frac": (16.0 * my_points / step_s / 1e9) / peak,
             "passes_per_point": ppp,
             "plan_GBps": 16.0 * ppp * my_points / step_s / 1e9 if ppp else None,
             "plan_frac": (16.0 * ppp * my_points / step_s / 1e9) / peak if ppp else None,
             "profiled_ms_per_step": ms_prof / args.steps,
             "note": "rank-0 view: 16 B/point/axis (per-axis model), 16 B/point (fused floor), and "
                     "16 B x points written by the plan's phases (plan: HBM round trips per point)"}

    # e2e through the C ABI with host buffers
    e2e = None
    if not args.no_e2e and not sharded and args.workload != "C5cycle":
        e2e = run_e2e(sgh, my_members, my_ids, dev, args.e2e_steps, world, rank)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.workload != "C5cycle":
        rate, sample, cores, _t, _n = oracle_rate(members, ids)
        cpu = {"value": rate, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        metric = METRIC.replace("hierarchized", "dehierarchized") if args.inverse else METRIC
        out = {"metric": metric, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong"
               if (args.workload in ("C5", "C5cycle") or sharded) else "weak", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic",
               "config": {"workload": desc, "points": total_points, "bytes": 8 * total_points,
                          "l2": ("L2 flushed before every step (256 MB write, outside the per-step events)"
                                 if flush_l2 else "inputs larger than L2 (no flush needed)"),
                          "parallelism": (f"grids LPT-balanced by planned time over {world} ranks" if args.workload == "C5" else
                                          f"contiguous grid blocks over {world} ranks, gather chain + broadcast"
                                          if args.workload == "C5cycle"
                                          else ((f"sharded along x_d, {'halo + coarse-lattice all-gather' if args.sharded == 'halo' else 'NCCL device-API (LSA) re-shard' if args.sharded == 'lsa' else 'NCCL all-to-all'}")
                                                if sharded else "replicas")),
                          "seed": si.SEED, **({"gather": gather_desc} if gather_desc else {})},
               "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
               "gpu_launches": launches, "kernels": kern_tab, "model": model}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_e2e(sgh, members, ids, dev, steps, world, rank):
    """Same metric through the public host-buffer API: H2D of every grid, the
    batched transform and D2H of every result, timed on the device."""
    import psutil
    import torch

    import sgh_inputs as si
    sizes = [si.num_points(l) for l in members]
    nbytes = 8 * sum(sizes)
    # ranks of this node pin their buffers at the same time: each takes its share of the host RAM
    avail = psutil.virtual_memory().available // max(1, int(os.environ.get("LOCAL_WORLD_SIZE", world)))
    sub_m, sub_i = members, ids
    note = "all grids of this rank"
    if nbytes * 1.3 > avail:
        # keep within host RAM: a deterministic prefix of the members
        keep, tot = [], 0
        for i, s in enumerate(sizes):
            if (tot + s) * 8 * 1.3 > avail:
                break
            keep.append(i)
            tot += s
        sub_m, sub_i = [members[i] for i in keep], [ids[i] for i in keep]
        note = f"{len(keep)} of {len(members)} grids (host RAM bound)"
    sub_sizes = [si.num_points(l) for l in sub_m]
    total = sum(sub_sizes)
    host = torch.empty(total, dtype=torch.float64, pin_memory=True)
    views, off = [], 0
    for n in sub_sizes:
        views.append(host[off:off + n])
        off += n
    # inputs: device fill, copied to the pinned host buffers (outside the timed region)
    tmp = sgh.GridBatch(sub_m, device=dev, grid_ids=sub_i)
    tmp.fill_uniform(si.SEED)
    for v, dv in zip(views, tmp.views):
        v.copy_(dv, non_blocking=True)
    torch.cuda.synchronize()
    del tmp
    buf = torch.empty(sgh.batched_host_buffer_bytes(sub_m) // 8 + 32, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream()
    sgh.transform_batched_host(views, sub_m, buf)   # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        sgh.transform_batched_host(views, sub_m, buf)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": total * world / (ms * 1e-3) / 1e9 if world > 1 else total / (ms * 1e-3) / 1e9,
            "unit": UNIT, "h2d_bytes_per_step": 8 * total, "d2h_bytes_per_step": 8 * total,
            "ms_per_step": ms, "steps": steps, "grids": note,
            "api": "sgh_transform_batched_host (pinned host buffers, chunked H2D/transform/D2H overlap)"}


if __name__ == "__main__":
    sys.exit(main())
