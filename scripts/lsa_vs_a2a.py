"""One-GPU timing of the sharded all-to-all path's two transports on a
one-rank communicator (the pool has one GPU): NCCL grouped send/recv with
pack / unpack copies vs the device-API (LSA) re-shard kernels, beside the
single-grid plan.  Prints one JSON line per (workload, path, direction)."""
import json
import socket
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, ".")
import paper_1309_0392_b200 as sgh  # noqa: E402
import sgh_inputs as si  # noqa: E402


def timeit(fn, steps=10, warmup=3):
    flush = torch.empty(256 << 17, dtype=torch.float64, device="cuda")
    for _ in range(warmup):
        fn()
    ts = []
    for _ in range(steps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return sorted(ts)[len(ts) // 2]


def main():
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
    comm = sgh.ShardComm()
    big = max(sgh.sharded_lsa_window_bytes(si.CONFIGS[w].levels, 1) for w in ("C2", "C3", "C4"))
    comm.enable_lsa(big)
    for w in ("C2", "C3", "C4"):
        lv = si.CONFIGS[w].levels
        N = si.num_points(lv)
        g = torch.empty(N, dtype=torch.float64, device="cuda")
        sgh.fill_uniform(g, si.SEED, 0)
        ws = torch.empty(sgh.sharded_workspace_bytes(lv, 1) // 8 + 1, dtype=torch.float64, device="cuda")
        for inv in (False, True):
            for path, fn in (("single_grid", lambda: sgh.transform(g, lv, inverse=inv)),
                             ("a2a_nccl", lambda: comm.transform(g, lv, ws, inverse=inv)),
                             ("a2a_lsa", lambda: comm.transform_lsa(g, lv, inverse=inv))):
                ms = timeit(fn)
                print(json.dumps({"workload": w, "levels": lv, "path": path, "inverse": inv, "ms": ms,
                                  "Gpoints_s": N / ms / 1e6}), flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
