"""bench.py's multi-rank launch, on CPU (--dry-run: no GPU work).

`python bench.py --gpus N` without a torchrun environment starts N ranks of
itself (torch.distributed.run, rendezvous on 127.0.0.1); every rank sees the
contract's RANK / WORLD_SIZE / LOCAL_RANK and selects the path DESIGN.md §9
names: C5 grids LPT-balanced over the ranks (the ranks' grids partition the
set), C4 sharded along x_d in dyadic row blocks.  A WORLD_SIZE that disagrees
with --gpus is refused (exit 2) instead of silently timing fewer GPUs."""
import json
import os
import subprocess
import sys

import pytest

import sgh_inputs as si

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(args, env_extra=None, expect_rc=0):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT", "LOCAL_WORLD_SIZE")}
    env.update(env_extra or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       env=env, cwd=ROOT, timeout=600)
    assert r.returncode == expect_rc, r.stderr[-3000:]
    return [json.loads(ln) for ln in r.stdout.splitlines() if ln.startswith("{")]


@pytest.mark.parametrize("n", [2, 4])
def test_self_launch_c5_ranks_partition_the_set(n):
    lines = _bench(["--gpus", str(n), "--dry-run"])
    assert sorted(d["rank"] for d in lines) == list(range(n))
    assert all(d["world_size"] == n and d["local_rank"] == d["rank"] for d in lines)
    assert all(d["path"].startswith("C5 grids LPT-balanced") for d in lines)
    members = si.combination_set(4, 22)
    assert sum(d["grids"] for d in lines) == len(members)
    assert sum(d["points"] for d in lines) == sum(si.num_points(l) for l in members)
    cost = [d["planned_ns"] for d in lines]                      # LPT by planned time
    assert max(cost) / (sum(cost) / n) < 1.001
    pts = [d["points"] for d in lines]
    assert max(pts) / (sum(pts) / n) < 1.05


def test_self_launch_c4_sharded_rows():
    lines = sorted(_bench(["--gpus", "4", "--workload", "C4", "--dry-run"]), key=lambda d: d["rank"])
    assert [d["rank"] for d in lines] == [0, 1, 2, 3]
    assert all("sharded along x_d" in d["path"] for d in lines)
    rows = [tuple(d["rows"]) for d in lines]
    assert rows[0][0] == 0 and rows[-1][1] == (1 << 13) - 1      # dyadic blocks cover x_d's 8191 rows
    assert all(rows[i][1] == rows[i + 1][0] for i in range(3))


@pytest.mark.parametrize("path,want", [("a2a", "NCCL all-to-all re-shard"),
                                       ("lsa", "NCCL device-API (LSA) re-shard in kernels")])
def test_self_launch_c4_sharded_transport(path, want):
    lines = _bench(["--gpus", "2", "--workload", "C4", "--sharded", path, "--dry-run"])
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["path"].endswith(want) for d in lines)


def test_world_size_mismatch_refused():
    _bench(["--gpus", "4", "--dry-run"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"}, expect_rc=2)


def test_single_rank_default():
    (d,) = _bench(["--dry-run"])
    assert d["rank"] == 0 and d["world_size"] == 1 and d["path"] == "single GPU"


def test_reference_arm_runs_on_rank_zero_only():
    """--impl reference under N ranks: rank 0 times the oracle, the others idle."""
    lines = sorted(_bench(["--gpus", "2", "--impl", "reference", "--dry-run"]), key=lambda d: d["rank"])
    assert [d["path"] for d in lines] == ["oracle on host cores (rank 0 only)", "idle (rank > 0)"]
    assert all(d["impl"] == "reference" and d["world_size"] == 2 for d in lines)
