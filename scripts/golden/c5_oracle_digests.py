"""Write tests/golden/c5_oracle_digests.json: over the whole C5 set (4,255
grids, 41 GB streamed grid by grid), the sums mod 2^64 of the per-grid
digests of the oracle's dehierarchize(fill) and dehierarchize(hierarchize(fill))
-- computed by oracle/ ONLY (fill, transform and digest twins in plain C), so
the GPU tests can check full-set dehierarchization against values that never
came from the CUDA path.
    python scripts/golden/c5_oracle_digests.py [threads]"""
import json
import os
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import sgh_inputs as si  # noqa: E402

SEED = si.SEED


def one(args):
    gid, lv = args
    n = si.num_points(lv)
    u = oracle.fill_uniform(n, SEED, gid)
    d = oracle.dehierarchize(u.copy(), lv)
    h = oracle.hierarchize(u, lv)
    dh = oracle.digest(h)
    rt = oracle.dehierarchize(h, lv)
    return oracle.digest(d), oracle.digest(rt), dh


def main():
    threads = int(sys.argv[1]) if len(sys.argv) > 1 else (os.cpu_count() or 1)
    cs = si.combination_set(4, 22)
    s_d = s_rt = s_h = 0
    with ThreadPoolExecutor(max_workers=threads) as ex:
        for dd, rt, dh in ex.map(one, list(enumerate(cs)), chunksize=8):
            s_d = (s_d + dd) % (1 << 64)
            s_rt = (s_rt + rt) % (1 << 64)
            s_h = (s_h + dh) % (1 << 64)
    # self-check against the survey's independent golden sum (a third implementation)
    sd = json.load(open(os.path.join(ROOT, "tests", "golden", "survey_digests.json")))
    assert s_h == int(sd["C5"]["sum_hierarchized"], 16), "oracle C5 hierarchized sum disagrees with the survey"
    out = {"_source": "scripts/golden/c5_oracle_digests.py (oracle/ only: fill, (de)hierarchize, digest)",
           "seed": SEED, "d": 4, "n": 22, "num_grids": len(cs),
           "sum_dehierarchized_fill": f"0x{s_d:016x}", "sum_round_trip": f"0x{s_rt:016x}"}
    path = os.path.join(ROOT, "tests", "golden", "c5_oracle_digests.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
