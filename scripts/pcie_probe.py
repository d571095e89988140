"""Host<->device copy ceilings on this box (pinned memory): H2D alone, D2H alone,
and both directions concurrently on two streams -- the bound of bench.py's e2e."""
import time

import torch

n = (4 << 30) // 8
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        if h2d:
            with torch.cuda.stream(s1):
                d_a.copy_(h_in, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out.copy_(d_b, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    return (h2d + d2h) * reps * n * 8 / dt / 1e9


run(True, True, 1)
print(f"H2D {run(True, False):.1f} GB/s  D2H {run(False, True):.1f} GB/s  both {run(True, True):.1f} GB/s total")
