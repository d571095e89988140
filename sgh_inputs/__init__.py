"""Seeded synthetic inputs for hierarchization workloads (arXiv 1309.0392).

This module holds NO arithmetic of the method.  It defines the workloads
(level vectors, the combination-grid member set) and the values the grids are
filled with; both the oracle-side tests and the CUDA-side tests / bench draw
their inputs from here.  Nothing here imports ``oracle`` or the product package.

Recipe:
  * uniform fill: splitmix64 counter-based generator keyed by (seed, grid_id,
    global row-major flat index): key = mix64(seed ^ mix64(grid_id)),
    value(i) = 2 * ((mix64(key + i) >> 11) * 2^-53) - 1  in [-1, 1).
  * smooth fill: f(x) = prod_k x_k (1 - x_k) at x_k = i_k 2^-l_k (BASELINE.json
    configs[0] closed form).
  * tent fill: c * prod_k (1 - |2 x_k - 1|) (the level-1 hat; reading R12).
  * combination set: all l with l_k >= 1 and |l|_1 in {n, n-1, ..,
    n-d+1}; member order = level sum descending, then lexicographic ascending
    (reading R16); grid_id = position in that order.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass

import numpy as np

SEED = 13090392

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def mix64(z):
    """splitmix64 finaliser, vectorised over uint64 numpy arrays (mod 2^64)."""
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = z + _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def num_points(levels) -> int:
    n = 1
    for l in levels:
        n *= (1 << int(l)) - 1
    return n


def fill_uniform(n: int, seed: int = SEED, grid_id: int = 0, index_offset: int = 0,
                 chunk: int = 1 << 22) -> np.ndarray:
    """Values in [-1, 1) for global flat indices index_offset .. index_offset+n-1."""
    out = np.empty(int(n), dtype=np.float64)
    key = mix64(np.uint64(seed) ^ mix64(np.uint64(grid_id)))
    with np.errstate(over="ignore"):
        for s in range(0, int(n), chunk):
            e = min(int(n), s + chunk)
            i = np.arange(index_offset + s, index_offset + e, dtype=np.uint64)
            u = (mix64(key + i) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
            out[s:e] = 2.0 * u - 1.0
    return out


def _coords(l: int) -> np.ndarray:
    return np.arange(1, 1 << l, dtype=np.float64) * (2.0 ** -l)


def fill_smooth(levels) -> np.ndarray:
    """f = prod_k x_k (1 - x_k), row-major with x_1 fastest."""
    f = np.ones(1, dtype=np.float64)
    for l in levels:  # x_1 first -> fastest axis is the last numpy axis
        x = _coords(int(l))
        f = np.multiply.outer(x * (1.0 - x), f)
    return f.ravel()


def fill_tent(levels, c: float = 1.0) -> np.ndarray:
    """c * prod_k (1 - |2 x_k - 1|): the nodal values of the level-1 tensor hat."""
    f = np.full(1, float(c), dtype=np.float64)
    for l in levels:
        x = _coords(int(l))
        f = np.multiply.outer(1.0 - np.abs(2.0 * x - 1.0), f)
    return f.ravel()


def combination_set(d: int, n: int, num_diagonals: int | None = None):
    """Level vectors of the combination technique, in grid_id order (reading R16).

    Diagonals |l|_1 = n, n-1, ..., n-num_diagonals+1 (default d diagonals),
    each lexicographically ascending in (l_1..l_d).
    """
    if num_diagonals is None:
        num_diagonals = d
    out = []
    for q in range(num_diagonals):
        s = n - q
        if s < d:
            break
        diag = [c for c in itertools.product(range(1, s - d + 2), repeat=d) if sum(c) == s]
        diag.sort()
        out.extend(diag)
    return out


def combination_coefficient(d: int, n: int, levels) -> int:
    """(-1)^q C(d-1, q) for |l|_1 = n - q (only needed by gather/scatter)."""
    from math import comb
    q = n - sum(levels)
    return (-1) ** q * comb(d - 1, q)


@dataclass(frozen=True)
class Config:
    name: str
    levels: tuple | None        # single-grid configs
    d: int = 0                  # combination set configs
    n: int = 0


# BASELINE.json "configs"
CONFIGS = {
    "C1": Config("C1", (5, 5)),
    "C2": Config("C2", (8, 8, 8)),
    "C3": Config("C3", (10, 4, 4, 4, 4)),
    "C4": Config("C4", (14, 13)),
    "C5": Config("C5", None, d=4, n=22),
}

# Paper-shaped sweeps (not BASELINE.json configs):
#   S1  -- the 1-D grid of Fig. fig:1DLayouts at its largest size, l = 27
#          ("1 GB when the levelsum |l|_1 = 27"): 134,217,727 points;
#   S10 -- the 10-D anisotropic grid of Fig. fig:10D, level (l_1, 2, ..., 2)
#          ("all other dimensions are fixed to 3 grid points") at the
#          largest l_1 with |l|_1 <= 27: l_1 = 9, 511 x 3^9 = 10,057,813 points.
SWEEPS = {
    "S1": Config("S1", (27,)),
    "S10": Config("S10", (9,) + (2,) * 9),
}


def sweep_levels(name: str, top: int):
    """Level vectors of a paper sweep up to `top` (1-D: l = 1..top; 10-D: l_1 = 1..top)."""
    if name == "S1":
        return [(l,) for l in range(1, top + 1)]
    if name == "S10":
        return [(l,) + (2,) * 9 for l in range(1, top + 1)]
    raise KeyError(name)


def lpt_partition(sizes, nparts: int):
    """Longest-processing-time-first assignment of items (by size) to parts.

    Returns a list of index lists.  Deterministic: ties broken by index.
    (Workload partitioning, not method arithmetic.)"""
    import heapq
    order = sorted(range(len(sizes)), key=lambda i: (-sizes[i], i))
    heap = [(0, p) for p in range(nparts)]
    parts = [[] for _ in range(nparts)]
    for i in order:
        load, p = heapq.heappop(heap)
        parts[p].append(i)
        heapq.heappush(heap, (load + sizes[i], p))
    for p in parts:
        p.sort()
    return parts


def contiguous_partition(sizes, nparts: int):
    """Split the ORDERED item list into nparts contiguous, non-empty blocks of
    about equal size sums: [(begin, end)].  (The multi-rank gather needs each
    rank to hold a contiguous block of the grid order; workload partitioning,
    not method arithmetic.)"""
    n = len(sizes)
    if nparts < 1 or n < nparts:
        raise ValueError("need at least one item per part")
    prefix = [0]
    for s in sizes:
        prefix.append(prefix[-1] + s)
    total = prefix[-1]
    bounds = [0]
    for k in range(1, nparts):
        target = total * k / nparts
        i = bounds[-1] + 1                          # smallest end whose prefix reaches the target
        while i < n - (nparts - k) and prefix[i] < target:
            i += 1
        if i > bounds[-1] + 1 and abs(prefix[i - 1] - target) <= abs(prefix[i] - target):
            i -= 1                                  # the nearer boundary
        bounds.append(i)
    bounds.append(n)
    return [(bounds[k], bounds[k + 1]) for k in range(nparts)]
