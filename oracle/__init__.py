"""ctypes binding of the plain C oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
module.  The product package ``paper_1309_0392_b200`` never imports it, and the
oracle imports nothing from the product.

Each wrapper cites the PAPER.md (P:n) passage its C routine transcribes; see
oracle/oracle.h for the full contracts and DESIGN.md for the readings R1..R20.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build(force: bool = False) -> str:
    """Compile liboracle.so with plain gcc (no FMA contraction, no vectorisation flags)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
        os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))
    ):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
               _SRC, "-o", _LIB, "-lm", "-lpthread"]
        subprocess.check_call(cmd, cwd=_HERE)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        L.sgo_num_points.argtypes = [_i32p, ctypes.c_int32]
        L.sgo_num_points.restype = ctypes.c_int64
        for name in ("sgo_hierarchize_axis", "sgo_dehierarchize_axis"):
            f = getattr(L, name)
            f.argtypes = [_f64p, _i32p, ctypes.c_int32, ctypes.c_int32]
            f.restype = ctypes.c_int
        for name in ("sgo_hierarchize", "sgo_dehierarchize"):
            f = getattr(L, name)
            f.argtypes = [_f64p, _i32p, ctypes.c_int32, _i32p]
            f.restype = ctypes.c_int
        L.sgo_transform_threads.argtypes = [_f64p, _i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32]
        L.sgo_transform_threads.restype = ctypes.c_int
        L.sgo_counted_hierarchize.argtypes = [_f64p, _i32p, ctypes.c_int32, _i64p, _i64p]
        L.sgo_counted_hierarchize.restype = ctypes.c_int
        L.sgo_flop_count.argtypes = [_i32p, ctypes.c_int32]
        L.sgo_flop_count.restype = ctypes.c_int64
        L.sgo_basis_solve.argtypes = [_f64p, _f64p, _i32p, ctypes.c_int32]
        L.sgo_basis_solve.restype = ctypes.c_int
        L.sgo_evaluate.argtypes = [_f64p, _i32p, ctypes.c_int32, _f64p]
        L.sgo_evaluate.restype = ctypes.c_double
        L.sgo_fill_uniform.argtypes = [_f64p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64]
        L.sgo_fill_uniform.restype = None
        L.sgo_digest.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64]
        L.sgo_digest.restype = ctypes.c_uint64
        L.sgo_sparse_num_points.argtypes = [ctypes.c_int32, ctypes.c_int32]
        L.sgo_sparse_num_points.restype = ctypes.c_int64
        _pp = ctypes.POINTER(ctypes.c_void_p)
        L.sgo_gather.argtypes = [_pp, _i32p, _f64p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _f64p]
        L.sgo_gather.restype = ctypes.c_int
        L.sgo_scatter.argtypes = [_pp, _i32p, ctypes.c_int64, ctypes.c_int32, ctypes.c_int32, _f64p]
        L.sgo_scatter.restype = ctypes.c_int
        _lib = L
    return _lib


def _levels(levels):
    a = np.ascontiguousarray(np.asarray(levels, dtype=np.int32))
    return a, a.ctypes.data_as(_i32p), int(a.size)


def _grid(g):
    if not (isinstance(g, np.ndarray) and g.dtype == np.float64 and g.flags.c_contiguous):
        raise TypeError("grid must be a C-contiguous float64 numpy array")
    return g.ctypes.data_as(_f64p)


def num_points(levels) -> int:
    """N = prod (2^l_k - 1)."""
    _a, p, d = _levels(levels)
    return int(lib().sgo_num_points(p, d))


def hierarchize(grid: np.ndarray, levels, axis_order=None) -> np.ndarray:
    """In place, literal Alg. 1; returns ``grid``."""
    _a, p, d = _levels(levels)
    if grid.size != num_points(levels):
        raise ValueError("grid size does not match levels")
    op = None
    if axis_order is not None:
        ob = np.ascontiguousarray(np.asarray(axis_order, dtype=np.int32))
        op = ob.ctypes.data_as(_i32p)
    rc = lib().sgo_hierarchize(_grid(grid), p, d, op)
    if rc:
        raise ValueError(f"sgo_hierarchize failed ({rc})")
    return grid


def transform_threads(grid: np.ndarray, levels, threads: int, inverse: bool = False) -> np.ndarray:
    """In place, Alg. 1 (or its inverse) with each axis pass's poles split over
    ``threads`` pthreads -- timing only (bench.py cpu_baseline), bitwise equal to
    ``hierarchize`` / ``dehierarchize``; returns ``grid``."""
    _a, p, d = _levels(levels)
    if grid.size != num_points(levels):
        raise ValueError("grid size does not match levels")
    rc = lib().sgo_transform_threads(_grid(grid), p, d, int(bool(inverse)), int(threads))
    if rc:
        raise ValueError(f"sgo_transform_threads failed ({rc})")
    return grid


def dehierarchize(grid: np.ndarray, levels, axis_order=None) -> np.ndarray:
    """In place inverse (reading R9)."""
    _a, p, d = _levels(levels)
    if grid.size != num_points(levels):
        raise ValueError("grid size does not match levels")
    op = None
    if axis_order is not None:
        ob = np.ascontiguousarray(np.asarray(axis_order, dtype=np.int32))
        op = ob.ctypes.data_as(_i32p)
    rc = lib().sgo_dehierarchize(_grid(grid), p, d, op)
    if rc:
        raise ValueError(f"sgo_dehierarchize failed ({rc})")
    return grid


def hierarchize_axis(grid: np.ndarray, levels, axis: int) -> np.ndarray:
    """One sweep of Alg. 1's outer loop, along 0-based ``axis``."""
    _a, p, d = _levels(levels)
    rc = lib().sgo_hierarchize_axis(_grid(grid), p, d, int(axis))
    if rc:
        raise ValueError("sgo_hierarchize_axis failed")
    return grid


def dehierarchize_axis(grid: np.ndarray, levels, axis: int) -> np.ndarray:
    _a, p, d = _levels(levels)
    rc = lib().sgo_dehierarchize_axis(_grid(grid), p, d, int(axis))
    if rc:
        raise ValueError("sgo_dehierarchize_axis failed")
    return grid


def counted_hierarchize(grid: np.ndarray, levels):
    """Alg. 1 instrumented; returns (adds, mults)."""
    _a, p, d = _levels(levels)
    a = ctypes.c_int64()
    m = ctypes.c_int64()
    rc = lib().sgo_counted_hierarchize(_grid(grid), p, d, ctypes.byref(a), ctypes.byref(m))
    if rc:
        raise ValueError("sgo_counted_hierarchize failed")
    return int(a.value), int(m.value)


def flop_count(levels) -> int:
    """Corrected Eq. 1 (reading R1)."""
    _a, p, d = _levels(levels)
    return int(lib().sgo_flop_count(p, d))


def basis_solve(nodal: np.ndarray, levels) -> np.ndarray:
    """alpha = B^-1 u, dense hat-basis matrix; N <= 2048."""
    _a, p, d = _levels(levels)
    u = np.ascontiguousarray(nodal, dtype=np.float64).ravel()
    out = np.empty_like(u)
    rc = lib().sgo_basis_solve(_grid(u), _grid(out), p, d)
    if rc:
        raise ValueError(f"sgo_basis_solve failed ({rc})")
    return out


def evaluate(alpha: np.ndarray, levels, x) -> float:
    """Hierarchical interpolant at x."""
    _a, p, d = _levels(levels)
    al = np.ascontiguousarray(alpha, dtype=np.float64).ravel()
    xx = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return float(lib().sgo_evaluate(_grid(al), p, d, xx.ctypes.data_as(_f64p)))


def fill_uniform(n: int, seed: int, grid_id: int, index_offset: int = 0) -> np.ndarray:
    """Oracle-side twin of the seeded fill."""
    g = np.empty(int(n), dtype=np.float64)
    lib().sgo_fill_uniform(_grid(g), int(n), ctypes.c_uint64(seed), ctypes.c_uint64(grid_id),
                           int(index_offset))
    return g


def digest(grid: np.ndarray, index_offset: int = 0) -> int:
    g = np.ascontiguousarray(grid, dtype=np.float64).ravel()
    return int(lib().sgo_digest(_grid(g), int(g.size), int(index_offset)))


# ----------------------------------------------- combination technique phase
def sparse_num_points(d: int, n: int) -> int:
    """Points of the sparse grid {W_lam : lam >= 1, |lam|_1 <= n} (oracle.h SG layout)."""
    return int(lib().sgo_sparse_num_points(int(d), int(n)))


def _ptrs(grids):
    return (ctypes.c_void_p * len(grids))(*[g.ctypes.data for g in grids])


def gather(grids, levels_list, coeffs, n: int) -> np.ndarray:
    """sparse = sum_g coeffs[g] * alpha_g, accumulated grid by grid in list order
    (the combination formula on surpluses)."""
    d = len(levels_list[0])
    for g, lv in zip(grids, levels_list):
        _grid(g)
        if g.size != num_points(lv):
            raise ValueError("grid size does not match levels")
    lv = np.ascontiguousarray(np.asarray(levels_list, dtype=np.int32))
    c = np.ascontiguousarray(np.asarray(coeffs, dtype=np.float64))
    out = np.empty(sparse_num_points(d, n), dtype=np.float64)
    rc = lib().sgo_gather(_ptrs(grids), lv.ctypes.data_as(_i32p), c.ctypes.data_as(_f64p), len(grids), d, int(n),
                          _grid(out))
    if rc:
        raise ValueError("sgo_gather failed")
    return out


def scatter(sparse: np.ndarray, levels_list, n: int):
    """Every point of every grid gets its sparse-grid value; returns new arrays."""
    d = len(levels_list[0])
    grids = [np.empty(num_points(lv), dtype=np.float64) for lv in levels_list]
    lv = np.ascontiguousarray(np.asarray(levels_list, dtype=np.int32))
    sp = np.ascontiguousarray(sparse, dtype=np.float64)
    rc = lib().sgo_scatter(_ptrs(grids), lv.ctypes.data_as(_i32p), len(grids), d, int(n), _grid(sp))
    if rc:
        raise ValueError("sgo_scatter failed")
    return grids
