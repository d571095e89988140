"""paper_1309_0392_b200 -- B200-native hierarchization of combination-technique grids.

Thin Python binding of the C ABI in ``include/sgh.h`` (libsgh.so, CUDA sm_100a).
Argument marshalling only: every step of the method runs in the library's
kernels.  PyTorch provides device memory, streams and process groups.

There is no CPU fallback: importing this module loads ``lib/libsgh.so`` and
raises ``ImportError`` if it is missing; the transforms require CUDA tensors.

Method (arXiv 1309.0392, Alg. 1): for each axis k = 1..d, every 1-D
pole is transformed from the nodal to the hierarchical basis, finest level
first, x[i] -= 0.5*left; x[i] -= 0.5*right; dehierarchization is the
inverse.  Grids are fp64, row-major with x_1 fastest,
n_k = 2^{l_k} - 1 points per axis.
"""
from __future__ import annotations

import ctypes
import os
from typing import Sequence

import torch

__all__ = [
    "lib", "num_points", "hierarchize", "dehierarchize", "transform", "GridBatch",
    "hierarchize_batched", "dehierarchize_batched", "batched_workspace_bytes",
    "transform_batched_host", "batched_host_buffer_bytes",
    "fill_uniform", "digest", "shard_rows", "shard_layout", "ShardComm", "sharded_workspace_bytes",
    "transform_sharded_loopback", "launch_count", "SGHError",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
# SGH_LIB_PATH selects a tuning variant built with `build.py --out` (experiments only)
LIB_PATH = os.environ.get("SGH_LIB_PATH") or os.path.join(_HERE, "lib", "libsgh.so")

FLAG_DEHIERARCHIZE = 1
FLAG_PER_AXIS = 2
FLAG_WHOLE_POLES = 4
FLAG_TWO_BLOCKED = 32
FLAG_TABLE_RESIDENT = 64
FLAG_SCATTER = 8
FLAG_ACCUMULATE = 16
FLAG_X1_BFS = 128
STATUS = {0: "SGH_OK", 1: "SGH_ERR_INVALID_ARGUMENT", 2: "SGH_ERR_CAPACITY", 3: "SGH_ERR_CUDA",
          4: "SGH_ERR_NCCL", 5: "SGH_ERR_WORKSPACE"}


class SGHError(RuntimeError):
    def __init__(self, status: int, detail: str):
        super().__init__(f"{STATUS.get(status, status)}: {detail}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python paper_1309_0392_b200/build.py` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i32p = ctypes.POINTER(ctypes.c_int32)
    i64p = ctypes.POINTER(ctypes.c_int64)
    u64p = ctypes.POINTER(ctypes.c_uint64)
    vp = ctypes.c_void_p
    vpp = ctypes.POINTER(ctypes.c_void_p)
    sz = ctypes.c_size_t
    st = ctypes.c_int
    sigs = {
        "sgh_num_points": (ctypes.c_int64, [i32p, ctypes.c_int32]),
        "sgh_hierarchize": (st, [vp, i32p, ctypes.c_int32, vp]),
        "sgh_dehierarchize": (st, [vp, i32p, ctypes.c_int32, vp]),
        "sgh_transform_ex": (st, [vp, i32p, ctypes.c_int32, i32p, ctypes.c_uint32, ctypes.c_uint32, vp]),
        "sgh_batched_workspace_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32]),
        "sgh_hierarchize_batched": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, vp, sz, vp]),
        "sgh_dehierarchize_batched": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, vp, sz, vp]),
        "sgh_workspace_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32]),
        "sgh_hierarchize_ex": (st, [vp, i32p, ctypes.c_int32, i32p, ctypes.c_uint32, vp, sz, vp]),
        "sgh_batched_host_buffer_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32]),
        "sgh_transform_batched_host": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, vp, sz, vp]),
        "sgh_shard_rows": (st, [i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, i64p, i64p]),
        "sgh_shard_layout": (st, [i32p, ctypes.c_int32, ctypes.c_int32, i64p, i64p, i64p, i64p]),
        "sgh_comm_create": (st, [vpp, vp, ctypes.c_int32, ctypes.c_int32]),
        "sgh_comm_destroy": (None, [vp]),
        "sgh_comm_unique_id": (st, [vp]),
        "sgh_sharded_workspace_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int32]),
        "sgh_hierarchize_sharded": (st, [vp, i32p, ctypes.c_int32, vp, vp, sz, vp]),
        "sgh_dehierarchize_sharded": (st, [vp, i32p, ctypes.c_int32, vp, vp, sz, vp]),
        "sgh_transform_sharded_loopback": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32, vp, sz, vp]),
        "sgh_sharded_halo_workspace_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int32]),
        "sgh_transform_sharded_halo": (st, [vp, i32p, ctypes.c_int32, vp, ctypes.c_uint32, vp, sz, vp]),
        "sgh_transform_sharded_halo_loopback": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                                                     vp, sz, vp]),
        "sgh_comm_lsa_enable": (st, [vp, sz]),
        "sgh_sharded_lsa_window_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int32]),
        "sgh_transform_sharded_lsa": (st, [vp, i32p, ctypes.c_int32, vp, ctypes.c_uint32, vp]),
        "sgh_transform_sharded_lsa_loopback": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_uint32,
                                                    vp, sz, vp]),
        "sgh_fill_uniform": (st, [vp, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, vp]),
        "sgh_fill_uniform_batched": (st, [vpp, i64p, u64p, ctypes.c_int64, ctypes.c_uint64, vp, sz, vp]),
        "sgh_digest": (st, [vp, ctypes.c_int64, ctypes.c_int64, u64p, vp]),
        "sgh_digest_batched": (st, [vpp, i64p, ctypes.c_int64, u64p, vp, sz, vp]),
        "sgh_launch_count": (ctypes.c_uint64, []),
        "sgh_plan_describe": (ctypes.c_int64, [i32p, ctypes.c_int32, ctypes.c_uint32, ctypes.c_char_p, sz]),
        "sgh_plan_cost": (ctypes.c_double, [i32p, ctypes.c_int32, ctypes.c_uint32]),
        "sgh_sharded_plan_bytes": (ctypes.c_double, [i32p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                                     ctypes.c_uint32, ctypes.c_int32]),
        "sgh_sparse_num_points": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32]),
        "sgh_combi_workspace_bytes": (sz, [i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, ctypes.c_uint32]),
        "sgh_gather": (st, [vpp, i32p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_int64,
                            ctypes.c_int32, vp, vp, sz, vp]),
        "sgh_scatter": (st, [vpp, i32p, ctypes.c_int32, ctypes.c_int64, ctypes.c_int32, vp, vp, sz, vp]),
        "sgh_permute_x1_bfs": (st, [vpp, vpp, i32p, ctypes.c_int32, ctypes.c_int64, vp]),
        "sgh_gather_ex": (st, [vpp, i32p, ctypes.POINTER(ctypes.c_double), ctypes.c_int32, ctypes.c_int64,
                               ctypes.c_int32, vp, ctypes.c_int64, ctypes.c_int64, ctypes.c_uint32, vp, sz, vp]),
        "sgh_sparse_num_subspaces": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32]),
        "sgh_sparse_subspace_offset": (ctypes.c_int64, [ctypes.c_int32, ctypes.c_int32, ctypes.c_int64]),
        "sgh_ablation_bfs_permute_1d": (st, [vp, vp, ctypes.c_int32, ctypes.c_int32, vp]),
        "sgh_ablation_bfs_hierarchize_1d": (st, [vp, vp, ctypes.c_int32, vp]),
        "sgh_ablation_bfs_dehierarchize_1d": (st, [vp, ctypes.c_int32, vp]),
        "sgh_profile_enable": (st, [ctypes.c_int32]),
        "sgh_profile_read": (ctypes.c_int64, [ctypes.c_void_p, ctypes.c_int64]),
        "sgh_status_string": (ctypes.c_char_p, [st]),
        "sgh_last_error": (ctypes.c_char_p, []),
        "sgh_version": (ctypes.c_char_p, []),
    }
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()
EXPORTED = ("sgh_num_points", "sgh_hierarchize", "sgh_dehierarchize", "sgh_transform_ex", "sgh_hierarchize_ex",
            "sgh_dehierarchize_batched", "sgh_workspace_bytes",
            "sgh_batched_workspace_bytes", "sgh_hierarchize_batched", "sgh_batched_host_buffer_bytes",
            "sgh_transform_batched_host", "sgh_shard_rows", "sgh_shard_layout", "sgh_comm_create", "sgh_comm_destroy",
            "sgh_comm_unique_id", "sgh_sharded_workspace_bytes", "sgh_hierarchize_sharded",
            "sgh_dehierarchize_sharded", "sgh_transform_sharded_loopback", "sgh_sharded_halo_workspace_bytes",
            "sgh_transform_sharded_halo", "sgh_transform_sharded_halo_loopback", "sgh_comm_lsa_enable",
            "sgh_sharded_lsa_window_bytes", "sgh_transform_sharded_lsa", "sgh_transform_sharded_lsa_loopback",
            "sgh_fill_uniform",
            "sgh_fill_uniform_batched", "sgh_digest", "sgh_digest_batched", "sgh_launch_count",
            "sgh_profile_enable", "sgh_profile_read", "sgh_plan_describe", "sgh_plan_cost", "sgh_sharded_plan_bytes", "sgh_sparse_num_points",
            "sgh_combi_workspace_bytes", "sgh_gather", "sgh_scatter", "sgh_gather_ex", "sgh_permute_x1_bfs",
            "sgh_sparse_num_subspaces", "sgh_sparse_subspace_offset", "sgh_ablation_bfs_permute_1d",
            "sgh_ablation_bfs_hierarchize_1d", "sgh_ablation_bfs_dehierarchize_1d",
            "sgh_status_string", "sgh_last_error", "sgh_version")


def _check(rc: int):
    if rc != 0:
        raise SGHError(rc, lib.sgh_last_error().decode())


def _levels_arr(levels: Sequence[int]):
    a = (ctypes.c_int32 * len(levels))(*[int(x) for x in levels])
    return a, len(levels)


def _stream(stream) -> ctypes.c_void_p:
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _keep_on(stream, *tensors):
    """Tensors allocated on the current stream but used by kernels launched on
    ``stream``: tell the caching allocator, so their blocks are not handed to
    another tensor while those kernels may still run."""
    if stream is not None and stream != torch.cuda.current_stream():
        for t in tensors:
            t.record_stream(stream)


def _grid_ptr(t: torch.Tensor, levels) -> ctypes.c_void_p:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError("grid must be a CUDA tensor (there is no CPU path)")
    if t.dtype != torch.float64:
        raise TypeError("grid must be float64 (the method is fp64)")
    if not t.is_contiguous():
        raise ValueError("grid must be contiguous (row-major, x_1 fastest)")
    if levels is not None and t.numel() != num_points(levels):
        raise ValueError(f"grid has {t.numel()} elements, levels {tuple(levels)} need {num_points(levels)}")
    return ctypes.c_void_p(t.data_ptr())


def num_points(levels: Sequence[int]) -> int:
    """N = prod (2^l_k - 1).  -1 if invalid / overflowing."""
    a, d = _levels_arr(levels)
    return int(lib.sgh_num_points(a, d))


def _flags(inverse: bool, fuse=True) -> int:
    """fuse: True (planner's choice, blocked groups allowed), "whole" (fused
    groups of whole poles only), "two_blocked" (the two-blocked plan wherever
    one exists) or False (one HBM round trip per axis)."""
    if fuse == "whole":
        f = FLAG_WHOLE_POLES
    elif fuse == "two_blocked":
        f = FLAG_TWO_BLOCKED
    elif fuse is True:
        f = 0
    elif fuse is False:
        f = FLAG_PER_AXIS
    else:
        raise ValueError(f"fuse must be True, False, 'whole' or 'two_blocked', not {fuse!r}")
    return (FLAG_DEHIERARCHIZE if inverse else 0) | f


def plan_describe(levels: Sequence[int], inverse: bool = False, fuse=True) -> str:
    """The library's plan for one grid (host-only, no CUDA call)."""
    a, d = _levels_arr(levels)
    fl = ctypes.c_uint32(_flags(inverse, fuse))
    n = int(lib.sgh_plan_describe(a, d, fl, None, 0))
    if n < 0:
        raise ValueError(f"invalid levels {tuple(levels)}")
    buf = ctypes.create_string_buffer(n + 1)
    lib.sgh_plan_describe(a, d, fl, buf, n + 1)
    return buf.value.decode()


def plan_cost(levels: Sequence[int], inverse: bool = False, fuse=True) -> float:
    """The planner's estimated transform time of one grid, ns (host-only)."""
    a, d = _levels_arr(levels)
    c = float(lib.sgh_plan_cost(a, d, ctypes.c_uint32(_flags(inverse, fuse))))
    if c < 0:
        raise ValueError(f"invalid levels {tuple(levels)}")
    return c


def sharded_plan_bytes(levels: Sequence[int], nranks: int, rank: int, *, inverse: bool = False,
                       path: str = "halo", fused: bool = True) -> float:
    """HBM bytes one sharded call plans on rank `rank` (host-only; network
    bytes excluded): path "a2a" (sgh_hierarchize_sharded) or "halo"
    (sgh_transform_sharded_halo; fused=False: its unfused hierarchization)."""
    a, d = _levels_arr(levels)
    fl = (FLAG_DEHIERARCHIZE if inverse else 0) | (0 if fused else FLAG_PER_AXIS)
    b = float(lib.sgh_sharded_plan_bytes(a, d, nranks, rank, ctypes.c_uint32(fl), {"a2a": 0, "halo": 1}[path]))
    if b < 0:
        raise ValueError(f"invalid sharded configuration {tuple(levels)} nranks={nranks} rank={rank}")
    return b


def transform(grid: torch.Tensor, levels: Sequence[int], *, inverse: bool = False, axis_order=None,
              axis_mask: int = 0, fuse: bool = True, stream=None) -> torch.Tensor:
    """In-place (de)hierarchization of one grid; returns ``grid``.

    fuse=False forces one HBM round trip per axis (no multi-axis FUSED tiles);
    the result is bitwise identical either way."""
    a, d = _levels_arr(levels)
    order = None
    if axis_order is not None:
        order = (ctypes.c_int32 * d)(*[int(x) for x in axis_order])
    ptr = _grid_ptr(grid, levels)
    with torch.cuda.device(grid.device):
        _check(lib.sgh_transform_ex(ptr, a, d, order, ctypes.c_uint32(axis_mask),
                                    ctypes.c_uint32(_flags(inverse, fuse)), _stream(stream)))
    return grid


def hierarchize(grid: torch.Tensor, levels: Sequence[int], stream=None) -> torch.Tensor:
    """Alg. 1 in place, axes 1..d."""
    a, d = _levels_arr(levels)
    ptr = _grid_ptr(grid, levels)
    with torch.cuda.device(grid.device):
        _check(lib.sgh_hierarchize(ptr, a, d, _stream(stream)))
    return grid


def dehierarchize(grid: torch.Tensor, levels: Sequence[int], stream=None) -> torch.Tensor:
    """Inverse base change in place."""
    a, d = _levels_arr(levels)
    ptr = _grid_ptr(grid, levels)
    with torch.cuda.device(grid.device):
        _check(lib.sgh_dehierarchize(ptr, a, d, _stream(stream)))
    return grid


def fill_uniform(grid: torch.Tensor, seed: int, grid_id: int = 0, index_offset: int = 0, stream=None) -> torch.Tensor:
    """Seeded counter-based fill (harness utility; DESIGN.md input recipe)."""
    with torch.cuda.device(grid.device):
        _check(lib.sgh_fill_uniform(_grid_ptr(grid, None), grid.numel(), ctypes.c_uint64(seed),
                                    ctypes.c_uint64(grid_id), int(index_offset), _stream(stream)))
    return grid


def digest(grid: torch.Tensor, index_offset: int = 0, stream=None) -> int:
    """Order-independent 64-bit digest (synchronises)."""
    out = ctypes.c_uint64()
    with torch.cuda.device(grid.device):
        _check(lib.sgh_digest(_grid_ptr(grid, None), grid.numel(), int(index_offset), ctypes.byref(out),
                              _stream(stream)))
    return int(out.value)


def launch_count() -> int:
    """Kernels libsgh has launched in this process."""
    return int(lib.sgh_launch_count())


class _LaunchRecord(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("level", ctypes.c_int32), ("inverse", ctypes.c_int32),
                ("variant", ctypes.c_int32), ("bytes", ctypes.c_double), ("ms", ctypes.c_double)]


KIND_NAMES = {0: "flat_slabs", 1: "flat_blocks", 2: "strided", 3: "reg", 4: "fused", 5: "gather", 6: "scatter",
              7: "fpipe"}


def profile_enable(on: bool = True):
    """Start (clearing) / stop per-launch event timing inside libsgh."""
    _check(lib.sgh_profile_enable(1 if on else 0))


def profile_read():
    """Per-launch records since profile_enable(True): list of dicts
    {kernel, level, inverse, bytes, ms} (waits for the events)."""
    n = int(lib.sgh_profile_read(None, 0))
    buf = (_LaunchRecord * max(n, 1))()
    n = int(lib.sgh_profile_read(ctypes.cast(buf, ctypes.c_void_p), n))
    out = []
    for r in buf[:n]:
        name = KIND_NAMES.get(r.kind, str(r.kind)) + (f"<{r.level}>" if r.kind in (2, 3, 4, 7) else "")
        name += {1: "B", 2: "L", 3: "BL"}.get(r.variant, "")   # blocked tiles / lattice views
        out.append({"kernel": name, "level": r.level, "inverse": bool(r.inverse), "bytes": r.bytes, "ms": r.ms,
                    "variant": r.variant})
    return out


# ----------------------------------------------------------------- batched
def _flat_levels(levels_list, d):
    flat = []
    for lv in levels_list:
        if len(lv) != d:
            raise ValueError("all grids of a batch need the same d (pad with level-1 axes)")
        flat.extend(int(x) for x in lv)
    return (ctypes.c_int32 * len(flat))(*flat)


def batched_workspace_bytes(levels_list, inverse: bool = False, fuse: bool = True) -> int:
    if not levels_list:
        return 0
    d = len(levels_list[0])
    return int(lib.sgh_batched_workspace_bytes(_flat_levels(levels_list, d), d, len(levels_list),
                                               _flags(inverse, fuse)))


class GridBatch:
    """A set of combination grids resident in ONE device allocation.

    Grid g occupies ``N_g`` doubles at a 256-byte aligned offset of a single
    torch buffer; ``views[g]`` is its 1-D float64 view.  The batched transform
    runs one grouped launch per (axis round, phase, kernel kind) over all
    grids ("all combination grids are hierarchized in parallel").
    """

    def __init__(self, levels_list, device=None, grid_ids=None):
        if device is None:
            device = torch.device("cuda", torch.cuda.current_device())
        self.device = torch.device(device)
        self.levels = [tuple(int(x) for x in lv) for lv in levels_list]
        self.d = len(self.levels[0]) if self.levels else 0
        self.sizes = [num_points(lv) for lv in self.levels]
        self.grid_ids = list(grid_ids) if grid_ids is not None else list(range(len(self.levels)))
        offs, off = [], 0
        for n in self.sizes:
            offs.append(off)
            off += (n + 31) // 32 * 32          # 256-byte aligned starts
        self.offsets = offs
        self.total_points = sum(self.sizes)
        self.buffer = torch.empty(max(off, 1), dtype=torch.float64, device=self.device)
        self.views = [self.buffer[o:o + n] for o, n in zip(offs, self.sizes)]
        base = self.buffer.data_ptr()
        G = len(self.levels)
        self._ptrs = (ctypes.c_void_p * max(G, 1))(*[base + 8 * o for o in offs])
        self._sizes = (ctypes.c_int64 * max(G, 1))(*self.sizes)
        self._ids = (ctypes.c_uint64 * max(G, 1))(*self.grid_ids)
        self._flat = _flat_levels(self.levels, self.d) if G else None
        ws = max([batched_workspace_bytes(self.levels, inv, fz) for inv in (False, True) for fz in (False, True)]
                 + [self._util_ws_bytes(), 256])
        self.workspace = torch.empty((ws + 7) // 8, dtype=torch.float64, device=self.device)
        self._table_key = None     # (flags, stream) of the task table the workspace holds

    def _util_ws_bytes(self):
        G = len(self.levels)
        return ((G * 32 + 255) // 256 * 256 + (G + 1) * 8 + 255) // 256 * 256 + G * 8 + 256

    def __len__(self):
        return len(self.levels)

    def _ws(self):
        return ctypes.c_void_p(self.workspace.data_ptr()), self.workspace.numel() * 8

    def transform(self, inverse: bool = False, stream=None, fuse: bool = True):
        if not self.levels:
            return self
        ws, wsb = self._ws()
        st = _stream(stream)
        key = (_flags(inverse, fuse), st.value)
        # the workspace is this batch's own and only the library writes it: when
        # the previous call used the same plan and stream, its task table is
        # still there (fill / digest calls reuse the workspace and reset this)
        flags = key[0] | (FLAG_TABLE_RESIDENT if key == self._table_key else 0)
        self._table_key = None
        with torch.cuda.device(self.device):
            _check(lib.sgh_hierarchize_batched(self._ptrs, self._flat, self.d, len(self.levels),
                                               flags, ws, wsb, st))
        self._table_key = key
        return self

    def hierarchize(self, stream=None, fuse: bool = True):
        return self.transform(False, stream, fuse)

    def dehierarchize(self, stream=None, fuse: bool = True):
        return self.transform(True, stream, fuse)

    def fill_uniform(self, seed: int, stream=None):
        if not self.levels:
            return self
        ws, wsb = self._ws()
        self._table_key = None                       # the fill's item list overwrites the workspace
        with torch.cuda.device(self.device):
            _check(lib.sgh_fill_uniform_batched(self._ptrs, self._sizes, self._ids, len(self.levels),
                                                ctypes.c_uint64(seed), ws, wsb, _stream(stream)))
        return self

    def digests(self, stream=None):
        G = len(self.levels)
        if not G:
            return []
        out = (ctypes.c_uint64 * G)()
        ws, wsb = self._ws()
        self._table_key = None                       # the digest's item list overwrites the workspace
        with torch.cuda.device(self.device):
            _check(lib.sgh_digest_batched(self._ptrs, self._sizes, G, out, ws, wsb, _stream(stream)))
        return [int(x) for x in out]


def hierarchize_batched(batch: GridBatch, stream=None) -> GridBatch:
    return batch.transform(False, stream)


def dehierarchize_batched(batch: GridBatch, stream=None) -> GridBatch:
    return batch.transform(True, stream)


def batched_host_buffer_bytes(levels_list, inverse: bool = False) -> int:
    if not levels_list:
        return 0
    d = len(levels_list[0])
    return int(lib.sgh_batched_host_buffer_bytes(_flat_levels(levels_list, d), d, len(levels_list),
                                                 FLAG_DEHIERARCHIZE if inverse else 0))


def transform_batched_host(host_grids, levels_list, device_buffer: torch.Tensor, inverse: bool = False, stream=None):
    """End-to-end transform of HOST grids (CPU float64 tensors, pinned for speed),
    streamed through ``device_buffer`` (>= batched_host_buffer_bytes bytes)."""
    G = len(host_grids)
    if G == 0:
        return
    d = len(levels_list[0])
    for h, lv in zip(host_grids, levels_list):
        if h.is_cuda or h.dtype != torch.float64 or not h.is_contiguous() or h.numel() != num_points(lv):
            raise ValueError("host grids must be contiguous CPU float64 tensors of the right size")
    ptrs = (ctypes.c_void_p * G)(*[h.data_ptr() for h in host_grids])
    with torch.cuda.device(device_buffer.device):
        _check(lib.sgh_transform_batched_host(ptrs, _flat_levels(levels_list, d), d, G,
                                              FLAG_DEHIERARCHIZE if inverse else 0,
                                              ctypes.c_void_p(device_buffer.data_ptr()),
                                              device_buffer.numel() * device_buffer.element_size(),
                                              _stream(stream)))


# ----------------------------------------------------------------- sharded
def shard_rows(levels, nranks: int, rank: int):
    """0-based rows [begin, end) of x_d owned by ``rank`` (host-only)."""
    a, d = _levels_arr(levels)
    b, e = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.sgh_shard_rows(a, d, int(nranks), int(rank), ctypes.byref(b), ctypes.byref(e)))
    return int(b.value), int(e.value)


def shard_layout(levels, nranks: int):
    """The library's exchange plan for a grid sharded along x_d over nranks:
    dict of lists row_begin, rows, col_begin, cols (host-only)."""
    a, d = _levels_arr(levels)
    arrs = [(ctypes.c_int64 * nranks)() for _ in range(4)]
    _check(lib.sgh_shard_layout(a, d, int(nranks), *arrs))
    return {k: [int(x) for x in v] for k, v in zip(("row_begin", "rows", "col_begin", "cols"), arrs)}


def sharded_workspace_bytes(levels, nranks: int) -> int:
    a, d = _levels_arr(levels)
    return int(lib.sgh_sharded_workspace_bytes(a, d, int(nranks)))


class ShardComm:
    """libsgh-owned NCCL communicator; the unique id travels over ``group``."""

    def __init__(self, group=None):
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = torch.zeros(128, dtype=torch.uint8)
        if rank == 0:
            buf = (ctypes.c_uint8 * 128)()
            _check(lib.sgh_comm_unique_id(buf))
            uid = torch.tensor(list(buf), dtype=torch.uint8)
        obj = [uid.tolist()]
        dist.broadcast_object_list(obj, src=0, group=group)
        raw = (ctypes.c_uint8 * 128)(*obj[0])
        h = ctypes.c_void_p()
        _check(lib.sgh_comm_create(ctypes.byref(h), raw, world, rank))
        self.handle, self.rank, self.world = h, rank, world

    def transform(self, shard: torch.Tensor, levels, workspace: torch.Tensor, inverse=False, stream=None):
        a, d = _levels_arr(levels)
        f = lib.sgh_dehierarchize_sharded if inverse else lib.sgh_hierarchize_sharded
        with torch.cuda.device(shard.device):
            _check(f(_grid_ptr(shard, None), a, d, self.handle, ctypes.c_void_p(workspace.data_ptr()),
                     workspace.numel() * workspace.element_size(), _stream(stream)))
        return shard

    def transform_halo(self, shard: torch.Tensor, levels, workspace: torch.Tensor, inverse=False, stream=None,
                       fused=True):
        """Halo + coarse-lattice sharded pass: ``shard`` = this rank's rows plus
        one spare row (sgh_transform_sharded_halo; fused=False: the unfused
        hierarchization)."""
        a, d = _levels_arr(levels)
        fl = (FLAG_DEHIERARCHIZE if inverse else 0) | (0 if fused else FLAG_PER_AXIS)
        with torch.cuda.device(shard.device):
            _check(lib.sgh_transform_sharded_halo(_grid_ptr(shard, None), a, d, self.handle,
                                                  ctypes.c_uint32(fl),
                                                  ctypes.c_void_p(workspace.data_ptr()),
                                                  workspace.numel() * workspace.element_size(), _stream(stream)))
        return shard

    def enable_lsa(self, window_bytes: int):
        """Collective: the device-API (NVLink load/store) exchange for
        ``transform_lsa`` with a library-owned symmetric window of
        ``window_bytes`` (>= sharded_lsa_window_bytes of the grid)."""
        _check(lib.sgh_comm_lsa_enable(self.handle, int(window_bytes)))

    def transform_lsa(self, shard: torch.Tensor, levels, inverse=False, stream=None):
        """All-to-all sharded pass with the re-shard inside kernels over peer
        memory (sgh_transform_sharded_lsa); ``shard`` = this rank's rows."""
        a, d = _levels_arr(levels)
        with torch.cuda.device(shard.device):
            _check(lib.sgh_transform_sharded_lsa(_grid_ptr(shard, None), a, d, self.handle,
                                                 ctypes.c_uint32(FLAG_DEHIERARCHIZE if inverse else 0),
                                                 _stream(stream)))
        return shard

    def close(self):
        if self.handle:
            lib.sgh_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def transform_sharded_loopback(shards, levels, workspace: torch.Tensor, inverse=False, stream=None):
    """All ranks' shards on one device; exchange = device copies (test utility)."""
    P = len(shards)
    a, d = _levels_arr(levels)
    ptrs = (ctypes.c_void_p * P)(*[s.data_ptr() for s in shards])
    with torch.cuda.device(workspace.device):
        _check(lib.sgh_transform_sharded_loopback(ptrs, a, d, P, FLAG_DEHIERARCHIZE if inverse else 0,
                                                  ctypes.c_void_p(workspace.data_ptr()),
                                                  workspace.numel() * workspace.element_size(), _stream(stream)))


def sharded_lsa_window_bytes(levels, nranks: int) -> int:
    a, d = _levels_arr(levels)
    return int(lib.sgh_sharded_lsa_window_bytes(a, d, int(nranks)))


def transform_sharded_lsa_loopback(shards, levels, workspace: torch.Tensor, inverse=False, stream=None):
    """The device-API exchange kernels for len(shards) virtual ranks on one
    device (test utility): window pointers from a table, no barriers."""
    P = len(shards)
    a, d = _levels_arr(levels)
    ptrs = (ctypes.c_void_p * P)(*[s.data_ptr() for s in shards])
    with torch.cuda.device(workspace.device):
        _check(lib.sgh_transform_sharded_lsa_loopback(ptrs, a, d, P, FLAG_DEHIERARCHIZE if inverse else 0,
                                                      ctypes.c_void_p(workspace.data_ptr()),
                                                      workspace.numel() * workspace.element_size(),
                                                      _stream(stream)))
    return shards


def sharded_halo_workspace_bytes(levels, nranks: int) -> int:
    a, d = _levels_arr(levels)
    return int(lib.sgh_sharded_halo_workspace_bytes(a, d, int(nranks)))


def transform_sharded_halo_loopback(shards, levels, workspace: torch.Tensor, inverse=False, stream=None,
                                    fused=True):
    """Halo path for len(shards) virtual ranks on one device (test utility);
    shards[r] = rank r's rows + one spare row; fused=False: the unfused
    hierarchization."""
    P = len(shards)
    a, d = _levels_arr(levels)
    ptrs = (ctypes.c_void_p * P)(*[s.data_ptr() for s in shards])
    fl = (FLAG_DEHIERARCHIZE if inverse else 0) | (0 if fused else FLAG_PER_AXIS)
    with torch.cuda.device(workspace.device):
        _check(lib.sgh_transform_sharded_halo_loopback(ptrs, a, d, P, fl,
                                                       ctypes.c_void_p(workspace.data_ptr()),
                                                       workspace.numel() * workspace.element_size(),
                                                       _stream(stream)))


# ------------------------------------------- combination technique gather / scatter
def sparse_num_points(d: int, n: int) -> int:
    """Points of the sparse grid {W_lam : |lam|_1 <= n} in the SG layout (sgh.h)."""
    return int(lib.sgh_sparse_num_points(int(d), int(n)))


def _combi_common(grids, levels_list):
    d = len(levels_list[0])
    for g, lv in zip(grids, levels_list):
        _grid_ptr(g, lv)
    flat = _flat_levels(levels_list, d)
    ptrs = (ctypes.c_void_p * len(grids))(*[g.data_ptr() for g in grids])
    return d, flat, ptrs


def permute_x1_bfs(src, dst, levels_list, stream=None):
    """dst[g] = src[g] with every x_1 row in BFS order (sgh_permute_x1_bfs):
    the layout ``gather(..., x1_bfs=True)`` reads."""
    d, flat, ptrs = _combi_common(src, levels_list)
    for g, lv in zip(dst, levels_list):
        _grid_ptr(g, lv)
    dptrs = (ctypes.c_void_p * len(dst))(*[g.data_ptr() for g in dst])
    with torch.cuda.device(src[0].device):
        _check(lib.sgh_permute_x1_bfs(ptrs, dptrs, flat, d, len(src), _stream(stream)))
    return dst


def gather(grids, levels_list, coeffs, n: int, sparse: torch.Tensor = None, stream=None,
           x1_bfs: bool = False) -> torch.Tensor:
    """sparse = sum_g coeffs[g] * grids[g] (hierarchical surpluses) in the SG layout.
    x1_bfs: the grids' x_1 rows are in BFS order (permute_x1_bfs)."""
    d, flat, ptrs = _combi_common(grids, levels_list)
    dev = grids[0].device
    if sparse is None:
        sparse = torch.empty(sparse_num_points(d, n), dtype=torch.float64, device=dev)
    if x1_bfs:
        return gather_ex(grids, levels_list, coeffs, n, sparse, 0, sparse_num_subspaces(d, n), stream=stream,
                         x1_bfs=True)
    wsb = int(lib.sgh_combi_workspace_bytes(flat, d, len(grids), int(n), 0))
    ws = torch.empty(max(wsb, 16) // 8 + 2, dtype=torch.float64, device=dev)
    c = (ctypes.c_double * len(grids))(*[float(x) for x in coeffs])
    with torch.cuda.device(dev):
        _check(lib.sgh_gather(ptrs, flat, c, d, len(grids), int(n), ctypes.c_void_p(sparse.data_ptr()),
                              ctypes.c_void_p(ws.data_ptr()), ws.numel() * 8, _stream(stream)))
    _keep_on(stream, ws, sparse)
    return sparse


def sparse_num_subspaces(d: int, n: int) -> int:
    """Subspaces W_lam of the sparse grid of level sum n (C(n, d))."""
    return int(lib.sgh_sparse_num_subspaces(int(d), int(n)))


def sparse_subspace_offset(d: int, n: int, index: int) -> int:
    """Sparse offset of subspace ``index`` in SG order (index == count: the total)."""
    r = int(lib.sgh_sparse_subspace_offset(int(d), int(n), int(index)))
    if r < 0:
        raise SGHError(1, "subspace index out of range")
    return r


def gather_ex(grids, levels_list, coeffs, n: int, sparse: torch.Tensor, sub_begin: int, sub_end: int,
              accumulate: bool = False, stream=None, x1_bfs: bool = False) -> torch.Tensor:
    """Gather restricted to subspaces [sub_begin, sub_end) (SG order); with
    ``accumulate`` every sum continues from the value already in ``sparse``
    (sgh.h sgh_gather_ex, SGH_FLAG_ACCUMULATE)."""
    d, flat, ptrs = _combi_common(grids, levels_list)
    dev = grids[0].device
    wsb = int(lib.sgh_combi_workspace_bytes(flat, d, len(grids), int(n), 0))
    ws = torch.empty(max(wsb, 16) // 8 + 2, dtype=torch.float64, device=dev)
    c = (ctypes.c_double * len(grids))(*[float(x) for x in coeffs])
    with torch.cuda.device(dev):
        _check(lib.sgh_gather_ex(ptrs, flat, c, d, len(grids), int(n), ctypes.c_void_p(sparse.data_ptr()),
                                 int(sub_begin), int(sub_end),
                                 (FLAG_ACCUMULATE if accumulate else 0) | (FLAG_X1_BFS if x1_bfs else 0),
                                 ctypes.c_void_p(ws.data_ptr()), ws.numel() * 8, _stream(stream)))
    _keep_on(stream, ws)
    return sparse


def subspace_chunks(d: int, n: int, chunks: int):
    """Split the subspaces (SG order) into at most ``chunks`` consecutive ranges
    of about equal point counts: [(sub_begin, sub_end, off_begin, off_end)]."""
    nsub = sparse_num_subspaces(d, n)
    total = sparse_subspace_offset(d, n, nsub)
    out, b = [], 0
    for k in range(1, chunks + 1):
        target = total * k // chunks
        lo, hi = b, nsub                       # smallest e with offset(e) >= target
        while lo < hi:
            mid = (lo + hi) // 2
            if sparse_subspace_offset(d, n, mid) >= target:
                hi = mid
            else:
                lo = mid + 1
        e = max(lo, b + 1) if k < chunks else nsub
        e = min(e, nsub)
        if e > b:
            out.append((b, e, sparse_subspace_offset(d, n, b), sparse_subspace_offset(d, n, e)))
            b = e
        if b >= nsub:
            break
    return out


def gather_chain(grids, levels_list, coeffs, n: int, sparse: torch.Tensor, group=None, chunks: int = 16,
                 gather_fn=None) -> torch.Tensor:
    """Multi-rank gather, bitwise equal to one gather over the
    concatenation of the ranks' grid lists in rank order: each rank must hold
    a CONTIGUOUS block of the global grid order.  Rank r receives the running
    sums of a subspace range from rank r-1, continues them over its own grids
    (SGH_FLAG_ACCUMULATE), and passes them on, range after range, so the ranks
    work on different ranges at once; the last rank then broadcasts the
    sparse grid to all (every rank's scatter needs it).  ``gather_fn(b, e,
    accumulate)`` replaces the device gather in CPU tests of the exchange."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    d = len(levels_list[0])
    if gather_fn is None:
        gather_fn = lambda b, e, acc: gather_ex(grids, levels_list, coeffs, n, sparse, b, e, accumulate=acc)  # noqa: E731
    for b, e, lo, hi in subspace_chunks(d, n, chunks):
        part = sparse[lo:hi]
        if rank > 0:
            dist.recv(part, src=dist.get_global_rank(group, rank - 1) if group is not None else rank - 1, group=group)
        gather_fn(b, e, rank > 0)
        if rank < world - 1:
            dist.send(part, dst=dist.get_global_rank(group, rank + 1) if group is not None else rank + 1, group=group)
    last = dist.get_global_rank(group, world - 1) if group is not None else world - 1
    dist.broadcast(sparse, src=last, group=group)
    return sparse


def scatter(sparse: torch.Tensor, grids, levels_list, n: int, stream=None):
    """Every grid point gets its sparse-grid value (in place into ``grids``)."""
    d, flat, ptrs = _combi_common(grids, levels_list)
    dev = grids[0].device
    wsb = int(lib.sgh_combi_workspace_bytes(flat, d, len(grids), int(n), FLAG_SCATTER))
    ws = torch.empty(max(wsb, 16) // 8 + 2, dtype=torch.float64, device=dev)
    with torch.cuda.device(dev):
        _check(lib.sgh_scatter(ptrs, flat, d, len(grids), int(n), ctypes.c_void_p(sparse.data_ptr()),
                               ctypes.c_void_p(ws.data_ptr()), ws.numel() * 8, _stream(stream)))
    _keep_on(stream, ws)
    return grids


# ------------------------------------------------------ ablation (report only)
def bfs_permute_1d(src: torch.Tensor, dst: torch.Tensor, level: int, to_bfs: bool = True, stream=None):
    """Natural <-> BFS order of a 1-D pole (sgh.h ablation section)."""
    with torch.cuda.device(src.device):
        _check(lib.sgh_ablation_bfs_permute_1d(_grid_ptr(src, [level]), _grid_ptr(dst, [level]), int(level),
                                                1 if to_bfs else 0, _stream(stream)))
    return dst


def bfs_hierarchize_1d(src: torch.Tensor, dst: torch.Tensor, level: int, stream=None):
    """Hierarchization of a BFS-ordered 1-D pole, out of place (ablation)."""
    with torch.cuda.device(src.device):
        _check(lib.sgh_ablation_bfs_hierarchize_1d(_grid_ptr(src, [level]), _grid_ptr(dst, [level]), int(level),
                                                    _stream(stream)))
    return dst


def bfs_dehierarchize_1d(grid: torch.Tensor, level: int, stream=None):
    """Dehierarchization of a BFS-ordered 1-D pole, in place (ablation)."""
    with torch.cuda.device(grid.device):
        _check(lib.sgh_ablation_bfs_dehierarchize_1d(_grid_ptr(grid, [level]), int(level), _stream(stream)))
    return grid

