"""Multi-process (world size 2, gloo, CPU) tests of the N > 1 host logic.

The GPU pool gives one GPU per call, so the NCCL paths cannot be run with two
ranks here.  These tests run the SAME decomposition on CPU processes:

* sharded grid: the library's own exchange plan
  (``sgh_shard_layout``, host-only C++), row shards of x_d, local axes,
  packing into column blocks, the point-to-point all-to-all (as the library's
  grouped ncclSend/ncclRecv), the axis-d pass on the slab, the way back --
  with the oracle as the per-rank compute.  The result must equal the
  single-process oracle bitwise.
* combination set (a6): LPT partition over ranks covers every grid exactly once
  and is balanced; per-rank digests gathered over gloo match the oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _init(rank, world, port):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _exchange(sends, recv_shapes, rank, world):
    """all-to-all over point-to-point messages (gloo has no alltoall)."""
    recvs = [None] * world
    reqs = []
    for q in range(world):
        if q == rank:
            recvs[q] = sends[q].copy()
            continue
        buf = torch.empty(int(np.prod(recv_shapes[q])), dtype=torch.float64)
        recvs[q] = buf
        reqs.append(dist.irecv(buf, src=q))
    for q in range(world):
        if q != rank:
            reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(sends[q]).ravel()), dst=q))
    for r in reqs:
        r.wait()
    return [np.asarray(recvs[q]).reshape(recv_shapes[q]) for q in range(world)]


def _sharded_worker(rank, world, port, levels, inverse):
    _init(rank, world, port)
    import oracle
    import paper_1309_0392_b200 as sgh
    import sgh_inputs as si
    L = sgh.shard_layout(levels, world)
    assert sgh.shard_rows(levels, world, rank) == (L["row_begin"][rank], L["row_begin"][rank] + L["rows"][rank])
    nd = (1 << levels[-1]) - 1
    C = si.num_points(levels) // nd
    rb, R = L["row_begin"][rank], L["rows"][rank]
    shard = si.fill_uniform(R * C, si.SEED, 3, rb * C).reshape(R, C)
    op = oracle.dehierarchize if inverse else oracle.hierarchize
    # 1. local axes 1..d-1: every x_d plane is a (d-1)-dim grid
    for r in range(R):
        plane = np.ascontiguousarray(shard[r])
        op(plane, levels[:-1])
        shard[r] = plane
    # 2. pack column blocks and exchange (forward re-shard)
    sends = [shard[:, L["col_begin"][q]:L["col_begin"][q] + L["cols"][q]] for q in range(world)]
    recvs = _exchange(sends, [(L["rows"][q], L["cols"][rank]) for q in range(world)], rank, world)
    slab = np.concatenate(recvs, axis=0)
    assert slab.shape == (nd, L["cols"][rank])
    # 3. the axis-d pass: complete poles along x_d
    for c in range(slab.shape[1]):
        pole = np.ascontiguousarray(slab[:, c])
        op(pole, [levels[-1]])
        slab[:, c] = pole
    # 4. back to row shards
    sends = [slab[L["row_begin"][q]:L["row_begin"][q] + L["rows"][q], :] for q in range(world)]
    recvs = _exchange(sends, [(R, L["cols"][q]) for q in range(world)], rank, world)
    for q in range(world):
        shard[:, L["col_begin"][q]:L["col_begin"][q] + L["cols"][q]] = recvs[q]
    # 5. gather and compare with the single-process oracle, bitwise
    flat = torch.from_numpy(np.ascontiguousarray(shard).ravel())
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([flat.numel()]))
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros(mx, dtype=torch.float64)
    pad[:flat.numel()] = flat
    parts = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, pad)
    if rank == 0:
        got = np.concatenate([p[:int(s.item())].numpy() for p, s in zip(parts, sizes)])
        want = op(si.fill_uniform(si.num_points(levels), si.SEED, 3), levels)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), "sharded decomposition differs"
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("levels", [(6, 5), (3, 4, 5), (5, 2, 6), (2, 3, 2, 4)], ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_sharded_decomposition_gloo(levels, inverse):
    mp.spawn(_sharded_worker, args=(2, _free_port(), levels, inverse), nprocs=2, join=True)


def _c5_worker(rank, world, port):
    _init(rank, world, port)
    import oracle
    import sgh_inputs as si
    cs = si.combination_set(4, 22)
    sizes = [si.num_points(l) for l in cs]
    parts = si.lpt_partition(sizes, world)
    mine = parts[rank]
    allparts = [None] * world
    dist.all_gather_object(allparts, mine)
    ids = sorted(i for p in allparts for i in p)
    assert ids == list(range(len(cs)))
    loads = [sum(sizes[i] for i in p) for p in allparts]
    assert max(loads) / (sum(loads) / world) < 1.0001
    # each rank hierarchizes its smallest few members; digests gathered over gloo
    small = sorted(mine, key=lambda i: sizes[i])[:6]
    dig = {}
    for i in small:
        g = oracle.fill_uniform(sizes[i], si.SEED, i)
        oracle.hierarchize(g, cs[i])
        dig[i] = oracle.digest(g)
    alld = [None] * world
    dist.all_gather_object(alld, dig)
    if rank == 0:
        merged = {k: v for d in alld for k, v in d.items()}
        assert len(merged) == 6 * world
        for i, v in merged.items():
            g = oracle.fill_uniform(sizes[i], si.SEED, i)
            assert oracle.digest(oracle.hierarchize(g, cs[i])) == v
    dist.barrier()
    dist.destroy_process_group()


def test_c5_partition_gloo():
    mp.spawn(_c5_worker, args=(2, _free_port()), nprocs=2, join=True)


def _halo_worker(rank, world, port, levels, inverse):
    """Halo + coarse-lattice sharded pass (sgh_transform_sharded_halo):
    local axes, ONE all-gather of the shards' first rows (halo + coarse lattice),
    the super-block interior along x_d from shard + halo, the coarse lattice as
    level-p poles -- the oracle for the local / coarse pieces, a plain loop of
    Alg. 1's update for the interior.  Equals the single-process oracle bitwise."""
    _init(rank, world, port)
    import oracle
    import paper_1309_0392_b200 as sgh
    import sgh_inputs as si
    ld = levels[-1]
    p = world.bit_length() - 1
    T = ld - p
    nd = (1 << ld) - 1
    C = si.num_points(levels) // nd
    rb, re = sgh.shard_rows(levels, world, rank)
    R = re - rb
    x = si.fill_uniform(R * C, si.SEED, 5, rb * C).reshape(R, C)
    sign = 1.0 if inverse else -1.0
    op = oracle.dehierarchize if inverse else oracle.hierarchize
    for r in range(R if len(levels) > 1 else 0):          # local axes 1..d-1
        plane = np.ascontiguousarray(x[r])
        op(plane, levels[:-1])
        x[r] = plane
    first = torch.from_numpy(np.ascontiguousarray(x[0]))
    rows = [torch.zeros(C, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(rows, first)                          # the only exchange
    G = np.stack([t.numpy() for t in rows])               # G[q] = rank q's first row
    lo = rank << T                                        # global index of the super-block start
    # view: global 1-based index i in [lo, lo + 2^T] -> local row (i - lo); row 0 = own first
    # row (rank >= 1) or the zero boundary (rank 0); row 2^T = the halo (next rank's first row)
    def coarse():
        if world > 2:
            Gc = np.ascontiguousarray(G[1:]).ravel()
            (oracle.dehierarchize_axis if inverse else oracle.hierarchize_axis)(
                Gc, tuple(levels[:-1]) + (p,), len(levels) - 1)
            G[1:] = Gc.reshape(world - 1, C)

    def interior():
        off = 0 if rank else 1                            # local row of shard row 0
        v = np.zeros((1 + (1 << T), C))
        v[off:off + R] = x
        if rank + 1 < world:
            v[1 << T] = G[rank + 1]                       # the halo row
        if not inverse:                                   # one-pass: values entering the pass
            out = v.copy()
            for k in range(1, 1 << T):
                i = lo + k
                s = i & -i
                y = v[k].copy()
                if i - s >= 1:
                    y = y + sign * 0.5 * v[k - s]
                if i + s <= nd:
                    y = y + sign * 0.5 * v[k + s]
                out[k] = y
            v = out
        else:                                             # coarse -> fine with nodal ends
            s = 1 << (T - 1)
            while s >= 1:
                for k in range(s, 1 << T, 2 * s):
                    i = lo + k
                    y = v[k]
                    if i - s >= 1:
                        y = y + 0.5 * v[k - s]
                    if i + s <= nd:
                        y = y + 0.5 * v[k + s]
                    v[k] = y
                s >>= 1
        x[1 - off:] = v[1:off + R]                        # every row but the own first row

    if not inverse:
        interior()
        coarse()
        if rank:
            x[0] = G[rank]
    else:
        coarse()
        if rank:
            x[0] = G[rank]
        interior()                                        # halo = the now nodal G[rank + 1]
    flat = torch.from_numpy(np.ascontiguousarray(x).ravel())
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([flat.numel()]))
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros(mx, dtype=torch.float64)
    pad[:flat.numel()] = flat
    parts = [torch.zeros(mx, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(parts, pad)
    if rank == 0:
        got = np.concatenate([q[:int(s.item())].numpy() for q, s in zip(parts, sizes)])
        want = op(si.fill_uniform(si.num_points(levels), si.SEED, 5), levels)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), "halo decomposition differs"
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("levels,world", [((6, 5), 2), ((3, 4, 5), 2), ((5, 2, 6), 4), ((2, 3, 2, 4), 4), ((7,), 4)],
                         ids=str)
@pytest.mark.parametrize("inverse", [False, True], ids=["hier", "dehier"])
def test_sharded_halo_decomposition_gloo(levels, world, inverse):
    mp.spawn(_halo_worker, args=(world, _free_port(), levels, inverse), nprocs=world, join=True)


def _chain_worker(rank, world, port, d, n, chunks):
    """Multi-rank gather (paper_1309_0392_b200.gather_chain):
    rank r holds a contiguous block of the combination set's grid order and
    continues, subspace range by range, the running sums received from rank
    r-1 (the library's exchange code, with the oracle's per-grid products as
    the per-rank compute); the last rank broadcasts.  Every rank ends with the
    single-process oracle gather, bitwise."""
    _init(rank, world, port)
    import oracle
    import paper_1309_0392_b200 as sgh
    import sgh_inputs as si
    cs = si.combination_set(d, n)
    co = [float(si.combination_coefficient(d, n, lv)) for lv in cs]
    hosts = [oracle.hierarchize(si.fill_uniform(si.num_points(lv), grid_id=g), lv) for g, lv in enumerate(cs)]
    b0, b1 = si.contiguous_partition([si.num_points(lv) for lv in cs], world)[rank]
    terms = [oracle.gather([hosts[g]], [cs[g]], [co[g]], n) for g in range(b0, b1)]   # coeff_g * alpha_g
    sparse = torch.full((sgh.sparse_num_points(d, n),), float("nan"), dtype=torch.float64)

    def gather_fn(b, e, accumulate):                  # the oracle's accumulation, grid after grid
        lo, hi = sgh.sparse_subspace_offset(d, n, b), sgh.sparse_subspace_offset(d, n, e)
        seg = sparse[lo:hi].numpy()
        if not accumulate:
            seg[:] = 0.0
        for t in terms:
            seg[:] = seg + t[lo:hi]

    sgh.gather_chain(None, cs[b0:b1], co[b0:b1], n, sparse, chunks=chunks, gather_fn=gather_fn)
    want = oracle.gather(hosts, cs, co, n)
    assert np.array_equal(sparse.numpy().view(np.uint64), want.view(np.uint64))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("d,n,world,chunks", [(3, 8, 2, 5), (2, 9, 3, 4), (4, 8, 4, 16)], ids=str)
def test_gather_chain_gloo(d, n, world, chunks):
    mp.spawn(_chain_worker, args=(world, _free_port(), d, n, chunks), nprocs=world, join=True)


def test_contiguous_partition():
    import sys
    sys.path.insert(0, ROOT)
    import sgh_inputs as si
    cs = si.combination_set(4, 22)
    sizes = [si.num_points(lv) for lv in cs]
    for P in (2, 4, 8):
        blocks = si.contiguous_partition(sizes, P)
        assert blocks[0][0] == 0 and blocks[-1][1] == len(cs)
        assert all(a[1] == b[0] and a[0] < a[1] for a, b in zip(blocks, blocks[1:] + [(len(cs), len(cs) + 1)]))
        loads = [sum(sizes[b:e]) for b, e in blocks]
        assert max(loads) / (sum(loads) / P) < 1.01
