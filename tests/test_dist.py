"""Multi-process (N > 1) host logic of the shift-sharded driver, on CPU with the gloo backend
(world_size 2, 127.0.0.1): block-cyclic column sharding, T broadcast, all-gather of the shards and
their exponents, unpacking.  The local solve is the CPU oracle here (tests may call it); on the GPU
path it is libmstrsm's trevc_*_cols.  Columns are independent, so the sharded result
must equal the unsharded one bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_1607_01477_b200 import dist as pdist
from paper_1607_01477_b200 import inputs


def test_shard_cols_partition_and_balance():
    for m, P, g in [(1, 2, 16), (37, 2, 4), (2048, 8, 16), (16384, 8, 16), (1000, 3, 7)]:
        shards = [pdist.shard_cols(m, P, r, g) for r in range(P)]
        allc = np.sort(np.concatenate(shards))
        assert np.array_equal(allc, np.arange(m))                         # disjoint cover
        for s in shards:
            assert np.all(np.diff(s) > 0)                                  # ascending (ABI)
    for m, P, g, tol in [(2048, 8, 16, 1.02), (16384, 8, 16, 1.001), (16384, 2, 16, 1.0001)]:
        work = [float(np.sum(pdist.shard_cols(m, P, r, g).astype(float) ** 2)) for r in range(P)]
        assert max(work) / min(work) < tol                                 # ~(k-1)^2 per column
    # a contiguous split would not be balanced (the reason for block-cyclic)
    m, P = 16384, 8
    last = np.arange(m)[m - m // P:]
    assert np.sum(last.astype(float) ** 2) / np.sum(np.arange(m, dtype=float) ** 2) > 0.3


def test_library_shard_map_is_the_driver_map():
    """libmstrsm's native multi-GPU entry (trevc_*_dist) deals columns exactly as dist.py does."""
    import paper_1607_01477_b200 as ms
    for m, P in [(1, 1), (37, 2), (1000, 3), (2048, 8), (16384, 8), (5000, 7)]:
        for r in range(P):
            assert np.array_equal(ms.dist_shard(m, P, r), pdist.shard_cols(m, P, r, 16))
    lib = ms.load()
    assert lib.mstrsm_dist_shard(10, 2, 2, None) == -1 and lib.mstrsm_dist_shard(-1, 1, 0, None) == -1


def test_unpack_inverts_the_shard_layout():
    m, P, g = 50, 3, 4
    Z = torch.arange(m * m, dtype=torch.float64).reshape(m, m).t()        # column-major
    mc = pdist.max_shard(m, P, g)
    gathered = []
    for r in range(P):
        cols = pdist.shard_cols(m, P, r, g)
        pad = torch.zeros((mc, m), dtype=torch.float64)
        pad[: len(cols)] = Z[:, torch.from_numpy(cols)].t()
        gathered.append(pad)
    assert torch.equal(pdist.unpack(gathered, m, P, g), Z)


def test_pack_upper_roundtrip_keeps_the_upper_triangle():
    m = 300
    T = torch.arange(m * m, dtype=torch.float64).reshape(m, m).t().contiguous().t()   # column-major
    buf = pdist.pack_upper(T, m, 128)
    assert buf.numel() == sum(min(m, c + 128) * (min(m, c + 128) - c) for c in range(0, m, 128))
    R = torch.full((m, m), -1.0, dtype=torch.float64).t()
    pdist.unpack_upper(buf, R, m, 128)
    assert torch.equal(torch.triu(R), torch.triu(T))


def test_block_panels_follow_the_block_partition():
    """T travels in the panels the op N blocks consume, bottom-up (R9: the top block is short):
    panel b = columns [lo_b, hi_b), rows 0 .. hi_b; together they cover the upper triangle once."""
    for m, nb in [(1, 128), (300, 128), (1100, 128), (2048, 64), (97, 7)]:
        pan = pdist.block_panels(m, nb)
        assert pan[0][1] == m and pan[-1][0] == 0
        for (lo, hi), (lo2, hi2) in zip(pan, pan[1:]):
            assert hi2 == lo and hi - lo == nb
        assert 0 < pan[-1][1] - pan[-1][0] <= nb
        cover = np.zeros((m, m), int)
        for lo, hi in pan:
            cover[:hi, lo:hi] += 1
        assert (np.triu(cover) == np.triu(np.ones((m, m), int))).all()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, m, nb, cplx, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dtype = torch.complex128 if cplx else torch.float64
        if rank == 0:
            Tn = inputs.c5_grcar_like(m=m) if cplx else inputs.c2_trevc_real(m=m)
            T = torch.from_numpy(np.ascontiguousarray(Tn))
        else:
            T = torch.zeros((m, m), dtype=dtype)

        def solve_cols(Tt, cols, out):
            Zl, el = oracle.trevc(Tt.numpy(), nb=nb, cols=cols, nthreads=1)
            out.copy_(torch.from_numpy(Zl))
            return torch.from_numpy(el)

        Z, e = pdist.trevc_sharded(T, m, solve_cols, rank=rank, world=world, g=4, nb=nb)
        out[rank] = (Z.contiguous().numpy().copy(), e.numpy().copy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("cplx", [False, True])
def test_sharded_trevc_world2_gloo_matches_unsharded(cplx):
    m, nb, world = (256 if cplx else 96), 16, 2     # the c5 shape rescales from m ~ 200 on
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, m, nb, cplx, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    Tn = inputs.c5_grcar_like(m=m) if cplx else inputs.c2_trevc_real(m=m)
    Zo, eo = oracle.trevc(Tn, nb=nb)
    for r in range(world):
        Z, e = out[r]
        assert np.array_equal(e, eo)
        assert np.array_equal(Z, Zo)          # bit for bit: columns are independent
    assert (eo < 0).any() or not cplx         # the c5-shaped case exercises rescaling
