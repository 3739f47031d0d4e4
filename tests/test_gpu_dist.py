"""GPU tests (-m gpu) of the native multi-GPU entries (trevc_*_dist over an NCCL communicator of
the library).  Only one GPU is available to this build, so the collectives run with nranks = 1
(broadcast, all-gather and unpack all execute); the shard map for nranks > 1 is tested on CPU
against dist.py (tests/test_dist.py) and the multi-rank host logic with gloo."""
import numpy as np
import pytest

from paper_1607_01477_b200 import inputs
from tests.gpu_util import dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


@pytest.mark.parametrize("cplx", [False, True])
def test_trevc_dist_single_rank_equals_trevc(ms, cplx):
    import torch
    m = 600
    T = inputs.c5_grcar_like(m) if cplx else inputs.c2_trevc_real(m)
    ms.comm_init(1, 0)
    try:
        Td = dev(T)
        Z1, s1, e1 = ms.trevc_dist(Td, m, nb=128)
        Z2, s2, e2 = ms.trevc(Td, nb=128)
        torch.cuda.synchronize()
        assert np.array_equal(host(Z1), host(Z2))
        assert np.array_equal(host(s1), host(s2)) and np.array_equal(host(e1), host(e2))
        if cplx:
            assert (host(e1) < -100).any()
    finally:
        ms.comm_destroy()


def test_trevc_dist_needs_a_communicator(ms):
    T = dev(inputs.c3_trevc_complex(64))
    with pytest.raises(ms.MstrsmError):
        ms.trevc_dist(T, 64, nb=32)


@pytest.mark.parametrize("op", ["N", "C"])
def test_solve_dist_single_rank_equals_solve(ms, op):
    import torch
    m, n = 300, 90
    rng = np.random.default_rng(8)
    U = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) * 3.0
    U[np.arange(m), np.arange(m)] = rng.uniform(-1e-2, 1e-2, m)
    s = inputs.random_shifts(n, True, 9, radius=1e-2)
    B = inputs.random_rhs(m, n, True, 10)
    ms.comm_init(1, 0)
    try:
        Ud, sd = dev(np.asfortranarray(U)), dev(np.ascontiguousarray(s))
        X1, _, e1 = ms.solve_dist(Ud, sd, dev(B), m, op=op, nb=64)
        X2, _, e2 = ms.solve(Ud, sd, dev(B), safe=True, op=op, nb=64)
        torch.cuda.synchronize()
        assert (host(e2) < 0).any()
        assert np.array_equal(host(X1), host(X2)) and np.array_equal(host(e1), host(e2))
    finally:
        ms.comm_destroy()


@pytest.mark.parametrize("cplx", [False, True])
def test_triangular_pack_unpack_roundtrip(ms, cplx):
    """The library's shard packing (the multi-GPU all-gather layout of dist.tri_layout) and its
    inverse: rows 0..k of eigenvector k travel, rows below come back as 0; the CUDA kernels match
    dist.py's CPU packing bit for bit."""
    import torch
    from paper_1607_01477_b200 import dist as pdist
    m, P = 300, 3
    rng = np.random.default_rng(3)
    Zfull = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    lay, L = pdist.tri_layout(m, P, 16)
    for r in range(P):
        c, h, off = lay[r]
        Zl = np.asfortranarray(Zfull[:, c])
        out_g = torch.zeros(L, dtype=dev(Zl).dtype, device="cuda")
        pdist._pack(dev(Zl), torch.from_numpy(h).cuda(), torch.from_numpy(off).cuda(), out_g)
        out_c = torch.zeros(L, dtype=out_g.dtype)
        pdist._pack(torch.from_numpy(Zl), torch.from_numpy(h), torch.from_numpy(off), out_c)
        torch.cuda.synchronize()
        assert np.array_equal(host(out_g), out_c.numpy())
        R = dev(np.full((m, m), 7.0 + (7j if cplx else 0)))
        pdist._unpack(out_g, torch.from_numpy(h).cuda(), torch.from_numpy(off).cuda(),
                      torch.from_numpy(c.astype(np.int64)).cuda(), m, R)
        torch.cuda.synchronize()
        Rh = host(R)
        for q, k in enumerate(c):
            assert np.array_equal(Rh[: k + 1, k], Zfull[: k + 1, k]) and not Rh[k + 1:, k].any()


def test_trevc_dist_streamed_panels_unpack_path_bit_identical():
    """The non-root side of the panel-streamed broadcast (panels unpacked from the broadcast buffer
    into a workspace copy of T, the solve waiting for each panel's event, delta received rather
    than computed) forced on the single rank with MSTRSM_DIST_TEST_UNPACK=1 (read at first use,
    hence a subprocess): m = 1100 (look-ahead path, ragged top block) equals trevc bit for bit."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = f"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
m = 1100
T = torch.from_numpy(np.asfortranarray(inputs.c5_grcar_like(m))).cuda()
ms.comm_init(1, 0)
Z1, s1, e1 = ms.trevc_dist(T, m, nb=128)
ms.comm_destroy()
Z2, s2, e2 = ms.trevc(T, nb=128)
torch.cuda.synchronize()
print(json.dumps({{"Z": bool(torch.equal(Z1, Z2)), "e": bool(torch.equal(e1, e2)), "s": bool(torch.equal(s1, s2)),
                   "rescaled": int((e2 < 0).sum().item())}}))
"""
    env = dict(os.environ, MSTRSM_DIST_TEST_UNPACK="1")
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["Z"] and r["e"] and r["s"] and r["rescaled"] > 0, r


@pytest.mark.parametrize("P,case", [(4, "c5"), (8, "c5"), (3, "c2")])
def test_trevc_dist_p_rank_layout_emulated_bit_identical(P, case):
    """The P-rank row-block gather (slab widths, offsets, the receiver's a.6 fix-up with the
    gathered E table) on one GPU: MSTRSM_DIST_EMULATE_P=P with MSTRSM_DIST_EMULATE_FULL=1 solves
    every rank's shard in turn and places its slabs, E table and exponents where the gathers would,
    so the unpack must reproduce trevc bit for bit."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    script = f"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
case = {case!r}
m, nb = (1100, 128) if case == "c5" else (700, 64)
T = inputs.c5_grcar_like(m) if case == "c5" else inputs.c2_trevc_real(m)
T = torch.from_numpy(np.asfortranarray(T)).cuda()
ms.comm_init(1, 0)
Z1, s1, e1 = ms.trevc_dist(T, m, nb=nb)
ms.comm_destroy()
Z2, s2, e2 = ms.trevc(T, nb=nb)
torch.cuda.synchronize()
print(json.dumps({{"Z": bool(torch.equal(Z1, Z2)), "e": bool(torch.equal(e1, e2)), "s": bool(torch.equal(s1, s2)),
                   "rescaled": int((e2 < 0).sum().item())}}))
"""
    env = dict(os.environ, MSTRSM_DIST_EMULATE_P=str(P), MSTRSM_DIST_EMULATE_FULL="1")
    out = subprocess.run([sys.executable, "-c", script], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["Z"] and r["e"] and r["s"], r
