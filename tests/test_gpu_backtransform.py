"""GPU parity tests (-m gpu) for SURVEY §8f row f2, the back-transformation of Eig:
trevc_qz (TriangEig then X = Q Z) and eig_backtransform (X = Q Z, TRMM-shaped DMMA panels)
through the C ABI against the CPU oracle on the same seeded inputs.  Bar as for TriangEig
(R20/R21): normwise 1e-9 after exponent alignment, |e_gpu - e_orc| <= 1."""
import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs
from tests.gpu_util import assert_parity, dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


def _sync():
    import torch
    torch.cuda.synchronize()


# m = 1100 spans two 1024-column panels (the second with K = m)
CASES = [(1, 8), (7, 8), (100, 32), (333, 64), (1100, 128)]


@pytest.mark.parametrize("m,nb", CASES)
@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_trevc_qz_parity(ms, m, nb, cplx):
    T, Q = inputs.schur_pair(m, cplx, seed=nb)
    X, sc, e = ms.trevc_qz(dev(T), dev(Q), nb=nb)
    _sync()
    Xo, eo = oracle.trevc_qz(T, Q, nb=nb)
    assert_parity(host(X), host(e), Xo, eo, what=f"trevc_qz m={m} nb={nb}")
    assert np.array_equal(host(sc), np.ldexp(1.0, host(e)))


def test_gpu_trevc_qz_heavy_rescaling(ms):
    """Config-5 growth (e << 0) through the back-transformation."""
    m = 640
    T = inputs.c5_grcar_like(m)
    _, Q = inputs.schur_pair(m, True, seed=5)
    X, _, e = ms.trevc_qz(dev(T), dev(Q), nb=64)
    _sync()
    Xo, eo = oracle.trevc_qz(T, Q, nb=64)
    assert (eo < -300).any()
    assert_parity(host(X), host(e), Xo, eo, what="trevc_qz c5")


@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_backtransform_column_subset(ms, cplx):
    """X = Q Z for a Z that is zero below row cols[q] in column q (trevc_*_cols layout); every
    entry against the fp64 product, per-column normwise."""
    m, n = 700, 150
    rng = np.random.default_rng(21)
    cols = np.sort(rng.choice(m, n, replace=False)).astype(np.int64)
    Z = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
    for q, c in enumerate(cols):
        Z[c + 1:, q] = 0
    _, Q = inputs.schur_pair(m, cplx, seed=3)
    X = host(ms.eig_backtransform(dev(Q), dev(Z), cols=cols))
    _sync()
    Xo = oracle.eig_backtransform(Q, Z)
    rel = np.max(np.abs(X - Xo), axis=0) / np.max(np.abs(Xo), axis=0)
    assert rel.max() <= 1e-12


@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_backtransform_identity(ms, cplx):
    """Q = I: real X = Z bit for bit (0 - sum of exact products, negated); complex within the
    rounding of the three-product form (Re exact, Im = (Zr + Zi) - Zr)."""
    m = 260
    T = inputs.c3_trevc_complex(m) if cplx else inputs.c2_trevc_real(m)
    Z, _, _ = ms.trevc(dev(T), nb=64)
    X = ms.eig_backtransform(dev(np.eye(m, dtype=T.dtype)), Z)
    _sync()
    Zh, Xh = host(Z), host(X)
    if cplx:
        assert np.array_equal(Xh.real, Zh.real)
        assert np.max(np.abs(Xh.imag - Zh.imag)) <= 2.0 ** -52 * np.max(np.abs(Zh))
    else:
        assert np.array_equal(Xh, Zh)


def test_gpu_backtransform_argument_errors(ms):
    import torch
    Q = torch.zeros((4, 4), dtype=torch.float64, device="cuda").t()      # column-major
    Z = torch.zeros((5, 4), dtype=torch.float64, device="cuda").t()
    with pytest.raises(ms.MstrsmError):
        ms.eig_backtransform(Q, Z)                      # n > m needs explicit row bounds
    with pytest.raises(ms.MstrsmError):
        ms.eig_backtransform(Q, Z, cols=[0, 1, 1, 2, 3])   # not strictly increasing
