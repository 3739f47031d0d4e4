"""GPU parity on the edge regimes of the diagonal-block kernels' safe path at sizes that run the
chunked / left-looking kernels with several chunks: pivots near the top of the double
range (the precheck's reciprocal bound then lands in the subnormals), a tiny diagonal under strong
coupling (Alg. 4's worst case: a rescale nearly every row, so the replay's exponent chain
and its frame bookkeeping run on every row), and a diagonal graded over 10^+-300.  Oracle =
oracle.mstrsm on the same inputs; bars as tests/test_gpu_parity.py (R20 1e-9 normwise, R21
|Delta e| <= 1)."""
import numpy as np
import pytest

import oracle
from tests.gpu_util import assert_parity, dev, host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


def _solve(ms, U, s, B, op, nb):
    import torch
    X, sc, e = ms.solve(dev(U), dev(np.ascontiguousarray(s)), dev(B), safe=True, op=op, nb=nb)
    torch.cuda.synchronize()
    return host(X), host(e)


def _case(kind, m, n, cplx, seed):
    rng = np.random.default_rng([91, kind, m, n, int(cplx), seed])
    U = np.triu(rng.standard_normal((m, m)))
    if cplx:
        U = U + 1j * np.triu(rng.standard_normal((m, m)))
    d = np.arange(m)
    if kind == 0:      # pivots in [2^1022, 2^1023) (1/|d| subnormal), off-diagonal ~ 2^1000
        U = U * 2.0 ** 1000
        U[d, d] = 2.0 ** 1022 * rng.uniform(1.0, 1.9, m)
        s = rng.uniform(-1, 1, n) * 2.0 ** 1010
    elif kind == 1:    # tiny diagonal, strong coupling: growth and a rescale nearly every row
        U = U * 1e3
        U[d, d] = 1e-3 * rng.uniform(0.5, 1.0, m)
        s = rng.uniform(-1e-4, 1e-4, n)
    else:              # diagonal graded over 10^+-300
        U[d, d] = 10.0 ** rng.uniform(-300, 300, m)
        s = rng.uniform(-1, 1, n) * 1e-300
    if cplx:
        s = s + 1j * rng.uniform(-1, 1, n) * np.abs(s)
    B = rng.standard_normal((m, n)) + (1j * rng.standard_normal((m, n)) if cplx else 0)
    return np.asfortranarray(U), np.asarray(s), np.asfortranarray(B)


@pytest.mark.parametrize("kind", [0, 1, 2])
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("nb", [64, 128])
@pytest.mark.parametrize("op", ["N", "C"])
def test_gpu_extreme_regimes(ms, kind, cplx, nb, op):
    m, n = 300, 40
    U, s, B = _case(kind, m, n, cplx, nb)
    Xg, eg = _solve(ms, U, s, B, op, nb)
    Xo, eo = oracle.mstrsm(U, s, B, safe=True, op=op, nb=nb)
    assert np.all(np.isfinite(Xg))
    assert_parity(Xg, eg, Xo, eo, what=f"extreme kind={kind} cplx={cplx} nb={nb} op={op}")
    if kind == 1:
        assert np.min(eo) < -100          # the regime rescales heavily (the point of the case)


@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_extreme_few_columns(ms, cplx):
    """Few columns (the 8-GPU shard regime: one warp per column, layout (32, 4) at n_b = 128)."""
    m, n = 640, 6
    U, s, B = _case(1, m, n, cplx, 7)
    Xg, eg = _solve(ms, U, s, B, "N", 128)
    Xo, eo = oracle.mstrsm(U, s, B, safe=True, op="N", nb=128)
    assert_parity(Xg, eg, Xo, eo, what=f"extreme few columns cplx={cplx}")
