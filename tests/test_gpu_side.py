"""GPU parity tests (-m gpu) for SURVEY §8f row f4 (P:58-62 footnote): left/right x
upper/lower multi-shift solves through the C ABI against the CPU oracle.  Bars as the standard
solve (R20/R21): normwise 1e-9 after exponent alignment, |e_gpu - e_orc| <= 1."""
import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs
from tests.gpu_util import assert_parity, dev, host

pytestmark = pytest.mark.gpu

CASES = [("L", "U"), ("L", "L"), ("R", "U"), ("R", "L")]


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


def _tri(m, uplo, cplx, seed, growth=False):
    rng = np.random.default_rng([41, m, seed])
    A = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    if growth:
        A = A * 4.0
        A[np.arange(m), np.arange(m)] = rng.uniform(-1e-3, 1e-3, m)
    else:
        A = A / np.sqrt(m)
        A[np.arange(m), np.arange(m)] = rng.uniform(1.0, 2.0, m)
    return np.asfortranarray(np.triu(A) if uplo == "U" else np.tril(A))


@pytest.mark.parametrize("side,uplo", CASES)
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("m,n,nb,growth", [(1, 1, 8, False), (75, 40, 16, False), (333, 129, 64, True)])
def test_gpu_side_parity(ms, side, uplo, cplx, m, n, nb, growth):
    A = _tri(m, uplo, cplx, nb, growth)
    s = inputs.random_shifts(n, cplx, m + nb, radius=1e-3 if growth else 0.5)
    B = inputs.random_rhs(m, n, cplx, nb)
    if side == "R":
        B = np.asfortranarray(B.T)
    for safe in (False, True) if not growth else (True,):
        Xg, _, eg = ms.solve_side(dev(A), dev(np.ascontiguousarray(s)), dev(B), side=side, uplo=uplo,
                                  safe=safe, nb=nb)
        import torch
        torch.cuda.synchronize()
        Xo, eo = oracle.mstrsm_side(A, s, B, side=side, uplo=uplo, safe=safe, nb=nb)
        Xg, eg = host(Xg), host(eg)
        if side == "R":
            Xg, Xo = Xg.T, Xo.T
        assert_parity(Xg, eg, Xo, eo, what=f"{side}{uplo} m={m} safe={safe}")
        if growth:
            assert (eo < 0).any()


def test_gpu_side_left_upper_is_the_standard_solve(ms):
    m, n = 200, 50
    A = _tri(m, "U", True, 3)
    s = inputs.random_shifts(n, True, 7, radius=0.5)
    B = inputs.random_rhs(m, n, True, 8)
    X1, _, e1 = ms.solve_side(dev(A), dev(np.ascontiguousarray(s)), dev(B), side="L", uplo="U", nb=32)
    X2, _, e2 = ms.solve(dev(A), dev(np.ascontiguousarray(s)), dev(B), safe=True, nb=32)
    import torch
    torch.cuda.synchronize()
    assert np.array_equal(host(X1), host(X2)) and np.array_equal(host(e1), host(e2))
