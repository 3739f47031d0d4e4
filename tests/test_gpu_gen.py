"""GPU parity tests (-m gpu) for SURVEY §8f row f1: the generalized (safe) multi-shift solve
(Alg. 7/8) and GeneralizedTriangEig (Alg. 9) through the C ABI, against the CPU oracle on the same
seeded inputs.  Bars as for the standard solve (R20/R21): normwise 1e-9 after exponent
alignment, |e_gpu - e_orc| <= 1; bit-exact where the arithmetic is exact."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs
from tests.gpu_util import assert_parity, dev, host

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
LD, CLD = np.longdouble, np.clongdouble


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


def _upper(m, cplx, seed, diag=(1.0, 2.0), scale=1.0):
    rng = np.random.default_rng([62, m, seed])
    A = np.triu(rng.standard_normal((m, m))) * scale / np.sqrt(max(m, 1))
    if cplx:
        A = A + 1j * np.triu(rng.standard_normal((m, m))) * scale / np.sqrt(max(m, 1))
    A[np.arange(m), np.arange(m)] = rng.uniform(*diag, m)
    return np.asfortranarray(A)


def gpu_gen(ms, U, V, s, B, *, safe=True, nb=32, row_end=None):
    X, sc, e = ms.solve_gen(dev(U), dev(V), dev(np.ascontiguousarray(s)), dev(B), safe=safe, nb=nb,
                            row_end=row_end)
    _sync()
    return host(X), host(sc), host(e)


@pytest.mark.parametrize("case", GOLD["gen_solve"], ids=lambda c: c["cite"][:24])
def test_gpu_golden_generalized_solves(ms, case):
    X, _, e = gpu_gen(ms, np.array(case["U"], float), np.array(case["V"], float),
                      np.array(case["shifts"], float), np.array(case["B"], float),
                      safe=case.get("safe", True), nb=case["nb"])
    assert np.array_equal(X, np.array(case["X"], float)) and list(e) == case["e"]


@pytest.mark.parametrize("case", GOLD["tgevc"], ids=lambda c: c["cite"][:24])
def test_gpu_golden_tgevc(ms, case):
    Z, lam, _, e = ms.tgevc(dev(np.array(case["T"], float)), dev(np.array(case["S"], float)), nb=2)
    _sync()
    assert np.array_equal(host(Z), np.array(case["Z"], float))
    assert np.array_equal(host(lam), np.array(case["lambda"], float)) and list(host(e)) == case["e"]


def test_gpu_generalized_hand_rescale_cases(ms):
    """The two hand-derived P:952 / R32 cases of tests/test_oracle_gen.py, bit for bit."""
    U, V = np.eye(2), np.array([[0.0, 2.0 ** 980], [0.0, 0.0]])
    X, sc, e = gpu_gen(ms, U, V, np.array([1.0]), np.array([[0.0], [1.0]]), nb=1)
    assert int(e[0]) == -11 and np.array_equal(X[:, 0], np.array([2.0 ** 969, 2.0 ** -11]))
    U, V = np.eye(3), np.zeros((3, 3))
    V[0, 1], V[0, 2] = 2.0 ** 980, -(2.0 ** 980)
    X, sc, e = gpu_gen(ms, U, V, np.array([1.0]), np.array([[0.0], [1.0], [1.0]]), nb=2)
    assert int(e[0]) == -12 and np.array_equal(X[:, 0], np.array([0.0, 2.0 ** -12, 2.0 ** -12]))


@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_V_identity_equals_the_standard_gpu_solve(ms, cplx):
    """V = I: the generalized solve reduces to the standard one (U - s*1, U(i,l) - s*0, zero V
    products are exact).  The standard path's diagonal step sums its in-block update on the tensor
    pipe (diag_tc.cuh) and the generalized one row by row, so the two agree to rounding (R24):
    same exponents, normwise 1e-12."""
    m, n = 300, 70
    U = _upper(m, cplx, 1)
    s = inputs.random_shifts(n, cplx, 3, radius=0.9)
    B = inputs.random_rhs(m, n, cplx, 4)
    for safe in (False, True):
        Xg, _, eg = gpu_gen(ms, U, np.eye(m, dtype=U.dtype), s, B, safe=safe, nb=64)
        X, _, e = ms.solve(dev(U), dev(np.ascontiguousarray(s)), dev(B), safe=safe, nb=64)
        _sync()
        rel, de = assert_parity(Xg, eg, host(X), host(e), tol=1e-12, what="V = I")
        assert not de.any()


SHAPES = [(1, 1, 8), (7, 3, 8), (100, 37, 32), (129, 64, 64), (333, 130, 64), (257, 129, 16)]


@pytest.mark.parametrize("m,n,nb", SHAPES)
@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_generalized_ragged_shapes(ms, m, n, nb, cplx):
    U, V = _upper(m, cplx, nb), _upper(m, cplx, nb + 1, diag=(0.2, 0.6))
    s = inputs.random_shifts(n, cplx, m, radius=0.5)
    B = inputs.random_rhs(m, n, cplx, nb)
    for safe in (False, True):
        Xg, _, eg = gpu_gen(ms, U, V, s, B, safe=safe, nb=nb)
        Xo, eo = oracle.mstrsm_gen(U, V, s, B, safe=safe, nb=nb)
        assert_parity(Xg, eg, Xo, eo, what=f"gen {m}x{n} nb={nb} safe={safe}")


@pytest.mark.parametrize("sorted_", [True, False])
def test_gpu_generalized_row_end(ms, sorted_):
    m, n, nb = 200, 90, 32
    U, V = _upper(m, True, 5), _upper(m, True, 6, diag=(0.2, 0.6))
    s = inputs.random_shifts(n, True, 7, radius=0.5)
    B = inputs.random_rhs(m, n, True, 8)
    r = np.sort(np.random.default_rng(9).integers(0, m + 1, n))
    if not sorted_:
        r = np.random.default_rng(10).permutation(r)
    Xg, _, eg = gpu_gen(ms, U, V, s, B, nb=nb, row_end=r)
    Xo, eo = oracle.mstrsm_gen(U, V, s, B, nb=nb, row_end=r)
    assert_parity(Xg, eg, Xo, eo, what="gen row_end")
    for j in range(n):
        assert not Xg[r[j]:, j].any()


@pytest.mark.parametrize("cplx", [False, True])
def test_gpu_tgevc_against_oracle_heavy_rescaling(ms, cplx):
    """GeneralizedTriangEig on the g1 pencil (c5-like growth: heavy rescaling, e << 0), full
    compare, plus the generalized eigen residual of the GPU output."""
    m = 640
    T, S = inputs.g1_pencil(m=m, complex_=cplx)
    Z, lam, sc, e = ms.tgevc(dev(T), dev(S), nb=64)
    _sync()
    Z, lam, e = host(Z), host(lam), host(e)
    Zo, lo, eo = oracle.tgevc(T, S, nb=64)
    assert np.max(np.abs(lam - lo) / np.abs(lo)) <= 4 * 2.0 ** -52
    assert_parity(Z, e, Zo, eo, what="tgevc")
    assert (eo < -100).any()
    Tl, Sl, Zl = (a.astype(CLD if cplx else LD) for a in (T, S, Z))
    nT, nS = np.max(np.sum(np.abs(Tl), axis=1)), np.max(np.sum(np.abs(Sl), axis=1))
    for k in range(0, m, 7):
        v = Zl[:, k]
        r = Tl @ v - lam[k] * (Sl @ v)
        assert np.max(np.abs(r)) <= 100 * m * 2.0 ** -52 * (nT + abs(lam[k]) * nS) * np.max(np.abs(v))
