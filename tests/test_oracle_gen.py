"""Pins for the generalized oracle (Alg. 7/8 GeneralizedMultiShiftTrsm, Alg. 9 GeneralizedTriangEig;
SURVEY §8f row f1), -m "not gpu".  Each ties oracle.mstrsm_gen / oracle.tgevc to something other
than themselves: hand-derived SPEC examples, the V = I and V = cI reductions to the (already pinned)
standard oracle, mpmath dense solves, extended precision, the generalized eigen residual and LAPACK's
generalized eigenvectors.  Readings R30-R32."""
import json
import os

import mpmath
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from paper_1607_01477_b200 import inputs

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
EPS = 2.0 ** -53
LD, CLD = np.longdouble, np.clongdouble


def _upper(m, cplx, seed, diag=(1.0, 2.0), scale=1.0):
    rng = np.random.default_rng([61, m, seed])
    A = np.triu(rng.standard_normal((m, m))) * scale / np.sqrt(m)
    if cplx:
        A = A + 1j * np.triu(rng.standard_normal((m, m))) * scale / np.sqrt(m)
    A[np.arange(m), np.arange(m)] = rng.uniform(*diag, m)
    return np.asfortranarray(A)


# ----------------------------------------------------------------------------- worked examples
@pytest.mark.parametrize("case", GOLD["gen_solve"], ids=lambda c: c["cite"][:24])
def test_golden_generalized_solves(case):
    U, V = np.array(case["U"], float), np.array(case["V"], float)
    X, e = oracle.mstrsm_gen(U, V, np.array(case["shifts"], float), np.array(case["B"], float),
                             nb=case["nb"], safe=case.get("safe", True))
    assert np.array_equal(X, np.array(case["X"], float)) and list(e) == case["e"]


@pytest.mark.parametrize("case", GOLD["tgevc"], ids=lambda c: c["cite"][:24])
def test_golden_tgevc(case):
    Z, lam, e = oracle.tgevc(np.array(case["T"], float), np.array(case["S"], float), nb=2)
    assert np.array_equal(Z, np.array(case["Z"], float))
    assert np.array_equal(lam, np.array(case["lambda"], float)) and list(e) == case["e"]


# ----------------------------------------------------------------------------- reductions
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("safe", [False, True])
def test_V_identity_reduces_to_the_standard_solve_bitwise(cplx, safe):
    """V = I gives Alg. 3 / Alg. 5 exactly (U - s*1 = U - s and U(i,l) - s*0 =
    U(i,l) in IEEE arithmetic; the V update adds exact zeros).  No exact zero pivots here (the
    delta of R31 differs from R4's by the |s| ||V|| term)."""
    m, n = 90, 17
    U = _upper(m, cplx, 1)
    s = inputs.random_shifts(n, cplx, 3, center=0.0, radius=0.9)
    B = inputs.random_rhs(m, n, cplx, 4)
    for nb in (1, 7, 32):
        Xg, eg = oracle.mstrsm_gen(U, np.eye(m), s, B, nb=nb, safe=safe)
        Xs, es = oracle.mstrsm(U, s, B, nb=nb, safe=safe)
        assert np.array_equal(Xg, Xs) and np.array_equal(eg, es)


def test_V_identity_reduction_with_heavy_rescaling_and_row_end():
    """The eigenvector RHS of the c5 shape (heavy rescaling, the P:503-508 shortcut): V = I
    reproduces TriangEig's solve bit for bit, including every scale exponent."""
    T = inputs.c5_grcar_like(m=300)
    m = T.shape[0]
    cols = np.arange(m)
    B = np.zeros((m, m), dtype=complex, order="F")
    for k in range(m):
        B[:k, k] = -T[:k, k]
    Xg, eg = oracle.mstrsm_gen(T, np.eye(m, dtype=complex), np.diag(T).copy(), B, nb=32, row_end=cols)
    Xs, es = oracle.mstrsm(T, np.diag(T).copy(), B, nb=32, row_end=cols)
    assert np.array_equal(Xg, Xs) and np.array_equal(eg, es)
    assert (es < -100).any()


def test_V_scalar_multiple_of_identity_is_a_shift_rescaling():
    """V = c I: (U - s c I) is the standard solve with shift s*c (same rounding of s*c)."""
    m, n = 70, 11
    U = _upper(m, True, 2)
    s = inputs.random_shifts(n, True, 5, radius=0.6)
    B = inputs.random_rhs(m, n, True, 6)
    c = 0.75 - 0.25j
    Xg, eg = oracle.mstrsm_gen(U, c * np.eye(m), s, B, nb=16)
    sc = np.array([complex(v.real * c.real - v.imag * c.imag, v.real * c.imag + v.imag * c.real) for v in s])
    Xs, es = oracle.mstrsm(U, sc, B, nb=16)
    assert np.array_equal(Xg, Xs) and np.array_equal(eg, es)


def test_S_identity_reduces_tgevc_to_trevc():
    """S = I -> GeneralizedTriangEig = TriangEig (lambda = T(k,k)/1; Z RHS 0*lambda - T = -T)."""
    T = inputs.c5_grcar_like(m=260)
    Zg, lam, eg = oracle.tgevc(T, np.eye(260, dtype=complex), nb=32)
    Zs, es = oracle.trevc(T, nb=32)
    assert np.array_equal(lam, np.diag(T)) and np.array_equal(Zg, Zs) and np.array_equal(eg, es)


# ----------------------------------------------------------------------------- exact solutions
@pytest.mark.parametrize("m", [1, 2, 5, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_tiny_m_against_mpmath_dense_generalized_solve(m, cplx):
    mpmath.mp.dps = 50
    U, V = _upper(m, cplx, 7), _upper(m, cplx, 8, diag=(0.2, 0.6))
    n = 4
    s = inputs.random_shifts(n, cplx, 9, radius=0.5)
    B = inputs.random_rhs(m, n, cplx, 10)
    for safe in (False, True):
        X, e = oracle.mstrsm_gen(U, V, s, B, nb=3, safe=safe)
        assert not e.any()
        for j in range(n):
            A = mpmath.matrix(m, m)
            for i in range(m):
                for k in range(m):
                    A[i, k] = mpmath.mpc(complex(U[i, k])) - mpmath.mpc(complex(s[j])) * mpmath.mpc(complex(V[i, k]))
            x = mpmath.lu_solve(A, mpmath.matrix([mpmath.mpc(complex(b)) for b in B[:, j]]))
            xe = np.array([complex(v) for v in x])
            assert np.max(np.abs(X[:, j] - xe)) <= 1e-13 * max(np.max(np.abs(xe)), 1e-300)


def _backsub_gen_longdouble(U, V, lam, b, r):
    cp = True
    A = (np.asarray(U)[:r, :r].astype(CLD) - CLD(lam) * np.asarray(V)[:r, :r].astype(CLD))
    x = np.asarray(b)[:r].astype(CLD).copy()
    for l in range(r - 1, -1, -1):
        x[l] = x[l] / A[l, l]
        x[:l] -= x[l] * A[:l, l]
    return x


def test_tgevc_extended_precision_pin():
    """Scaled safe generalized solve vs the unscaled long-double back substitution of
    (T - lambda_k S) z = -T(:k,k) + lambda_k S(:k,k): normwise after exponent alignment."""
    T, S = inputs.g1_pencil(m=400)
    cols = [100, 200, 300, 399]
    Z, lam, e = oracle.tgevc(T, S, nb=64, cols=cols)
    rescaled = 0
    for q, k in enumerate(cols):
        rhs = S[:k, k] * lam[q] - T[:k, k]
        xt = _backsub_gen_longdouble(T, S, lam[q], rhs, k)
        xs = Z[:k, q].astype(CLD) * np.ldexp(LD(1.0), -int(e[q]))
        assert float(np.max(np.abs(xs - xt)) / np.max(np.abs(xt))) <= 1e-11
        rescaled += e[q] < 0
    assert rescaled >= 2


@pytest.mark.parametrize("cplx", [False, True])
def test_tgevc_generalized_eigen_residual(cplx):
    """||T z_k - lambda_k S z_k||_inf <= 100 m eps (||T|| + |lambda_k| ||S||) ||z_k|| (the P:770-772
    bound carried to the pencil), incl. heavily rescaled columns; Z upper triangular, diag = c."""
    m = 300
    T, S = inputs.g1_pencil(m=m, complex_=cplx)
    Z, lam, e = oracle.tgevc(T, S, nb=32)
    Tl, Sl, Zl = (a.astype(CLD if cplx else LD) for a in (T, S, Z))
    nT, nS = np.max(np.sum(np.abs(Tl), axis=1)), np.max(np.sum(np.abs(Sl), axis=1))
    for k in range(m):
        v = Zl[:, k]
        r = Tl @ v - lam[k] * (Sl @ v)
        assert np.max(np.abs(r)) <= 100 * m * 2.0 ** -52 * (nT + abs(lam[k]) * nS) * np.max(np.abs(v))
    assert np.array_equal(np.triu(Z), Z)
    assert np.array_equal(np.diag(Z), np.ldexp(1.0, e).astype(Z.dtype))
    ref = np.diag(T) / np.diag(S)                        # numpy's complex divide != Smith's to the ulp
    assert np.max(np.abs(lam - ref) / np.abs(ref)) <= 4 * EPS
    assert (e < -50).any()


def test_tgevc_matches_lapack_generalized_eigenvectors():
    """Directions vs scipy.linalg.eig(T, S) (LAPACK zggev) on a small well-conditioned pencil."""
    m = 25
    rng = np.random.default_rng(11)
    T = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) * 0.2
    T[np.arange(m), np.arange(m)] = np.exp(2j * np.pi * np.arange(m) / m) * (1 + np.arange(m) / m)
    S = np.triu(rng.standard_normal((m, m))) * 0.1
    S[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m)
    Z, lam, _ = oracle.tgevc(T, S, nb=8)
    w, Vr = sla.eig(T, S)
    for k in range(m):
        j = int(np.argmin(np.abs(w - lam[k])))
        a, b = Z[:, k] / np.linalg.norm(Z[:, k]), Vr[:, j] / np.linalg.norm(Vr[:, j])
        ph = np.vdot(b, a)
        assert abs(abs(ph) - 1) < 1e-10 and np.linalg.norm(a - ph * b) < 1e-9


def test_generalized_rescale_branch_column_bound_with_V_term():
    """Hand case for the panel term of P:952 with |lambda| ||V(I0,k)||: U = [[1, 0], [0, 1]],
    V = [[0, 2^980], [0, 0]], lambda = 1, b = [0, 1], n_b = 1.  Block {2}: x2 = 1 (U' = 1);
    G = 1 + (0 + 1 * 2^980) * 1 >= Omega -> k = 11, x = (0, 2^-11), c = 2^-11; then
    x1 = 0 - U(1,2) x2 + V(1,2) (lambda x2) = 2^980 * 2^-11 = 2^969, and (U - V) x = c b exactly."""
    U = np.eye(2)
    V = np.array([[0.0, 2.0 ** 980], [0.0, 0.0]])
    X, e = oracle.mstrsm_gen(U, V, np.array([1.0]), np.array([[0.0], [1.0]]), nb=1)
    assert int(e[0]) == -11
    assert np.array_equal(X[:, 0], np.array([2.0 ** 969, 2.0 ** -11]))
    # R32: C is formed after the rescale; forming it before would give x1 = 2^980 (inconsistent)
    assert np.array_equal((U - V) @ X[:, 0], np.ldexp(1.0, -11) * np.array([0.0, 1.0]))


def test_generalized_panel_term_alone_triggers_the_column_rescale():
    """Only the panel bound of P:952 can trigger here (the actual contributions cancel): m = 3,
    U = I, V(1,2) = 2^980, V(1,3) = -2^980, lambda = 1, b = (0, 1, 1), n_b = 2.  Block {2,3}:
    x2 = x3 = 1, G = 1 + (0 + 2^980) + (0 + 2^980) = 2^981 -> k = 12; C = lambda x(I1) = 2^-12 (1, 1);
    x1 = V(1,2) C2 + V(1,3) C3 = 0 exactly.  Result e = -12, x = (0, 2^-12, 2^-12); dropping the
    |lambda| ||V|| term would leave e = 0."""
    U = np.eye(3)
    V = np.zeros((3, 3))
    V[0, 1], V[0, 2] = 2.0 ** 980, -(2.0 ** 980)
    X, e = oracle.mstrsm_gen(U, V, np.array([1.0]), np.array([[0.0], [1.0], [1.0]]), nb=2)
    assert int(e[0]) == -12
    assert np.array_equal(X[:, 0], np.array([0.0, 2.0 ** -12, 2.0 ** -12]))
    assert np.array_equal((U - V) @ X[:, 0], np.ldexp(1.0, -12) * np.array([0.0, 1.0, 1.0]))
