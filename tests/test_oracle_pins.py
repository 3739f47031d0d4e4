"""Pins for the CPU oracle (-m "not gpu").  Each test ties an oracle function to something
other than itself: hand-derived values, closed forms, LAPACK/SVD/mpmath, extended precision,
identities.  A plausible mistake anywhere in oracle/ (a dropped term, wrong sign or index, a
transposed operand, a wrong threshold) fails at least one of them.  See DESIGN.md §4.
"""
import json
import os

import mpmath
import numpy as np
import pytest
import scipy.linalg as sla

import oracle
from paper_1607_01477_b200 import inputs
from tests import refmath as R

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
EPS = 2.0 ** -53


def _num(v):
    if isinstance(v, str):
        sgn = -1.0 if v.startswith("-") else 1.0
        return sgn * 2.0 ** float(v.lstrip("-").split("^")[1])
    return float(v)


def _cplx(v):
    return complex(v[0], v[1])


# ----------------------------------------------------------------------------- scalar helpers
def test_zmod_matches_mpmath_and_is_scale_exact():
    rng = np.random.default_rng(7)
    for _ in range(2000):
        ex = rng.integers(-1070, 1020)
        re, im = rng.standard_normal(2) * 2.0 ** ex
        exact = mpmath.sqrt(mpmath.mpf(re) ** 2 + mpmath.mpf(im) ** 2)
        got = oracle.zmod(complex(re, im))
        assert abs(mpmath.mpf(got) - exact) <= max(1.01 * mpmath.mpf(2.0 ** -52) * exact,
                                                  mpmath.mpf(2.0 ** -1074))
    assert oracle.zmod(3 + 4j) == 5.0
    assert oracle.zmod(complex(3 * 2.0 ** 1000, 4 * 2.0 ** 1000)) == 5 * 2.0 ** 1000
    assert oracle.zmod(complex(3 * 2.0 ** -1060, 4 * 2.0 ** -1060)) == 5 * 2.0 ** -1060
    for x in (1.0, -2.5e-310, 7e300):   # |x + 0i| = |x| exactly (real == complex with im = 0)
        assert oracle.zmod(complex(x, 0.0)) == abs(x)


def test_zdiv_matches_mpmath():
    rng = np.random.default_rng(8)
    mpmath.mp.dps = 40
    for _ in range(2000):
        a = complex(*rng.standard_normal(2)) * 2.0 ** rng.integers(-200, 200)
        b = complex(*rng.standard_normal(2)) * 2.0 ** rng.integers(-200, 200)
        q = oracle.zdiv(a, b)
        exact = mpmath.mpc(a) / mpmath.mpc(b)
        assert abs(mpmath.mpc(q) - exact) <= 8 * EPS * abs(exact)
    assert oracle.zdiv(6 + 0j, 2 + 0j) == 3 + 0j


def test_minpow2_definition_brute_force():
    rng = np.random.default_rng(9)
    for _ in range(3000):
        L = 2.0 ** rng.integers(-100, 960) * rng.uniform(0.5, 1.0)
        a = L * 2.0 ** rng.uniform(0, 50)
        k = oracle.minpow2(a, L)
        assert k >= 1
        assert np.ldexp(a, -k) < L
        if k > 1:
            assert not (np.ldexp(a, -(k - 1)) < L)
    assert oracle.minpow2(2.0 ** 971, 2.0 ** 970) == 2          # 2^970 is not < Omega
    assert oracle.minpow2(1.0, 2.0 ** -52) == 53


# ----------------------------------------------------------------------------- worked examples
@pytest.mark.parametrize("case", GOLD["solve"], ids=lambda c: c["cite"][:24])
def test_golden_solves(case):
    U = np.array(case["U"], dtype=float)
    B = np.array(case["B"], dtype=float)
    X, e = oracle.mstrsm(U, np.array(case["shifts"], float), B, safe=True, nb=case["nb"])
    assert np.array_equal(X, np.array(case["X"], dtype=float)) or np.allclose(X, case["X"], rtol=1e-15)
    assert list(e) == case["e"]
    if "X_exact_log2" in case:
        assert X[0, 0] == 2.0 ** case["X_exact_log2"][0]
    piv = np.diag(U)[:, None] - np.array(case["shifts"], float)[None, :]
    if all(v == 0 for v in case["e"]) and np.all(piv != 0):   # no rescale, no delta -> plain == safe
        Xp, _ = oracle.mstrsm(U, np.array(case["shifts"], float), B, safe=False, nb=case["nb"])
        assert np.array_equal(Xp, X)


def test_golden_complex_solve():
    case = GOLD["solve_complex"][0]
    U = np.array([[_cplx(v) for v in row] for row in case["U"]])
    B = np.array([[_cplx(v) for v in row] for row in case["B"]])
    X, e = oracle.mstrsm(U, [0j], B, safe=True, nb=2)
    assert np.array_equal(X, np.array([[_cplx(v) for v in row] for row in case["X"]]))
    assert list(e) == case["e"]


@pytest.mark.parametrize("case", GOLD["rescale_pins"], ids=lambda c: c["cite"][:20])
def test_rescale_pins_exact(case):
    """One exact pin per rescale branch of Alg. 4 / Alg. 5 (hand-derived)."""
    U = np.array([[_num(v) for v in row] for row in case["U"]])
    X, e = oracle.mstrsm(U, [0.0], np.array(case["B"], float), safe=True, nb=case["nb"])
    assert int(e[0]) == case["e"]
    assert np.array_equal(X[:, 0], np.array([_num(v) for v in case["X"]]))
    # The scaled pair still solves the (well-posed part of the) system: U x = c b.
    assert np.all(np.abs(X) < R.OMEGA)


def test_rescale_pin_sigma_matches_analytic_solution():
    """x = c (-s^-2, s^-1) to the last digit (mpmath)."""
    s = 1e-300
    X, e = oracle.mstrsm(np.array([[s, 1.0], [0.0, s]]), [0.0], [0.0, 1.0], nb=2)
    c = mpmath.ldexp(1, int(e[0]))
    sm = mpmath.mpf(s)
    assert abs(mpmath.mpf(X[0, 0]) - c * (-1 / sm ** 2)) <= 2 * EPS * abs(c / sm ** 2)
    assert abs(mpmath.mpf(X[1, 0]) - c / sm) <= 2 * EPS * abs(c / sm)


@pytest.mark.parametrize("case", GOLD["column_norms"], ids=lambda c: c["cite"])
def test_golden_column_norms(case):
    U = np.array(case["U"], float)
    cnl, P, un = oracle.norms(U, op="N", nb=U.shape[0])          # one block: cnl = full norms
    assert list(cnl) == case["cnl_nb_inf"]
    assert P[0] == 0.0
    assert un == np.max(np.sum(np.abs(np.triu(U)), axis=1))


def test_norm_pass_panel_sums_by_definition():
    """P_b = sum_{k in I1} ||U(I0,k)||_inf and block-local cnl, evaluated by brute force."""
    U, _, _ = inputs.c1_plain_real(m=37, n=1)
    nb = 8
    cnl, P, _ = oracle.norms(U, op="N", nb=nb)
    m = 37
    for b in range((m + nb - 1) // nb):
        hi = m - b * nb
        lo = max(0, hi - nb)
        assert P[b] == pytest.approx(sum(np.max(np.abs(U[:lo, k])) if lo else 0.0 for k in range(lo, hi)),
                                     rel=1e-15)
        for k in range(lo, hi):
            assert cnl[k] == (np.max(np.abs(U[lo:k, k])) if k > lo else 0.0)


@pytest.mark.parametrize("case", GOLD["trevc"], ids=lambda c: c["cite"][:10])
def test_golden_trevc(case):
    Z, e = oracle.trevc(np.array(case["T"], float), nb=2)
    assert np.array_equal(Z, np.array(case["Z"], float))
    assert list(e) == case["e"]


@pytest.mark.parametrize("case", GOLD["pseudospectra"], ids=lambda c: c["cite"][:10])
def test_golden_pseudospectra(case):
    U = np.array(case["U"], dtype=complex)
    z = np.array([_cplx(v) for v in case["z"]])
    v0 = np.ones(U.shape[0], complex) / np.sqrt(U.shape[0])
    sig, flags = oracle.pseudospectra(U, z, iters=15, v0=v0, nb=1)
    assert np.allclose(sig, case["sigma"], rtol=1e-13)
    assert not flags.any()


# ----------------------------------------------------------------------------- plain solve
def test_diagonal_U_is_exact_division_real():
    rng = np.random.default_rng(11)
    m, n = 40, 9
    d = rng.uniform(1, 2, m)
    U = np.diag(d)
    s = rng.uniform(-0.5, 0.5, n)
    B = rng.standard_normal((m, n))
    for safe in (False, True):
        X, e = oracle.mstrsm(U, s, B, safe=safe, nb=7)
        assert np.array_equal(X, B / (d[:, None] - s[None, :]))   # correctly-rounded division
        assert not e.any()


def test_diagonal_U_complex_within_ulps():
    rng = np.random.default_rng(12)
    m, n = 30, 5
    d = rng.standard_normal(m) + 1j * rng.standard_normal(m) + 3
    s = inputs.random_shifts(n, True, 1)
    B = inputs.random_rhs(m, n, True, 1)
    X, _ = oracle.mstrsm(np.diag(d), s, B, safe=True, nb=4)
    mpmath.mp.dps = 40
    for i in range(m):
        for j in range(n):
            ex = mpmath.mpc(B[i, j]) / (mpmath.mpc(d[i]) - mpmath.mpc(s[j]))
            assert abs(mpmath.mpc(X[i, j]) - ex) <= 8 * EPS * abs(ex)


@pytest.mark.parametrize("cplx", [False, True])
def test_zero_shift_equals_lapack_trtrs(cplx):
    """Alg. 2 reduction: zero shifts is the ordinary triangular solve (LAPACK ?trtrs)."""
    if cplx:
        U = inputs.e1_hermitian_triangle(120, seed=1)
        B = inputs.random_rhs(120, 11, True, 2)
    else:
        U, _, B = inputs.c1_plain_real(m=150, n=13)
    n = B.shape[1]
    X, e = oracle.mstrsm(U, np.zeros(n, dtype=U.dtype), B, safe=True, nb=32)
    ref = sla.solve_triangular(U, B)
    assert not e.any()
    assert np.max(np.abs(X - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("m", [1, 2, 3, 5, 8])
@pytest.mark.parametrize("cplx", [False, True])
def test_tiny_m_against_mpmath_dense_solve(m, cplx):
    rng = np.random.default_rng([13, m, int(cplx)])
    U = np.triu(rng.standard_normal((m, m)))
    if cplx:
        U = U + 1j * np.triu(rng.standard_normal((m, m)))
    U[np.arange(m), np.arange(m)] += 3.0
    s = inputs.random_shifts(3, cplx, m)
    B = inputs.random_rhs(m, 3, cplx, m)
    mpmath.mp.dps = 50
    for safe in (False, True):
        for nb in (1, 2, m):
            X, e = oracle.mstrsm(U, s, B, safe=safe, nb=nb)
            for j in range(3):
                A = mpmath.matrix([[mpmath.mpc(U[i, k]) if k >= i else 0 for k in range(m)] for i in range(m)])
                for i in range(m):
                    A[i, i] -= mpmath.mpc(s[j])
                xe = mpmath.lu_solve(A, mpmath.matrix([mpmath.mpc(v) for v in B[:, j]]))
                nrm = max(abs(v) for v in xe)
                err = max(abs(mpmath.mpc(X[i, j]) - xe[i]) for i in range(m))
                assert err <= 1e-13 * nrm


def test_block_size_invariance():
    """Blocked == unblocked up to rounding: nb = 1, 7, 32, m."""
    U, s, B = inputs.c1_plain_real(m=96, n=10)
    ref, _ = oracle.mstrsm(U, s, B, safe=False, nb=1)
    for nb in (7, 32, 96):
        X, _ = oracle.mstrsm(U, s, B, safe=False, nb=nb)
        assert np.max(np.abs(X - ref)) <= 100 * EPS * 96 * np.max(np.abs(ref))


def test_safe_equals_plain_bitwise_when_no_rescale():
    """c = 1 -> the safe path is exactly the plain path (config 1 never rescales)."""
    U, s, B = inputs.c1_plain_real(m=256, n=64)
    Xs, e = oracle.mstrsm(U, s, B, safe=True, nb=32)
    Xp, _ = oracle.mstrsm(U, s, B, safe=False, nb=32)
    assert not e.any()
    assert np.array_equal(Xs, Xp)


def test_shift_permutation_equivariance():
    U, s, B = inputs.c1_plain_real(m=64, n=12)
    perm = np.random.default_rng(3).permutation(12)
    X, e = oracle.mstrsm(U, s, B, nb=16)
    Xp, ep = oracle.mstrsm(U, s[perm], B[:, perm], nb=16)
    assert np.array_equal(X[:, perm], Xp) and np.array_equal(e[perm], ep)


# ----------------------------------------------------------------------------- op C
def _flip(U):
    return np.asfortranarray(U.conj().T[::-1, ::-1])


@pytest.mark.parametrize("kind", ["c1", "c3", "c5", "adversarial"])
def test_op_C_flip_identity_bitwise(kind):
    """solve_C(U, s, b) = J solve_N(J U^H J, conj(s), J b), bit for bit, incl. (x, e)."""
    if kind == "c1":
        U, s, B = inputs.c1_plain_real(m=70, n=9)
    elif kind == "c3":
        U = inputs.c3_trevc_complex(m=150)
        s = np.diag(U)[::7].copy()
        B = inputs.random_rhs(150, s.shape[0], True, 3)
    elif kind == "c5":
        U = inputs.c5_grcar_like(m=300)
        s = np.diag(U)[5::9].copy() + 1e-9
        B = inputs.random_rhs(300, s.shape[0], True, 4)
    else:
        U = np.triu(np.random.default_rng(5).standard_normal((41, 41)))
        U[np.arange(41), np.arange(41)] = 10.0 ** np.random.default_rng(6).uniform(-300, 3, 41)
        U[3, 3] = 0.0
        s = np.array([0.0, 1e-290, U[7, 7]])
        B = inputs.random_rhs(41, 3, False, 5)
    for nb in (8, 32):
        XC, eC = oracle.mstrsm(U, s, B, op="C", safe=True, nb=nb)
        XN, eN = oracle.mstrsm(_flip(U), np.conj(s), B[::-1], op="N", safe=True, nb=nb)
        assert np.array_equal(XC, XN[::-1])
        assert np.array_equal(eC, eN)
        if kind in ("c1", "c3"):          # the plain (Alg. 3) variant mirrors too
            XC, _ = oracle.mstrsm(U, s, B, op="C", safe=False, nb=nb)
            XN, _ = oracle.mstrsm(_flip(U), np.conj(s), B[::-1], op="N", safe=False, nb=nb)
            assert np.array_equal(XC, XN[::-1], equal_nan=True)
    if kind in ("c5", "adversarial"):
        assert (eC < 0).all()          # the rescale branches are exercised by the identity


@pytest.mark.parametrize("safe", [False, True])
@pytest.mark.parametrize("cplx", [False, True])
def test_op_C_against_lapack_on_shifted_matrix(cplx, safe):
    if cplx:
        U = inputs.e1_hermitian_triangle(90, seed=2)
        s = inputs.random_shifts(6, True, 7, center=0.0, radius=0.4)
        B = inputs.random_rhs(90, 6, True, 7)
    else:
        U, s, B = inputs.c1_plain_real(m=90, n=6)
    X, e = oracle.mstrsm(U, s, B, op="C", safe=safe, nb=16)
    assert not e.any()
    for j in range(B.shape[1]):
        ref = sla.solve_triangular(R.shifted(U, s[j]), B[:, j], trans="C")
        assert np.max(np.abs(X[:, j] - ref)) <= 1e-12 * np.max(np.abs(ref))


# ----------------------------------------------------------------------------- safe solve
def _adversarial_suite():
    rng = np.random.default_rng(21)
    cases = []
    for t in range(50):
        m = int(rng.integers(2, 40))
        kind = t % 5
        if kind == 0:        # Jordan block, shift on the eigenvalue
            U = np.eye(m) * 0.5 + np.diag(np.ones(m - 1), 1)
            s = [0.5, 0.5 + 1e-12, 0.0]
        elif kind == 1:      # exact zero pivots
            U = np.triu(rng.standard_normal((m, m)))
            U[rng.integers(0, m, 3), rng.integers(0, m, 3)] = 0.0
            U = np.triu(U)
            s = [0.0, U[m // 2, m // 2], 1.0]
        elif kind == 2:      # graded 10^+-300
            U = np.triu(rng.standard_normal((m, m)))
            U[np.arange(m), np.arange(m)] = 10.0 ** rng.uniform(-300, 300, m)
            s = [0.0, 1e-300, -1.0]
        elif kind == 3:      # repeated eigenvalues
            U = np.triu(rng.standard_normal((m, m)))
            U[np.arange(m), np.arange(m)] = 1.0
            s = [1.0, 1.0 - 1e-15, 2.0]
        else:                # tiny diagonal, strong coupling (Alg. 4 worst case)
            U = np.triu(rng.standard_normal((m, m))) * 1e3
            U[np.arange(m), np.arange(m)] = 1e-3 * rng.uniform(0.5, 1.0, m)
            s = [0.0, 1e-3, 1e-4]
        B = rng.standard_normal((m, len(s)))
        cases.append((U, np.array(s, float), B, int(rng.integers(1, 9))))
    return cases


def test_safety_invariants_adversarial():
    """finite outputs, c in [0,1], ||x|| < Omega, small backward error."""
    for U, s, B, nb in _adversarial_suite():
        m = U.shape[0]
        X, e = oracle.mstrsm(U, s, B, safe=True, nb=nb)
        assert np.all(np.isfinite(X))
        assert np.all(e <= 0)
        assert np.max(np.abs(X)) < R.OMEGA
        # delta-perturbed system: replace exact-zero pivots of U - sI by delta
        unorm = np.max(np.sum(np.abs(np.triu(U)), axis=1))
        delta = np.ldexp(unorm, -52) if unorm > 0 else np.finfo(float).tiny
        for j in range(len(s)):
            Ud = np.triu(U).copy()
            dd = Ud[np.arange(m), np.arange(m)] - s[j]
            Ud[np.arange(m), np.arange(m)] = np.where(dd == 0, delta + s[j], Ud[np.arange(m), np.arange(m)])
            if np.any((dd == 0) & (delta + s[j] - s[j] != delta)):
                continue   # s + delta - s not exact in fp64: skip the residual for that column
            r = R.residual_ratio(Ud, s[j], X[:, j], e[j], B[:, j])
            assert r <= 64 * m * 2.0 ** -53, (m, j, r)


def test_direction_invariance_b_to_2b():
    """b -> 2b gives a parallel solution."""
    for U, s, B, nb in _adversarial_suite()[:25]:
        X1, e1 = oracle.mstrsm(U, s, B, nb=nb)
        X2, e2 = oracle.mstrsm(U, s, 2 * B, nb=nb)
        for j in range(len(s)):
            a = X1[:, j] * np.ldexp(1.0, int(e2[j]) - int(e1[j]) + 1)
            nrm = np.max(np.abs(X2[:, j]))
            if nrm > 0:
                assert np.max(np.abs(a - X2[:, j])) <= 1e-12 * nrm


@pytest.mark.parametrize("gen,m,nb", [("c2", 300, 64), ("c3", 320, 128), ("c5", 512, 128)])
def test_extended_precision_pin_eigen_rhs(gen, m, nb):
    """Scaled safe solve vs the unscaled long-double back substitution (exponent range
    2^+-16382): normwise after exponent alignment, plus e <= 970 - floor(log2 ||x_true||)."""
    T = {"c2": inputs.c2_trevc_real, "c3": inputs.c3_trevc_complex, "c5": inputs.c5_grcar_like}[gen](m=m)
    cols = [m // 4, m // 2, 3 * m // 4, m - 1]
    Z, e = oracle.trevc(T, nb=nb, cols=cols)
    rescaled = 0
    for q, k in enumerate(cols):
        xt = R.backsub_longdouble(T, T[k, k], -T[:k, k], r=k)
        assert R.normwise_diff_aligned(Z[:k, q], e[q], xt) <= 1e-11
        lg = float(np.log2(np.max(np.abs(xt))))
        assert e[q] <= 970 - np.floor(lg) + 1
        rescaled += e[q] < 0
    if gen == "c5":
        assert rescaled >= 2      # the c5 generator grows ~5 bits/row: rescaling is exercised


# ----------------------------------------------------------------------------- eigenvectors
@pytest.mark.parametrize("gen,m,nb", [("c2", 200, 64), ("c3", 192, 128), ("c5", 420, 128)])
def test_trevc_eigen_residual(gen, m, nb):
    """||T v - lambda v||_inf <= 100 m eps ||T||_inf ||v||_inf (BASELINE north star)."""
    T = {"c2": inputs.c2_trevc_real, "c3": inputs.c3_trevc_complex, "c5": inputs.c5_grcar_like}[gen](m=m)
    Z, e = oracle.trevc(T, nb=nb)
    cp = np.iscomplexobj(T)
    Tl = T.astype(np.clongdouble if cp else np.longdouble)
    Zl = Z.astype(np.clongdouble if cp else np.longdouble)
    nT = np.max(np.sum(np.abs(Tl), axis=1))
    for k in range(m):
        v = Zl[:, k]
        r = Tl @ v - Tl[k, k] * v
        nv = np.max(np.abs(v))
        assert nv > 0
        assert np.max(np.abs(r)) <= 100 * m * 2.0 ** -52 * nT * nv
    if gen == "c5":
        assert (e < -300).any()                               # heavy rescaling exercised
    assert np.array_equal(np.triu(Z), Z)                      # upper triangular
    assert np.array_equal(np.diag(Z), np.ldexp(1.0, e).astype(Z.dtype))   # diag(Z) = s


def test_trevc_diagonal_T_gives_identity():
    T = np.diag(np.arange(1.0, 11.0))
    Z, e = oracle.trevc(T, nb=4)
    assert np.array_equal(Z, np.eye(10)) and not e.any()


def test_trevc_matches_numpy_eig_directions():
    rng = np.random.default_rng(4)
    m = 30
    T = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) * 0.3
    T[np.arange(m), np.arange(m)] = np.exp(2j * np.pi * np.arange(m) / m) * (1 + 0.5 * np.arange(m) / m)
    Z, _ = oracle.trevc(T, nb=8)
    w, V = np.linalg.eig(T)
    for k in range(m):
        j = int(np.argmin(np.abs(w - T[k, k])))
        a, b = Z[:, k] / np.linalg.norm(Z[:, k]), V[:, j] / np.linalg.norm(V[:, j])
        ph = np.vdot(b, a)
        assert abs(abs(ph) - 1) < 1e-10
        assert np.linalg.norm(a - ph * b) < 1e-9


def test_trevc_column_subset_is_exact():
    T = inputs.c5_grcar_like(m=200)
    Zf, ef = oracle.trevc(T, nb=32)
    cols = [0, 1, 77, 150, 199]
    Zs, es = oracle.trevc(T, nb=32, cols=cols)
    assert np.array_equal(Zs, Zf[:, cols]) and np.array_equal(es, ef[cols])


# ----------------------------------------------------------------------------- pseudospectra
def test_tridiag_lmax_vs_lapack():
    rng = np.random.default_rng(31)
    for k in range(1, 16):
        a = rng.standard_normal(k) * 3
        b = np.abs(rng.standard_normal(max(k - 1, 0)))
        ref = sla.eigvalsh_tridiagonal(a, b)[-1] if k > 1 else a[0]
        assert oracle.tridiag_lmax(a, b) == pytest.approx(ref, rel=1e-14, abs=1e-14)


@pytest.mark.parametrize("m", [1, 3, 8, 14])
def test_pseudospectra_small_m_exact_against_svd(m):
    """For m <= 15 the 15 Lanczos steps exhaust the Krylov space: exact vs the SVD."""
    rng = np.random.default_rng([32, m])
    U = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m)
    z = inputs.c4_grid(5, -1.2, 1.3)
    v0 = rng.standard_normal(m) + 1j * rng.standard_normal(m)
    v0 /= np.linalg.norm(v0)
    sig, flags = oracle.pseudospectra(U, z, iters=15, v0=v0, nb=4)
    for p, zz in enumerate(z):
        ref = np.linalg.svd(U - zz * np.eye(m), compute_uv=False)[-1]
        assert sig[p] == pytest.approx(ref, rel=1e-9)
    assert not flags.any()


def test_pseudospectra_one_by_one_closed_form():
    U = np.array([[0.3 - 0.2j]])
    z = np.array([1.0 + 1j, -2.0, 0.5j])
    sig, _ = oracle.pseudospectra(U, z, iters=3, v0=np.array([1.0 + 0j]), nb=1)
    assert np.allclose(sig, np.abs(U[0, 0] - z), rtol=1e-15)


def test_pseudospectra_unitary_invariance():
    """the resolvent norm is invariant under unitary similarity."""
    rng = np.random.default_rng(33)
    m = 12
    A = rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))
    T1, _ = sla.schur(A, output="complex")
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m)))
    T2, _ = sla.schur(Q @ T1 @ Q.conj().T, output="complex")
    z = np.array([0.3 + 0.1j, 2.0 - 1.0j, -1.5j])
    v0 = np.ones(m, complex) / np.sqrt(m)
    s1, _ = oracle.pseudospectra(T1, z, iters=15, v0=v0, nb=4)
    s2, _ = oracle.pseudospectra(T2, z, iters=15, v0=v0, nb=4)
    assert np.allclose(s1, s2, rtol=1e-8)


def test_pseudospectra_real_matrix_conjugate_symmetric():
    rng = np.random.default_rng(34)
    m = 40
    U = np.triu(rng.standard_normal((m, m))) / np.sqrt(m) + np.diag(rng.uniform(-1, 1, m))
    z = np.array([0.2 + 0.7j, -0.4 + 0.3j, 1.1 + 0.05j])
    v0 = np.ones(m, complex) / np.sqrt(m)       # real start vector
    s1, _ = oracle.pseudospectra(U.astype(complex), z, iters=15, v0=v0, nb=8)
    s2, _ = oracle.pseudospectra(U.astype(complex), np.conj(z), iters=15, v0=v0, nb=8)
    assert np.allclose(s1, s2, rtol=1e-12)


def test_pseudospectra_ritz_values_monotone():
    """lambda_max estimates grow with the number of Lanczos steps (sigma shrinks)."""
    U, z, v0 = inputs.c4_pseudospectra(m=64, npx=4)
    prev = None
    for k in range(1, 16):
        s, _ = oracle.pseudospectra(U, z, iters=k, v0=v0, nb=16)
        if prev is not None:
            assert np.all(s <= prev * (1 + 1e-12))
        prev = s


def test_pseudospectra_singular_point_is_flagged_upper_bound():
    """A shift on an eigenvalue: never Inf/NaN.  One exact zero pivot -> the delta
    step gives a tiny finite sigma; a Jordan block (growth (1/delta)^m >> Omega)
    makes the safe solve rescale, and sigma is the rigorous bound c1/||y||_2 (R25)."""
    U = np.triu(np.ones((6, 6))) * 0.5 + 0j
    U[np.arange(6), np.arange(6)] = np.arange(6)
    sig, flags = oracle.pseudospectra(U, np.array([2.0 + 0j, 0.5 + 0.5j]), iters=15,
                                      v0=np.ones(6, complex) / np.sqrt(6), nb=2)
    assert flags[0] == 0 and np.isfinite(sig[0]) and 0 < sig[0] < 1e-13
    ref = np.linalg.svd(U - (0.5 + 0.5j) * np.eye(6), compute_uv=False)[-1]
    assert flags[1] == 0 and sig[1] == pytest.approx(ref, rel=1e-9)
    m = 30
    J = (2.0 * np.eye(m) + np.diag(np.ones(m - 1), 1)).astype(complex)
    sig, flags = oracle.pseudospectra(J, np.array([2.0 + 0j]), iters=15,
                                      v0=np.ones(m, complex) / np.sqrt(m), nb=8)
    assert flags[0] == 1 and np.isfinite(sig[0]) and 0 <= sig[0] < 1e-200
