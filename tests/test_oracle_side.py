"""Pins (-m "not gpu") for the SURVEY §8f row f4 oracle (P:58-62 footnote): left/right,
upper/lower multi-shift solves.  Pinned against LAPACK triangular solves on the explicitly
shifted matrices (scipy.linalg.solve_triangular, plain case), the diagonal closed form, and the
safe variant's scaled equations in extended precision."""
import numpy as np
import pytest

import oracle

CASES = [("L", "U"), ("L", "L"), ("R", "U"), ("R", "L")]


def _tri(m, uplo, cplx, seed):
    rng = np.random.default_rng([31, m, seed])
    A = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    A = A / np.sqrt(m)
    A[np.arange(m), np.arange(m)] = rng.uniform(1.0, 2.0, m)
    return np.asfortranarray(np.triu(A) if uplo == "U" else np.tril(A))


@pytest.mark.parametrize("side,uplo", CASES)
@pytest.mark.parametrize("cplx", [False, True])
def test_side_plain_matches_lapack(side, uplo, cplx):
    scipy_linalg = pytest.importorskip("scipy.linalg")
    m, n = 37, 9
    A = _tri(m, uplo, cplx, 1)
    rng = np.random.default_rng(5)
    s = rng.uniform(-0.5, 0.5, n) + (1j * rng.uniform(-0.5, 0.5, n) if cplx else 0)
    B = rng.standard_normal((m, n) if side == "L" else (n, m))
    X, e = oracle.mstrsm_side(A, s, B, side=side, uplo=uplo, safe=False, nb=8)
    assert not e.any()
    for j in range(n):
        As = A - s[j] * np.eye(m)
        if side == "L":
            ref = scipy_linalg.solve_triangular(As, B[:, j], lower=(uplo == "L"))
            got = X[:, j]
        else:   # x^T As = b^T  <=>  As^T x = b
            ref = scipy_linalg.solve_triangular(As, B[j, :], lower=(uplo == "L"), trans="T")
            got = X[j, :]
        assert np.max(np.abs(got - ref)) <= 1e-12 * np.max(np.abs(ref))


@pytest.mark.parametrize("side,uplo", CASES)
def test_side_diagonal_is_division(side, uplo):
    m, n = 6, 4
    d = np.arange(1.0, 7.0) + 0.5j
    A = np.diag(d)
    s = np.array([0.25, -1.0, 2.0j, 0.0])
    B = np.ones((m, n) if side == "L" else (n, m), dtype=complex)
    X, e = oracle.mstrsm_side(A, s, B, side=side, uplo=uplo, safe=False, nb=2)
    Xc = X if side == "L" else X.T
    for j in range(n):
        assert np.allclose(Xc[:, j], 1.0 / (d - s[j]), rtol=1e-15, atol=0)


@pytest.mark.parametrize("side,uplo", CASES)
def test_side_safe_scaled_equations(side, uplo):
    """Safe variant on a growth-heavy lower / upper triangle: the scaled system holds in long
    double, ||(A - sI) x - c b|| <= 64 m eps (||A - sI|| ||x|| + c ||b||) (R19), e <= 0 and some
    column rescales."""
    m, n = 120, 6
    rng = np.random.default_rng(9)
    A = rng.standard_normal((m, m)) * 4.0
    A[np.arange(m), np.arange(m)] = rng.uniform(-1e-3, 1e-3, m)
    A = np.triu(A) if uplo == "U" else np.tril(A)
    s = rng.uniform(-1e-3, 1e-3, n)
    B = rng.standard_normal((m, n) if side == "L" else (n, m))
    X, e = oracle.mstrsm_side(A, s, B, side=side, uplo=uplo, safe=True, nb=16)
    assert (e <= 0).all() and (e < 0).any() and np.isfinite(X).all()
    L = np.longdouble
    for j in range(n):
        As = (A - s[j] * np.eye(m)).astype(L)
        x = (X[:, j] if side == "L" else X[j, :]).astype(L)
        b = (B[:, j] if side == "L" else B[j, :]).astype(L)
        r = (As @ x if side == "L" else x @ As) - np.ldexp(L(1), int(e[j])) * b
        nA = np.max(np.sum(np.abs(As), axis=1 if side == "L" else 0))
        bound = 64 * m * 2.0 ** -53 * (nA * np.max(np.abs(x)) + np.ldexp(1.0, int(e[j])) * np.max(np.abs(b)))
        assert np.max(np.abs(r)) <= bound
