"""Pins (-m "not gpu") for the back-transformation oracle:
X = Q Z with Z = TriangEig(T) gives the eigenvectors of A = Q T Q^H.  Pinned against the
eigen-invariant of A in extended precision (heavy rescaling included), exact identity /
permutation reductions, and LAPACK's eigenvectors of A (scipy.linalg.eig)."""
import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs

LD, CLD = np.longdouble, np.clongdouble


def _unitary(m, cplx, seed):
    rng = np.random.default_rng([7, m, seed])
    G = rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cplx else 0)
    return np.asfortranarray(np.linalg.qr(G)[0])


@pytest.mark.parametrize("gen,m,nb", [("c3", 150, 32), ("c2", 150, 32), ("c5", 320, 64)])
def test_backtransform_eigen_residual_of_A(gen, m, nb):
    """||A x_k - lambda_k x_k||_inf <= 100 m eps ||A||_inf ||x_k||_inf for A = Q T Q^H (the
    north-star invariant carried through X = Q Z; Q unitary keeps the bound)."""
    T = {"c2": inputs.c2_trevc_real, "c3": inputs.c3_trevc_complex, "c5": inputs.c5_grcar_like}[gen](m=m)
    cp = np.iscomplexobj(T)
    Q = _unitary(m, cp, 1)
    X, e = oracle.trevc_qz(T, Q, nb=nb)
    Al = (Q.astype(CLD if cp else LD) @ T.astype(CLD if cp else LD)) @ Q.conj().T.astype(CLD if cp else LD)
    Xl = X.astype(CLD if cp else LD)
    nA = np.max(np.sum(np.abs(Al), axis=1))
    R = Al @ Xl - Xl * np.diag(T).astype(CLD if cp else LD)[None, :]
    for k in range(m):
        nx = np.max(np.abs(Xl[:, k]))
        assert nx > 0
        assert np.max(np.abs(R[:, k])) <= 100 * m * 2.0 ** -52 * nA * nx
    if gen == "c5":
        assert (e < -300).any()                                # heavy rescaling exercised


@pytest.mark.parametrize("cplx", [False, True])
def test_backtransform_identity_and_permutation_are_exact(cplx):
    m = 90
    T = inputs.c3_trevc_complex(m) if cplx else inputs.c2_trevc_real(m)
    Z, e = oracle.trevc(T, nb=16)
    X, e2 = oracle.trevc_qz(T, np.eye(m, dtype=T.dtype), nb=16)
    assert np.array_equal(X, Z) and np.array_equal(e, e2)
    perm = np.random.default_rng(3).permutation(m)
    P = np.eye(m, dtype=T.dtype)[perm]
    assert np.array_equal(oracle.eig_backtransform(P, Z), Z[perm])


def test_backtransform_matches_lapack_eigenvectors():
    """Directions agree with LAPACK's eigenvectors of A (zgeev via scipy): |<x_k, v_k>| = 1 after
    normalisation, eigenvalues matched to diag(T)."""
    scipy_linalg = pytest.importorskip("scipy.linalg")
    m = 40
    T = inputs.c3_trevc_complex(m)
    Q = _unitary(m, True, 2)
    X, _ = oracle.trevc_qz(T, Q, nb=8)
    A = Q @ T @ Q.conj().T
    w, V = scipy_linalg.eig(A)
    for k in range(m):
        j = int(np.argmin(np.abs(w - T[k, k])))
        x = X[:, k] / np.linalg.norm(X[:, k])
        v = V[:, j] / np.linalg.norm(V[:, j])
        assert abs(abs(np.vdot(v, x)) - 1.0) < 1e-8
