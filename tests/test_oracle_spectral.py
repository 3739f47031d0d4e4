"""Pins (-m "not gpu") for the SURVEY §8f row f3 oracle: SpectralCloud with per-point deflation
(R33), SpectralWindow's grid and SpectralPortrait's automatic window (R34) -- P:683-691, S:392,
S:407-415.  Pinned against the fixed-iteration Alg. VL oracle (itself pinned in
test_oracle_pins.py), dense SVD, closed forms and the stop rule re-derived from independent
fixed-step runs."""
import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs


def _c4(m=48, npx=5):
    U, z, v0 = inputs.c4_pseudospectra(m=m, npx=npx)
    return U, z, v0


def test_tol_zero_is_the_fixed_iteration_algorithm():
    U, z, v0 = _c4()
    s0, f0 = oracle.pseudospectra(U, z, iters=12, v0=v0, nb=16)
    s1, f1, its = oracle.spectral_cloud(U, z, maxit=12, tol=0.0, v0=v0, nb=16)
    assert np.array_equal(s0, s1) and np.array_equal(f0, f1)
    assert (its <= 12).all()


def test_deflation_is_per_point_independent():
    """Removing converged shifts from the batch does not change the others: the batch
    result equals every point run alone, bit for bit."""
    U, z, v0 = _c4()
    s, f, its = oracle.spectral_cloud(U, z, maxit=25, tol=1e-11, v0=v0, nb=16)
    for p in range(0, z.shape[0], 3):
        s1, f1, i1 = oracle.spectral_cloud(U, z[p:p + 1], maxit=25, tol=1e-11, v0=v0, nb=16)
        assert s1[0] == s[p] and f1[0] == f[p] and i1[0] == its[p]


def test_stop_rule_from_independent_fixed_step_runs():
    """its[p] = k is the first k >= 2 with |theta_k - theta_{k-1}| <= tol theta_k, theta_j =
    1/sigma_j^2 from the fixed j-step algorithm (rounding slack 1e-9 relative on the test)."""
    U, z, v0 = _c4(m=40, npx=3)
    tol = 1e-9
    s, f, its = oracle.spectral_cloud(U, z, maxit=30, tol=tol, v0=v0, nb=8)
    for p in range(z.shape[0]):
        k = int(its[p])
        th = [None] + [1.0 / oracle.pseudospectra(U, z[p:p + 1], iters=j, v0=v0, nb=8)[0][0] ** 2
                       for j in range(1, k + 1)]
        if f[p] == 0 and k < 30:
            assert abs(th[k] - th[k - 1]) <= tol * th[k] * (1 + 1e-9)
        for j in range(2, k):
            assert abs(th[j] - th[j - 1]) > tol * th[j] * (1 - 1e-9)


def test_converged_points_match_the_svd():
    U, z, v0 = _c4(m=64, npx=6)
    s, f, its = oracle.spectral_cloud(U, z, maxit=40, tol=1e-12, v0=v0, nb=16)
    sv = np.array([np.linalg.svd(U - zz * np.eye(U.shape[0]), compute_uv=False)[-1] for zz in z])
    ok = f == 0
    assert ok.sum() >= z.shape[0] - 2
    assert np.max(np.abs(s[ok] - sv[ok]) / sv[ok]) <= 1e-6


def test_unsettled_points_are_flagged():
    U, z, v0 = _c4()
    s, f, its = oracle.spectral_cloud(U, z, maxit=3, tol=1e-14, v0=v0, nb=16)
    assert ((f & 2) != 0).sum() > 0
    assert np.all(((f & 2) != 0) == (its == 3))


def test_one_by_one_closed_form():
    s, f, its = oracle.spectral_cloud(np.array([[1.0 + 0j]]), np.array([3.0 + 0j]), maxit=15, tol=1e-12,
                                      v0=np.array([1.0 + 0j]), nb=1)
    assert s[0] == 2.0 and f[0] == 0 and its[0] == 1                # sigma_min(1 - 3) = 2; Krylov exhausted


def test_window_grid_order_and_real_symmetry():
    """R15 order (ix + nx iy, endpoint-inclusive); a real U gives a field symmetric about the real
    axis for a grid symmetric in y."""
    g = oracle.window_grid(-1.0, 1.0, 3, -2.0, 2.0, 5)
    assert g[0] == -1 - 2j and g[2] == 1 - 2j and g[3] == -1 - 1j and g[-1] == 1 + 2j
    rng = np.random.default_rng(4)
    m = 30
    U = np.triu(rng.standard_normal((m, m))) / np.sqrt(m) + np.diag(rng.uniform(-1, 1, m))
    nx, ny = 4, 5
    s, f, _ = oracle.spectral_window(U.astype(complex), -1.5, 1.5, nx, -1.0, 1.0, ny, maxit=40, tol=1e-12,
                                     v0=np.ones(m, complex) / np.sqrt(m), nb=8)
    F = s.reshape(ny, nx)
    assert np.allclose(F, F[::-1, :], rtol=1e-8)


def test_portrait_window_closed_forms():
    x0, x1, y0, y1 = oracle.portrait_window(np.diag([-1.0, 1.0]).astype(complex))
    assert (x0, x1, y0, y1) == (-1.5, 1.5, -0.5, 0.5)                # pad 0.25 * max(2, 0, 0.01)
    U = np.array([[1j, 100.0], [0, 1j]])                 # one point: pad from ||U||_inf = 1 + 100
    x0, x1, y0, y1 = oracle.portrait_window(U)
    pad = 0.25 * (1e-2 * 101.0)
    assert (x0, x1, y0, y1) == (0.0 - pad, 0.0 + pad, 1.0 - pad, 1.0 + pad)
    s, f, its, win = oracle.spectral_portrait(np.diag([-1.0, 1.0]).astype(complex), 3, 3, maxit=10,
                                              tol=1e-12, v0=np.ones(2, complex) / np.sqrt(2), nb=1)
    assert win == (-1.5, 1.5, -0.5, 0.5)
    # diagonal U: sigma_min(U - z) = distance from z to the spectrum (normal matrix)
    z = oracle.window_grid(-1.5, 1.5, 3, -0.5, 0.5, 3)
    dist = np.minimum(np.abs(z + 1), np.abs(z - 1))
    assert np.allclose(s, dist, rtol=1e-12)


def test_breakdown_at_the_last_step_is_not_flagged():
    """R33: bit1 marks a point that neither settled nor broke down within maxit steps.  A 4 x 4 U
    exhausts its Krylov space; the breakdown test (beta_k <= m eps max alpha) fires at step 5.  With
    maxit = 5 the point breaks down exactly at the last step: not flagged (the rule "k == maxit"
    would flag it); with maxit = 4 it has done neither: flagged.  The exhausted space makes sigma
    the exact sigma_min (numpy SVD)."""
    rng = np.random.default_rng(11)
    m = 4
    U = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / 2 + np.diag([1.5, 2.0 + 0.5j, -1.0, 0.7j])
    U = np.asfortranarray(U)
    z = np.array([0.3 + 0.1j, -0.2 + 0.4j])
    v0 = np.ones(m, complex) / 2
    sv = np.array([np.linalg.svd(U - zz * np.eye(m), compute_uv=False)[-1] for zz in z])
    s, f, its = oracle.spectral_cloud(U, z, maxit=5, tol=1e-300, v0=v0, nb=2)
    assert list(its) == [5, 5] and list(f) == [0, 0]
    assert np.max(np.abs(s - sv) / sv) <= 1e-12
    s4, f4, its4 = oracle.spectral_cloud(U, z, maxit=4, tol=1e-300, v0=v0, nb=2)
    assert list(its4) == [4, 4] and list(f4) == [2, 2]
