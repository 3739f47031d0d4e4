"""GPU parity tests (-m gpu) for SURVEY §8f row f3: SpectralCloud with per-point
deflation and batch compaction (R33), SpectralWindow, SpectralPortrait (R34), against the CPU
oracle on the same seeded inputs.  Bars: sigma 1e-8 relative (R22), flags equal, Lanczos step
counts equal up to a deflation decision taken one step apart at a rounding-level tie."""
import numpy as np
import pytest

import oracle
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


def _sync():
    import torch
    torch.cuda.synchronize()


def _c4(m, npx):
    U, z, v0 = inputs.c4_pseudospectra(m=m, npx=npx)
    return U, z, v0


def _check(sg, fg, ig, so, fo, io, what, min_equal=0.95):
    assert np.array_equal(fg, fo), f"{what}: flags differ"
    rel = np.abs(sg - so) / np.abs(so)
    assert rel.max() <= 1e-8, f"{what}: sigma rel {rel.max():.3e}"
    d = np.abs(ig.astype(int) - io.astype(int))
    assert d.max() <= 1 and (d == 0).mean() >= min_equal, f"{what}: its differ ({(d != 0).sum()} points)"


def test_gpu_cloud_tol_zero_equals_pseudospectra(ms):
    U, z, v0 = _c4(160, 9)
    s0, f0 = ms.pseudospectra(dev(U), dev(z), dev(v0), iters=10, nb=32)
    s1, f1, i1 = ms.spectral_cloud(dev(U), dev(z), dev(v0), maxit=10, tol=0.0, nb=32)
    _sync()
    assert np.array_equal(host(s0), host(s1)) and np.array_equal(host(f0), host(f1))
    assert host(i1).max() <= 10


@pytest.mark.parametrize("m,npx,nb,tol", [(1, 3, 8, 1e-10), (97, 7, 32, 1e-10), (300, 12, 64, 1e-11)])
def test_gpu_cloud_parity(ms, m, npx, nb, tol):
    U, z, v0 = _c4(m, npx)
    sg, fg, ig = ms.spectral_cloud(dev(U), dev(z), dev(v0), maxit=30, tol=tol, nb=nb)
    _sync()
    so, fo, io = oracle.spectral_cloud(U, z, maxit=30, tol=tol, v0=v0, nb=nb)
    # m = 1: the breakdown test b <= m eps max(alpha) is a rounding-level tie (w - alpha v ~ ulp), so
    # a point may take one extra, immediately settled step on either side
    _check(host(sg), host(fg), host(ig), so, fo, io, f"cloud m={m}", min_equal=0.95 if m > 1 else 0.0)
    if m > 1:
        assert io.min() < io.max()                      # points really left the batch at different steps


def test_gpu_cloud_compaction_keeps_survivors_bitwise(ms):
    """A point's result does not depend on which other points share (and leave) the batch."""
    U, z, v0 = _c4(200, 10)
    s, f, i = (host(t) for t in ms.spectral_cloud(dev(U), dev(z), dev(v0), maxit=25, tol=1e-10, nb=32))
    sub = np.arange(0, z.shape[0], 7)
    s2, f2, i2 = (host(t) for t in ms.spectral_cloud(dev(U), dev(z[sub]), dev(v0), maxit=25, tol=1e-10, nb=32))
    _sync()
    assert np.array_equal(s[sub], s2) and np.array_equal(f[sub], f2) and np.array_equal(i[sub], i2)


def test_gpu_window_grid_and_parity(ms):
    U, _, v0 = _c4(128, 4)
    args = (-1.5, 1.5, 11, -1.25, 1.0, 6)
    sg, fg, ig = (host(t) for t in ms.spectral_window(dev(U), *args, dev(v0), maxit=30, tol=1e-10, nb=32))
    z = oracle.window_grid(*args)
    sc, fc, ic = (host(t) for t in ms.spectral_cloud(dev(U), dev(z), dev(v0), maxit=30, tol=1e-10, nb=32))
    _sync()
    assert np.array_equal(sg, sc) and np.array_equal(ig, ic)          # the device grid is numpy's
    so, fo, io = oracle.spectral_window(U, *args, maxit=30, tol=1e-10, v0=v0, nb=32)
    _check(sg, fg, ig, so, fo, io, "window")


def test_gpu_portrait(ms):
    U, _, v0 = _c4(150, 4)
    sg, fg, ig, win = ms.spectral_portrait(dev(U), 9, 8, dev(v0), maxit=30, tol=1e-10, nb=32)
    _sync()
    so, fo, io, wo = oracle.spectral_portrait(U, 9, 8, maxit=30, tol=1e-10, v0=v0, nb=32)
    assert np.allclose(win, wo, rtol=1e-13, atol=0)
    _check(host(sg), host(fg), host(ig), so, fo, io, "portrait")


def test_gpu_cloud_unsettled_flag(ms):
    U, z, v0 = _c4(100, 6)
    sg, fg, ig = (host(t) for t in ms.spectral_cloud(dev(U), dev(z), dev(v0), maxit=3, tol=1e-14, nb=32))
    _sync()
    so, fo, io = oracle.spectral_cloud(U, z, maxit=3, tol=1e-14, v0=v0, nb=32)
    assert np.array_equal(fg, fo) and ((fg & 2) != 0).any()
    assert np.max(np.abs(sg - so) / so) <= 1e-8


def test_gpu_breakdown_at_the_last_step_matches_oracle(ms):
    """R33 pin on the GPU: a 4 x 4 U breaks down at step 5; maxit = 5 -> not flagged, maxit = 4 ->
    flagged (test_oracle_spectral.py::test_breakdown_at_the_last_step_is_not_flagged)."""
    rng = np.random.default_rng(11)
    m = 4
    U = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / 2 + np.diag([1.5, 2.0 + 0.5j, -1.0, 0.7j])
    U = np.asfortranarray(U)
    z = np.array([0.3 + 0.1j, -0.2 + 0.4j])
    v0 = np.ones(m, complex) / 2
    for maxit, want in ((5, [0, 0]), (4, [2, 2])):
        sg, fg, ig = ms.spectral_cloud(dev(U), dev(z), dev(v0), maxit=maxit, tol=1e-300, nb=2)
        _sync()
        so, fo, io = oracle.spectral_cloud(U, z, maxit=maxit, tol=1e-300, v0=v0, nb=2)
        assert list(host(fg)) == list(fo) == want
        assert list(host(ig)) == list(io) == [maxit, maxit]
        assert np.max(np.abs(host(sg) - so) / so) <= 1e-8
