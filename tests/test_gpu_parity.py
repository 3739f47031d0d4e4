"""GPU parity tests (-m gpu): the CUDA path through the C ABI vs the CPU oracle on the same seeded
inputs (paper_1607_01477_b200/inputs.py).  Bars (BASELINE north star, R20-R22):
  * normwise ||2^(e_o-e_g) x_gpu - x_orc||_inf / ||x_orc||_inf <= 1e-9
  * |e_gpu - e_orc| <= 1 (scale factors within a factor of 2)
  * sigma_min within 1e-8 relative of the oracle's identical 15-step Lanczos
  * bit-exact where the arithmetic is exact (diagonal U, hand-derived rescale pins, column
    subsets vs the full run, safe-with-c=1 vs plain)
"""
import json
import os

import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs
from tests import refmath as R
from tests.gpu_util import assert_parity, dev, host

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


@pytest.fixture(scope="module")
def ms():
    import torch
    assert torch.cuda.is_available(), "gpu tests need a GPU"
    import paper_1607_01477_b200 as m
    m.load()
    return m


def _num(v):
    if isinstance(v, str):
        sgn = -1.0 if v.startswith("-") else 1.0
        return sgn * 2.0 ** float(v.lstrip("-").split("^")[1])
    return float(v)


def _log_parity(what, rel, de, extra=None):
    """Print the R20 normwise differences and the R21 Delta-e histogram of a parity check; with
    MSTRSM_PARITY_LOG set, also append them as one JSON line to that file (GPU round evidence)."""
    hist = {int(k): int(v) for k, v in zip(*np.unique(np.asarray(de, dtype=np.int64), return_counts=True))}
    rec = {"what": what, "columns": int(len(rel)), "max_rel": float(np.max(rel)) if len(rel) else 0.0,
           "median_rel": float(np.median(rel)) if len(rel) else 0.0, "delta_e_hist": hist}
    if extra:
        rec.update(extra)
    print(json.dumps(rec))
    path = os.environ.get("MSTRSM_PARITY_LOG")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def gpu_solve(ms, U, s, B, *, safe=True, op="N", nb=32, row_end=None):
    Ud, sd, Bd = dev(U), dev(np.ascontiguousarray(s)), dev(B)
    X, sc, e = ms.solve(Ud, sd, Bd, safe=safe, op=op, nb=nb, row_end=row_end)
    import torch
    torch.cuda.synchronize()
    return host(X), host(sc), host(e)


def _well_conditioned(m, cplx, seed):
    rng = np.random.default_rng([77, m, seed])
    U = np.triu(rng.standard_normal((m, m))) / np.sqrt(max(m, 1))
    if cplx:
        U = U + 1j * np.triu(rng.standard_normal((m, m))) / np.sqrt(max(m, 1))
    U[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m) + (1j * rng.uniform(-0.3, 0.3, m) if cplx else 0)
    return np.asfortranarray(U)


# ------------------------------------------------------------------------------- exactness
def test_gpu_diagonal_U_exact_division(ms):
    rng = np.random.default_rng(1)
    m, n = 150, 70
    d = rng.uniform(1, 2, m)
    s = rng.uniform(-0.5, 0.5, n)
    B = rng.standard_normal((m, n))
    for safe in (False, True):
        X, sc, e = gpu_solve(ms, np.diag(d), s, B, safe=safe, nb=32)
        assert np.array_equal(X, B / (d[:, None] - s[None, :]))
        assert not e.any() and np.all(sc == 1.0)


@pytest.mark.parametrize("case", GOLD["rescale_pins"], ids=lambda c: c["cite"][:20])
def test_gpu_rescale_pins_bit_exact(ms, case):
    U = np.array([[_num(v) for v in row] for row in case["U"]])
    X, sc, e = gpu_solve(ms, U, np.zeros(1), np.array(case["B"], float).reshape(-1, 1), nb=case["nb"])
    assert int(e[0]) == case["e"]
    assert np.array_equal(X[:, 0], np.array([_num(v) for v in case["X"]]))
    assert sc[0] == 2.0 ** case["e"]


@pytest.mark.parametrize("case", GOLD["solve"], ids=lambda c: c["cite"][:24])
def test_gpu_golden_solves(ms, case):
    U = np.array(case["U"], float)
    X, sc, e = gpu_solve(ms, U, np.array(case["shifts"], float), np.array(case["B"], float), nb=case["nb"])
    assert np.allclose(X, np.array(case["X"], float), rtol=1e-15, atol=0)
    assert list(e) == case["e"]


def test_gpu_zero_column_and_zero_pivot(ms):
    U = _well_conditioned(40, False, 3)
    B = inputs.random_rhs(40, 5, False, 9)
    B[:, 2] = 0.0
    s = np.array([0.1, U[5, 5], 0.0, U[39, 39], -0.2])    # exact zero pivots -> delta
    X, sc, e = gpu_solve(ms, U, s, B, nb=16)
    Xo, eo = oracle.mstrsm(U, s, B, nb=16)
    assert np.all(X[:, 2] == 0) and sc[2] == 1.0
    assert_parity(X, e, Xo, eo, what="zero pivots")


# ------------------------------------------------------------------------------- config 1
def test_gpu_c1_plain_and_safe(ms):
    U, s, B = inputs.c1_plain_real()
    Xo, eo = oracle.mstrsm(U, s, B, safe=False, nb=32)
    Xp, _, ep = gpu_solve(ms, U, s, B, safe=False, nb=32)
    assert_parity(Xp, ep, Xo, eo, what="c1 plain")
    Xs, sc, es = gpu_solve(ms, U, s, B, safe=True, nb=32)
    Xso, eso = oracle.mstrsm(U, s, B, safe=True, nb=32)
    assert not es.any() and not eso.any()                 # config 1 never rescales
    assert_parity(Xs, es, Xso, eso, what="c1 safe")
    assert np.array_equal(Xs, Xp)                        # safe with c = 1 == plain, bit for bit
    # normwise backward error (north star), extended precision
    for j in range(0, 64, 7):
        assert R.residual_ratio(U, s[j], Xs[:, j], es[j], B[:, j]) <= 64 * 256 * 2.0 ** -53


# ------------------------------------------------------------------------------- ragged shapes
# odd n_b: ragged k-tiles in every update and, for op C, odd block offsets (the 3M kernel's
# sum-plane alignment fails and the register-sum kernel takes over)
SHAPES = [(1, 1, 8), (7, 3, 8), (100, 37, 32), (129, 64, 64), (333, 130, 64), (300, 70, 128), (257, 129, 128),
          (200, 50, 7), (97, 40, 1), (150, 33, 13)]


@pytest.mark.parametrize("m,n,nb", SHAPES)
@pytest.mark.parametrize("cplx", [False, True])
@pytest.mark.parametrize("op", ["N", "C"])
def test_gpu_ragged_shapes(ms, m, n, nb, cplx, op):
    U = _well_conditioned(m, cplx, nb)
    s = inputs.random_shifts(n, cplx, m, center=0.0, radius=0.4)
    B = inputs.random_rhs(m, n, cplx, nb)
    for safe in (False, True):
        Xg, _, eg = gpu_solve(ms, U, s, B, safe=safe, op=op, nb=nb)
        Xo, eo = oracle.mstrsm(U, s, B, safe=safe, op=op, nb=nb)
        assert_parity(Xg, eg, Xo, eo, what=f"{m}x{n} nb={nb} {op} safe={safe}")


@pytest.mark.parametrize("sorted_", [True, False])
def test_gpu_row_end(ms, sorted_):
    m, n, nb = 200, 90, 32
    U = _well_conditioned(m, True, 5)
    s = inputs.random_shifts(n, True, 6, radius=0.3)
    B = inputs.random_rhs(m, n, True, 7)
    r = np.random.default_rng(8).integers(0, m + 1, n)
    if sorted_:
        r = np.sort(r)
    Xg, _, eg = gpu_solve(ms, U, s, B, nb=nb, row_end=r)
    Xo, eo = oracle.mstrsm(U, s, B, nb=nb, row_end=r)
    assert_parity(Xg, eg, Xo, eo, what="row_end")
    for j in range(n):
        assert np.all(Xg[r[j]:, j] == 0)


@pytest.mark.parametrize("sorted_", [True, False])
def test_gpu_row_end_device_pointer(ms, sorted_):
    """row_end as a device array (include/mstrsm.h): the same result, bit for bit, as
    the host array, and parity with the oracle; out-of-range values are clamped to [0, m]."""
    import torch
    m, n, nb = 300, 70, 64
    U = _well_conditioned(m, True, 9)
    s = inputs.random_shifts(n, True, 10, radius=0.3)
    B = inputs.random_rhs(m, n, True, 11)
    r = np.random.default_rng(12).integers(-5, m + 20, n)
    if sorted_:
        r = np.sort(r)
    Xh, _, eh = gpu_solve(ms, U, s, B, nb=nb, row_end=r)
    Xd, _, ed = gpu_solve(ms, U, s, B, nb=nb, row_end=torch.from_numpy(r).cuda())
    assert np.array_equal(Xh, Xd) and np.array_equal(eh, ed)
    rc = np.clip(r, 0, m)
    Xo, eo = oracle.mstrsm(U, s, B, nb=nb, row_end=rc)
    assert_parity(Xd, ed, Xo, eo, what="row_end device")


# ------------------------------------------------------------------------------- safety
def test_gpu_adversarial_safety(ms):
    """finite, c in [0,1], ||x|| < Omega, backward error <= 64 m 2^-53 on the adversarial
    suite (Jordan, zero pivots, graded 10^+-300, repeated eigenvalues)."""
    from tests.test_oracle_pins import _adversarial_suite
    for U, s, B, nb in _adversarial_suite():
        m = U.shape[0]
        X, sc, e = gpu_solve(ms, U, s, B, nb=nb)
        Xo, eo = oracle.mstrsm(U, s, B, nb=nb)
        assert np.all(np.isfinite(X)) and np.all(e <= 0) and np.max(np.abs(X)) < R.OMEGA
        assert np.all((sc >= 0) & (sc <= 1))
        unorm = np.max(np.sum(np.abs(np.triu(U)), axis=1))
        delta = np.ldexp(unorm, -52) if unorm > 0 else np.finfo(float).tiny
        for j in range(len(s)):
            dd = np.diag(U) - s[j]
            if np.any((dd == 0) & (delta + s[j] - s[j] != delta)):
                continue
            Ud = np.triu(U).copy()
            Ud[np.arange(m), np.arange(m)] = np.where(dd == 0, delta + s[j], np.diag(U))
            assert R.residual_ratio(Ud, s[j], X[:, j], e[j], B[:, j]) <= 64 * m * 2.0 ** -53


def test_gpu_nonfinite_input_status(ms):
    U = _well_conditioned(30, False, 1)
    U[3, 10] = np.nan
    gpu_solve(ms, U, np.zeros(2), np.ones((30, 2)), nb=8)
    assert ms.status() == 2
    assert ms.status() == 0          # cleared


def test_gpu_nonfinite_input_sync_status(ms):
    """mstrsm_set_sync_status(1): the call itself synchronises and returns code 2."""
    U = _well_conditioned(30, True, 2)
    U[4, 20] = complex(np.inf, 0)
    ms.mstrsm_set_sync_status(1)
    try:
        with pytest.raises(ms.MstrsmError, match="returned 2"):
            gpu_solve(ms, U, np.zeros(2, complex), np.ones((30, 2), complex), nb=8)
        assert ms.status() == 0      # the call cleared the flag
        gpu_solve(ms, _well_conditioned(30, True, 3), np.zeros(2, complex), np.ones((30, 2), complex), nb=8)
        T = _well_conditioned(40, False, 4)
        T[1, 30] = np.nan
        with pytest.raises(ms.MstrsmError, match="returned 2"):
            gpu_trevc(ms, T, 16)
    finally:
        ms.mstrsm_set_sync_status(0)
    gpu_solve(ms, U, np.zeros(2, complex), np.ones((30, 2), complex), nb=8)   # asynchronous again
    assert ms.status() == 2


# ------------------------------------------------------------------------------- eigenvectors
def gpu_trevc(ms, T, nb, cols=None):
    import torch
    Z, sc, e = ms.trevc(dev(T), nb=nb, cols=cols)
    torch.cuda.synchronize()
    return host(Z), host(sc), host(e)


def _eig_residual_ok(T, Z, cols):
    cp = np.iscomplexobj(T)
    Tl = T.astype(np.clongdouble if cp else np.longdouble)
    nT = np.max(np.sum(np.abs(Tl), axis=1))
    m = T.shape[0]
    for q, k in enumerate(cols):
        v = Z[:, q].astype(Tl.dtype)
        r = Tl[:k + 1, :k + 1] @ v[:k + 1] - Tl[k, k] * v[:k + 1]
        assert np.max(np.abs(r)) <= 100 * m * 2.0 ** -52 * nT * np.max(np.abs(v))


def test_gpu_trevc_small_exact_cases(ms):
    for case in GOLD["trevc"]:
        Z, sc, e = gpu_trevc(ms, np.array(case["T"], float), 2)
        assert np.array_equal(Z, np.array(case["Z"], float)) and list(e) == case["e"]


def test_gpu_trevc_c2_full(ms):
    """Config 2 at full size (m = 2048, real, n_b = 64) against the full oracle."""
    T = inputs.c2_trevc_real()
    Zg, sc, eg = gpu_trevc(ms, T, 64)
    Zo, eo = oracle.trevc(T, nb=64)
    rel, de = assert_parity(Zg, eg, Zo, eo, what="c2")
    _log_parity("c2 full", rel, de, {"rescaled": int((eo < 0).sum()), "min_e": int(eo.min())})
    assert np.array_equal(np.triu(Zg), Zg)
    assert np.array_equal(np.diag(Zg), np.ldexp(1.0, eg))
    _eig_residual_ok(T, Zg[:, ::97], list(range(0, 2048, 97)))


def test_gpu_trevc_c3_sampled_full_size(ms):
    """Config 3 (m = 8192 complex, n_b = 128): full GPU run, oracle on sampled columns."""
    T = inputs.c3_trevc_complex()
    Zg, sc, eg = gpu_trevc(ms, T, 128)
    # 1024 columns: both ends of every block boundary region plus a seeded uniform sample
    rng = np.random.default_rng(33)
    fixed = [0, 1, 2, 127, 128, 129, 4095, 4096] + list(range(8128, 8192))
    rest = sorted(set(int(c) for c in rng.choice(8128, 1200, replace=False)) - set(fixed))
    cols = sorted(fixed + rest[:1024 - len(fixed)])
    assert len(cols) == 1024
    Zo, eo = oracle.trevc(T, nb=128, cols=cols)
    rel, de = assert_parity(Zg[:, cols], eg[cols], Zo, eo, what="c3")
    _log_parity("c3 full size, sampled columns", rel, de, {"rescaled": int((eo < 0).sum()), "min_e": int(eo.min())})
    _eig_residual_ok(T, Zg[:, cols[-3:]], cols[-3:])


def test_gpu_trevc_c3_shape_full_compare(ms):
    T = inputs.c3_trevc_complex(m=1000)
    Zg, sc, eg = gpu_trevc(ms, T, 128)
    Zo, eo = oracle.trevc(T, nb=128)
    assert_parity(Zg, eg, Zo, eo, what="c3 m=1000")


def test_gpu_trevc_c5_sampled_full_size(ms):
    """Config 5 (m = n = 16384 complex, safe, n_b = 128) exactly as bench.py launches it; the oracle
    computes a sample of columns one by one (columns are independent)."""
    T = inputs.c5_grcar_like()
    Zg, sc, eg = gpu_trevc(ms, T, 128)
    # 512 columns: the last 64, block-boundary columns, a seeded uniform sample
    rng = np.random.default_rng(55)
    fixed = [0, 1, 2, 3, 4, 100, 127, 128, 1023, 1024, 4000, 8191, 8192, 12000] + list(range(16320, 16384))
    rest = sorted(set(int(c) for c in rng.choice(16320, 600, replace=False)) - set(fixed))
    cols = sorted(fixed + rest[:512 - len(fixed)])
    assert len(cols) == 512
    Zo, eo = oracle.trevc(T, nb=128, cols=cols)
    rel, de = assert_parity(Zg[:, cols], eg[cols], Zo, eo, what="c5")
    _log_parity("c5 full size, sampled columns", rel, de, {"rescaled": int((eo < 0).sum()), "min_e": int(eo.min())})
    assert (eg < -1000).sum() > 1000               # extreme rescaling is exercised
    assert np.all(np.isfinite(Zg))
    _eig_residual_ok(T, Zg[:, [4000]], [4000])


def test_gpu_trevc_column_subset_bit_identical(ms):
    """Columns are independent: a shard (block-cyclic subset, as multi-GPU runs use) reproduces the
    full run bit for bit (fixed reduction order, no shape-dependent split)."""
    T = inputs.c5_grcar_like(m=1500)
    Zf, sf, ef = gpu_trevc(ms, T, 128)
    for P, r in [(2, 1), (4, 3), (8, 0)]:
        cols = [k for k in range(1500) if (k // 16) % P == r]
        Zs, ss, es = gpu_trevc(ms, T, 128, cols=cols)
        assert np.array_equal(Zs, Zf[:, cols]) and np.array_equal(es, ef[cols])


def test_gpu_trevc_real_and_complex_agree(ms):
    """A real T run through the complex path gives the real path's answer."""
    T = inputs.c2_trevc_real(m=300)
    Zr, _, er = gpu_trevc(ms, T, 64)
    Zc, _, ec = gpu_trevc(ms, T.astype(complex), 64)
    assert np.array_equal(er, ec)
    assert np.max(np.abs(Zc - Zr)) <= 1e-12 * np.max(np.abs(Zr))


# ------------------------------------------------------------------------------- pseudospectra
def gpu_ps(ms, U, z, v0, iters=15, nb=64):
    import torch
    sig, flags = ms.pseudospectra(dev(U), dev(z), dev(v0), iters=iters, nb=nb)
    torch.cuda.synchronize()
    return host(sig), host(flags)


def test_gpu_pseudospectra_small_full_grid(ms):
    U, z, v0 = inputs.c4_pseudospectra(m=100, npx=16)
    sg, fg = gpu_ps(ms, U, z, v0, nb=32)
    so, fo = oracle.pseudospectra(U, z, iters=15, v0=v0, nb=32)
    assert np.array_equal(fg, fo)
    assert np.max(np.abs(sg - so) / so) <= 1e-8


def test_gpu_pseudospectra_golden(ms):
    for case in GOLD["pseudospectra"]:
        U = np.array(case["U"], complex)
        z = np.array([complex(*v) for v in case["z"]])
        v0 = np.ones(U.shape[0], complex) / np.sqrt(U.shape[0])
        sg, fg = gpu_ps(ms, U, z, v0, nb=1)
        assert np.allclose(sg, case["sigma"], rtol=1e-13)


def test_gpu_pseudospectra_c4_full_size_sampled(ms):
    """Config 4 at full size (m = 1024, 128^2 points, 15 steps); oracle on a sample of points."""
    U, z, v0 = inputs.c4_pseudospectra()
    sg, fg = gpu_ps(ms, U, z, v0, nb=64)
    idx = np.random.default_rng(4).choice(z.shape[0], 1020, replace=False)
    idx = np.unique(np.concatenate([idx, [0, 127, 128 * 64 + 64, 16383]]))
    so, fo = oracle.pseudospectra(U, z[idx], iters=15, v0=v0, nb=64)
    assert np.array_equal(fg[idx], fo) and not fo.any()
    rel = np.abs(sg[idx] - so) / so
    assert rel.max() <= 1e-8
    _log_parity("c4 full size, sampled points (sigma_min rel. diff)", rel, np.zeros(len(idx), np.int64))
    assert np.all(np.isfinite(sg)) and np.all(sg > 0)


def test_gpu_pseudospectra_singular_point(ms):
    m = 30
    J = (2.0 * np.eye(m) + np.diag(np.ones(m - 1), 1)).astype(complex)
    z = np.array([2.0 + 0j, 0.5 + 0.5j])
    v0 = np.ones(m, complex) / np.sqrt(m)
    sg, fg = gpu_ps(ms, J, z, v0, nb=8)
    so, fo = oracle.pseudospectra(J, z, iters=15, v0=v0, nb=8)
    assert list(fg) == list(fo) == [1, 0]
    assert np.isfinite(sg[0]) and sg[0] < 1e-200
    assert abs(sg[1] - so[1]) <= 1e-8 * so[1]


# ------------------------------------------------------------------------------- probes
def test_gpu_fp64_peak_probe(ms):
    dmma, dfma = ms.fp64_peak(20.0)
    assert 5.0 < dmma < 100.0 and 5.0 < dfma < 100.0
