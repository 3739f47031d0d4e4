"""CPU oracle for the blocked (safe) multi-shift triangular solve (arXiv 1607.01477).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py`` (its ``cpu_baseline`` leg and ``--impl reference``) may import
this package.  It shares no code with the CUDA product path in
``paper_1607_01477_b200/``; the two meet only in the seeded input generators
(``paper_1607_01477_b200/inputs.py``, which holds none of the method's
arithmetic).

The arithmetic lives in plain C (``mstrsm_oracle.c`` + ``oracle_algo.inc``),
built with ``-O2 -ffp-contract=off`` into ``liboracle.so``; this module only
marshals numpy arrays.  Every C function cites the PAPER.md passage it follows.

Parity pins (tests/test_oracle_pins.py) tie each function to something other
than itself: closed forms, hand-derived rescale cases, LAPACK/SVD/mpmath
cross-checks, extended-precision references, identities.  See DESIGN.md §4.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

OMEGA = 2.0 ** 970  # R1

c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double
c_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile liboracle.so (plain C, no FMA contraction, no fast-math)."""
    src = [os.path.join(_HERE, "mstrsm_oracle.c")]
    deps = src + [os.path.join(_HERE, f) for f in ("oracle_algo.inc", "oracle_gen.inc", "oracle_scalar.h")]
    if not force and os.path.exists(_LIB_PATH):
        lib_m = os.path.getmtime(_LIB_PATH)
        if all(os.path.getmtime(d) <= lib_m for d in deps):
            return _LIB_PATH
    cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared",
           "-pthread", "-o", _LIB_PATH] + src + ["-lm"]
    subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        for sfx in ("d", "z"):
            f = getattr(lib, f"oracle_mstrsm_{sfx}")
            f.restype = c_int
            f.argtypes = [c_int, c_int, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64,
                          c_vp, c_vp, c_int, c_int]
            f = getattr(lib, f"oracle_norms_{sfx}")
            f.restype = None
            f.argtypes = [c_int, c_vp, c_i64, c_i64, c_int, c_vp, c_vp, c_vp]
            f = getattr(lib, f"oracle_trevc_{sfx}")
            f.restype = c_int
            f.argtypes = [c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_int, c_int]
            f = getattr(lib, f"oracle_mstrsm_gen_{sfx}")
            f.restype = c_int
            f.argtypes = [c_int, c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_i64,
                          c_vp, c_vp, c_int, c_int]
            f = getattr(lib, f"oracle_tgevc_{sfx}")
            f.restype = c_int
            f.argtypes = [c_vp, c_i64, c_vp, c_i64, c_i64, c_vp, c_i64, c_vp, c_i64, c_vp, c_vp,
                          c_int, c_int]
        lib.oracle_pseudospectra_z.restype = c_int
        lib.oracle_pseudospectra_z.argtypes = [c_vp, c_i64, c_i64, c_vp, c_i64, c_int, c_vp, c_vp,
                                               c_vp, c_int, c_int]
        lib.oracle_spectral_cloud_z.restype = c_int
        lib.oracle_spectral_cloud_z.argtypes = [c_vp, c_i64, c_i64, c_vp, c_i64, c_int, c_dbl, c_vp, c_vp,
                                                c_vp, c_vp, c_int, c_int]
        lib.oracle_tridiag_lmax.restype = c_dbl
        lib.oracle_tridiag_lmax.argtypes = [c_vp, c_vp, c_int]
        lib.oracle_zmod.restype = c_dbl
        lib.oracle_zmod.argtypes = [c_dbl, c_dbl]
        lib.oracle_zdiv.restype = None
        lib.oracle_zdiv.argtypes = [c_dbl, c_dbl, c_dbl, c_dbl, c_vp]
        lib.oracle_minpow2.restype = c_int
        lib.oracle_minpow2.argtypes = [c_dbl, c_dbl]
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(c_vp) if a is not None else None


def _sfx(dtype) -> str:
    if dtype == np.float64:
        return "d"
    if dtype == np.complex128:
        return "z"
    raise TypeError(f"oracle supports float64/complex128, got {dtype}")


def _fortran(a: np.ndarray, dtype) -> np.ndarray:
    return np.asfortranarray(np.asarray(a, dtype=dtype))


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def mstrsm(U, shifts, B, *, op: str = "N", safe: bool = True, nb: int = 64, row_end=None,
           nthreads: int = 0):
    """Solve (U - s_j I) x_j = c_j b_j (op N) or (U - s_j I)^H x_j = c_j b_j (op C).

    Alg. 3 (safe=False, c_j = 1) or Alg. 5 (safe=True) of the paper, one column at a
    time.  Returns (X, e) with c_j = 2**e_j.  Rows >= row_end[j] of column j are zero.
    """
    lib = _load()
    U = np.asarray(U)
    dtype = np.complex128 if (np.iscomplexobj(U) or np.iscomplexobj(B) or np.iscomplexobj(shifts)) \
        else np.float64
    sfx = _sfx(dtype)
    U = _fortran(U, dtype)
    X = np.array(B, dtype=dtype, order="F", copy=True)
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    m, n = X.shape
    assert U.shape == (m, m)
    s = np.ascontiguousarray(np.asarray(shifts, dtype=dtype).reshape(-1))
    assert s.shape[0] == n
    re = None
    if row_end is not None:
        re = np.ascontiguousarray(np.asarray(row_end, dtype=np.int64).reshape(-1))
        assert re.shape[0] == n
    e = np.zeros(n, dtype=np.int32)
    rc = getattr(lib, f"oracle_mstrsm_{sfx}")(0 if op == "N" else 1, 1 if safe else 0, _ptr(U),
                                              max(1, m), m, _ptr(s), 1, _ptr(X), max(1, m), n,
                                              _ptr(re), _ptr(e), nb, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_mstrsm_{sfx} returned {rc}")
    return X, e


def mstrsm_side(A, shifts, B, *, side: str = "L", uplo: str = "U", safe: bool = True, nb: int = 64,
                nthreads: int = 0):
    """The footnote family of P:58-62, each case written as the triangular system
    it is, then solved by the (pinned) op N / op C oracle:

      L,U: (A - s I) x = c b                       -> mstrsm(A, s, B, op N)
      L,L: (A - s I) x = c b,  A lower              =  (A^H - conj(s) I)^H x = c b   -> op C on A^H
      R,U: x^T (A - s I) = c b^T                    =  (A^T - s I) x = c b = (conj(A) - conj(s) I)^H x
      R,L: x^T (A - s I) = c b^T,  A lower          =  (A^T - s I) x = c b, A^T upper -> op N on A^T

    Right cases: B is n x m (row j = b_j^T) and so is the returned X.  Returns (X, e)."""
    A = np.asarray(A)
    s = np.asarray(shifts).reshape(-1)
    B = np.asarray(B)
    cx = np.iscomplexobj(A) or np.iscomplexobj(s) or np.iscomplexobj(B)
    cj = (lambda v: np.conj(v)) if cx else (lambda v: v)
    if side == "L" and uplo == "U":
        return mstrsm(A, s, B, op="N", safe=safe, nb=nb, nthreads=nthreads)
    if side == "L":
        return mstrsm(np.triu(cj(A.T)), cj(s), B, op="C", safe=safe, nb=nb, nthreads=nthreads)
    if uplo == "U":
        X, e = mstrsm(np.triu(cj(A)), cj(s), B.T, op="C", safe=safe, nb=nb, nthreads=nthreads)
    else:
        X, e = mstrsm(np.triu(A.T), s, B.T, op="N", safe=safe, nb=nb, nthreads=nthreads)
    return np.asfortranarray(X.T), e


def norms(U, *, op: str = "N", nb: int = 64):
    """The norm pass: block-local column norms cnl, panel sums P, ||U||_inf (op N) or
    ||U^H||_inf (op C)."""
    lib = _load()
    U = np.asarray(U)
    dtype = np.complex128 if np.iscomplexobj(U) else np.float64
    U = _fortran(U, dtype)
    m = U.shape[0]
    nblk = (m + nb - 1) // nb
    cnl = np.zeros(m)
    P = np.zeros(max(nblk, 1))
    un = np.zeros(1)
    getattr(lib, f"oracle_norms_{_sfx(dtype)}")(0 if op == "N" else 1, _ptr(U), max(1, m), m, nb,
                                                _ptr(cnl), _ptr(P), _ptr(un))
    return cnl, P[:nblk], float(un[0])


def trevc(T, *, nb: int = 64, cols=None, nthreads: int = 0):
    """TriangEig (Alg. 6): eigenvectors Z of upper-triangular T, Z(k,k) = c_k = 2**e_k.

    With ``cols`` (sorted global indices), returns only those columns (m x len(cols))."""
    lib = _load()
    T = np.asarray(T)
    dtype = np.complex128 if np.iscomplexobj(T) else np.float64
    T = _fortran(T, dtype)
    m = T.shape[0]
    c = None
    if cols is not None:
        c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64).reshape(-1))
        ncols = c.shape[0]
    else:
        ncols = m
    Z = np.zeros((m, ncols), dtype=dtype, order="F")
    e = np.zeros(ncols, dtype=np.int32)
    rc = getattr(lib, f"oracle_trevc_{_sfx(dtype)}")(_ptr(T), max(1, m), m, _ptr(c), ncols, _ptr(Z),
                                                     max(1, m), _ptr(e), nb, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_trevc returned {rc}")
    return Z, e


def eig_backtransform(Q, Z):
    """X := Q Z, the back-transformation step of Eig (`X := Q Z  (xGEMM)`).

    The step is a plain matrix product, taken as the library primitive (numpy matmul in fp64);
    column q of X keeps the scale c_q of Z(:, q)."""
    return np.asfortranarray(np.asarray(Q) @ np.asarray(Z))


def trevc_qz(T, Q, *, nb: int = 64, nthreads: int = 0):
    """Eig's last two steps: Z = TriangEig(T) (Alg. 6, ``trevc``), X = Q Z.
    Returns (X, e): eigenvectors of A = Q T Q^H, column k scaled by c_k = 2**e_k."""
    Z, e = trevc(T, nb=nb, nthreads=nthreads)
    return eig_backtransform(Q, Z), e


def mstrsm_gen(U, V, shifts, B, *, safe: bool = True, nb: int = 64, row_end=None,
               nthreads: int = 0):
    """Generalized multi-shift solve (U - s_j V) x_j = c_j b_j: Alg. 7 (safe=False) or Alg. 8
    (safe=True) of the paper's appendix, one column at a time.  Returns (X, e), c_j = 2**e_j."""
    lib = _load()
    cplx = any(np.iscomplexobj(a) for a in (U, V, shifts, B))
    dtype = np.complex128 if cplx else np.float64
    sfx = _sfx(dtype)
    U = _fortran(np.asarray(U), dtype)
    V = _fortran(np.asarray(V), dtype)
    X = np.array(B, dtype=dtype, order="F", copy=True)
    if X.ndim == 1:
        X = X.reshape(-1, 1, order="F")
    m, n = X.shape
    assert U.shape == (m, m) and V.shape == (m, m)
    s = np.ascontiguousarray(np.asarray(shifts, dtype=dtype).reshape(-1))
    assert s.shape[0] == n
    re = None
    if row_end is not None:
        re = np.ascontiguousarray(np.asarray(row_end, dtype=np.int64).reshape(-1))
    e = np.zeros(n, dtype=np.int32)
    rc = getattr(lib, f"oracle_mstrsm_gen_{sfx}")(1 if safe else 0, _ptr(U), max(1, m), _ptr(V),
                                                  max(1, m), m, _ptr(s), 1, _ptr(X), max(1, m), n,
                                                  _ptr(re), _ptr(e), nb, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_mstrsm_gen_{sfx} returned {rc}")
    return X, e


def tgevc(T, S, *, nb: int = 64, cols=None, nthreads: int = 0):
    """GeneralizedTriangEig (Alg. 9): eigenvectors of the upper-triangular pencil (T, S),
    lambda_k = T(k,k)/S(k,k), Z(k,k) = c_k = 2**e_k.  Returns (Z, lambda, e)."""
    lib = _load()
    cplx = np.iscomplexobj(T) or np.iscomplexobj(S)
    dtype = np.complex128 if cplx else np.float64
    T = _fortran(np.asarray(T), dtype)
    S = _fortran(np.asarray(S), dtype)
    m = T.shape[0]
    c = None
    if cols is not None:
        c = np.ascontiguousarray(np.asarray(cols, dtype=np.int64).reshape(-1))
        ncols = c.shape[0]
    else:
        ncols = m
    Z = np.zeros((m, ncols), dtype=dtype, order="F")
    lam = np.zeros(ncols, dtype=dtype)
    e = np.zeros(ncols, dtype=np.int32)
    rc = getattr(lib, f"oracle_tgevc_{_sfx(dtype)}")(_ptr(T), max(1, m), _ptr(S), max(1, m), m, _ptr(c),
                                                     ncols, _ptr(Z), max(1, m), _ptr(lam), _ptr(e), nb,
                                                     nthreads)
    if rc != 0:
        raise ValueError(f"oracle_tgevc returned {rc}")
    return Z, lam, e


def pseudospectra(U, z, *, iters: int = 15, v0=None, nb: int = 64, nthreads: int = 0):
    """sigma_min(U - z I) for every point z by `iters` inverse-Lanczos steps (Alg. VL)."""
    lib = _load()
    U = _fortran(U, np.complex128)
    m = U.shape[0]
    z = np.ascontiguousarray(np.asarray(z, dtype=np.complex128).reshape(-1))
    if v0 is None:
        v0 = np.ones(m, dtype=np.complex128) / np.sqrt(m)
    v0 = np.ascontiguousarray(np.asarray(v0, dtype=np.complex128))
    sig = np.zeros(z.shape[0])
    flags = np.zeros(z.shape[0], dtype=np.int32)
    rc = lib.oracle_pseudospectra_z(_ptr(U), max(1, m), m, _ptr(z), z.shape[0], iters, _ptr(v0),
                                    _ptr(sig), _ptr(flags), nb, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_pseudospectra_z returned {rc}")
    return sig, flags


def spectral_cloud(U, z, *, maxit: int = 15, tol: float = 1e-10, v0=None, nb: int = 64,
                   nthreads: int = 0):
    """SpectralCloud: resolvent-norm estimates 1/sigma_min(U - z I) are returned
    as sigma_min per point.  Alg. VL's Lanczos with per-point deflation (R33): a point stops after
    the first step k >= 2 whose Ritz value theta_k = lambda_max(T_k) satisfies
    |theta_k - theta_{k-1}| <= tol theta_k.  Returns (sigma, flags, its): flags bit0 = rescaled
    solve (R25), bit1 = not settled within maxit steps; its = Lanczos steps taken."""
    lib = _load()
    U = _fortran(U, np.complex128)
    m = U.shape[0]
    z = np.ascontiguousarray(np.asarray(z, dtype=np.complex128).reshape(-1))
    if v0 is None:
        v0 = np.ones(m, dtype=np.complex128) / np.sqrt(m)
    v0 = np.ascontiguousarray(np.asarray(v0, dtype=np.complex128))
    sig = np.zeros(z.shape[0])
    flags = np.zeros(z.shape[0], dtype=np.int32)
    its = np.zeros(z.shape[0], dtype=np.int32)
    rc = lib.oracle_spectral_cloud_z(_ptr(U), max(1, m), m, _ptr(z), z.shape[0], maxit, float(tol),
                                     _ptr(v0), _ptr(sig), _ptr(flags), _ptr(its), nb, nthreads)
    if rc != 0:
        raise ValueError(f"oracle_spectral_cloud_z returned {rc}")
    return sig, flags, its


def window_grid(x0: float, x1: float, nx: int, y0: float, y1: float, ny: int):
    """SpectralWindow's grid: endpoint-inclusive linspace on both axes, point index
    ix + nx * iy (R15)."""
    gx = np.linspace(x0, x1, nx)
    gy = np.linspace(y0, y1, ny)
    return (gx[None, :] + 1j * gy[:, None]).reshape(-1)


def spectral_window(U, x0, x1, nx, y0, y1, ny, **kw):
    """SpectralWindow: SpectralCloud over the grid of window_grid."""
    return spectral_cloud(U, window_grid(x0, x1, nx, y0, y1, ny), **kw)


def portrait_window(U):
    """SpectralPortrait's automatic window (R34, after S:411): the bounding box of
    diag(U) padded on each side by 0.25 max(box width, box height, 1e-2 ||U||_inf), ||U||_inf the
    max row sum of |U(i, k)| over k >= i.  Returns (x0, x1, y0, y1)."""
    U = np.asarray(U)
    d = np.diag(U)
    x0, x1 = float(np.min(d.real)), float(np.max(d.real))
    y0, y1 = float(np.min(d.imag)), float(np.max(d.imag))
    unorm = float(np.max(np.sum(np.abs(np.triu(U)), axis=1)))
    pad = 0.25 * max(x1 - x0, y1 - y0, 1e-2 * unorm)
    return x0 - pad, x1 + pad, y0 - pad, y1 + pad


def spectral_portrait(U, nx, ny, **kw):
    """SpectralPortrait: SpectralWindow over portrait_window(U).  Returns
    (sigma, flags, its, window)."""
    x0, x1, y0, y1 = portrait_window(U)
    sig, flags, its = spectral_window(U, x0, x1, nx, y0, y1, ny, **kw)
    return sig, flags, its, (x0, x1, y0, y1)


def tridiag_lmax(a, b) -> float:
    lib = _load()
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    b = np.ascontiguousarray(np.asarray(b, dtype=np.float64))
    return float(lib.oracle_tridiag_lmax(_ptr(a), _ptr(b), a.shape[0]))


def zmod(z: complex) -> float:
    return float(_load().oracle_zmod(float(np.real(z)), float(np.imag(z))))


def zdiv(a: complex, b: complex) -> complex:
    out = np.zeros(2)
    _load().oracle_zdiv(a.real, a.imag, b.real, b.imag, _ptr(out))
    return complex(out[0], out[1])


def minpow2(a: float, L: float) -> int:
    return int(_load().oracle_minpow2(a, L))
