"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs).

This module is shared by the oracle tests and the CUDA path.  It holds NONE of
the method's arithmetic: it only draws random numbers into arrays (U, shifts,
right-hand sides, grid points, Lanczos start vectors).  Everything is generated
on the host with numpy so that the oracle and the GPU see identical inputs.

Recipe:
  * generator ``numpy.random.default_rng([160701477, cfg])`` per config;
  * draw order: diagonal, strictly-upper entries (column-major packed: for
    column k, rows 0..k-1; complex entries as ``standard_normal(2*cnt)`` split
    into (re, im) pairs), then shifts, then right-hand sides, then v0;
  * N(mu, v) means variance v; a complex N(0, v) is circular with E|z|^2 = v.

Paper workload -> stand-in (P = PAPER.md line):
  c1  P:714-719 (E1 scaling study) -> real, diag U[1,2], off-diag N(0,1/m)
  c2  BASELINE config 2 (real triangular eigenvectors)
  c3  P:729-731, P:745-746 (unit-ball matrices, Schur-factor shaped) -> complex
  c4  P:800-807, P:821-825 (Fox/Li pseudospectra; Fox/Li is NOT in this
      container) -> random complex triangular, diag in the unit disk
  c5  BASELINE config 5 (Grcar-like, scale-out)
"""
from __future__ import annotations

import numpy as np

SEED = 160701477


def _rng(cfg: int, salt: int = 0) -> np.random.Generator:
    return np.random.default_rng([SEED, cfg] if salt == 0 else [SEED, cfg, salt])


def _fill_strict_upper_real(U: np.ndarray, rng: np.random.Generator, std: float) -> None:
    m = U.shape[0]
    cnt = m * (m - 1) // 2
    v = rng.standard_normal(cnt) * std
    off = 0
    for k in range(1, m):
        U[:k, k] = v[off:off + k]
        off += k


def _fill_strict_upper_complex(U: np.ndarray, rng: np.random.Generator, std_per_part: float,
                               col_fn=None) -> None:
    """Strictly-upper complex entries, packed column-major; col_fn(k, vals) may edit column k."""
    m = U.shape[0]
    cnt = m * (m - 1) // 2
    v = rng.standard_normal(2 * cnt) * std_per_part
    off = 0
    for k in range(1, m):
        seg = v[2 * off:2 * (off + k)]
        col = seg[0::2] + 1j * seg[1::2]
        if col_fn is not None:
            col = col_fn(k, col)
        U[:k, k] = col
        off += k


def c1_plain_real(m: int = 256, n: int = 64):
    """Config 1: real U, diag Uniform[1,2], off-diag N(0,1/m); shifts U[-0.5,0.5]; B N(0,1)."""
    rng = _rng(1)
    U = np.zeros((m, m), order="F")
    U[np.arange(m), np.arange(m)] = rng.uniform(1.0, 2.0, m)
    _fill_strict_upper_real(U, rng, 1.0 / np.sqrt(m))
    shifts = rng.uniform(-0.5, 0.5, n)
    B = np.asfortranarray(rng.standard_normal((m, n)))
    return U, shifts, B


def c2_trevc_real(m: int = 2048):
    """Config 2: real T, diag = sorted distinct Uniform[-1,1], off-diag N(0,1)."""
    rng = _rng(2)
    while True:
        d = np.sort(rng.uniform(-1.0, 1.0, m))
        if np.all(np.diff(d) > 0):
            break
    T = np.zeros((m, m), order="F")
    T[np.arange(m), np.arange(m)] = d
    _fill_strict_upper_real(T, rng, 1.0)
    return T


def c3_trevc_complex(m: int = 8192):
    """Config 3: complex T, diag e^{i theta}, theta ~ U[0, 2pi); off-diag complex N(0,1)."""
    rng = _rng(3)
    theta = rng.uniform(0.0, 2.0 * np.pi, m)
    T = np.zeros((m, m), dtype=np.complex128, order="F")
    T[np.arange(m), np.arange(m)] = np.exp(1j * theta)
    _fill_strict_upper_complex(T, rng, np.sqrt(0.5))
    return T


def c4_grid(npx: int = 128, lo: float = -1.5, hi: float = 1.5):
    """Config 4 grid: endpoint-inclusive linspace on both axes, index = ix + npx*iy (R15)."""
    g = np.linspace(lo, hi, npx)
    return (g[None, :] + 1j * g[:, None]).reshape(-1)


def c4_pseudospectra(m: int = 1024, npx: int = 128):
    """Config 4: complex U, diag uniform in the unit disk, off-diag complex N(0,1/m);
    grid of npx^2 shifts over [-1.5,1.5]^2; v0 complex N(0,1) normalised."""
    rng = _rng(4)
    r = np.sqrt(rng.uniform(0.0, 1.0, m))
    phi = rng.uniform(0.0, 2.0 * np.pi, m)
    U = np.zeros((m, m), dtype=np.complex128, order="F")
    U[np.arange(m), np.arange(m)] = r * np.exp(1j * phi)
    _fill_strict_upper_complex(U, rng, np.sqrt(0.5 / m))
    z = c4_grid(npx)
    v = rng.standard_normal(2 * m)
    v0 = v[0::2] + 1j * v[1::2]
    v0 = v0 / np.linalg.norm(v0)
    return U, z, v0


def c5_grcar_like(m: int = 16384):
    """Config 5: diag 1 + complex N(0,1e-3); superdiagonals 1..3 = 1; col-row >= 4:
    complex N(0,1)/sqrt(m) (R16)."""
    rng = _rng(5)
    dz = rng.standard_normal(2 * m) * np.sqrt(0.5e-3)
    T = np.zeros((m, m), dtype=np.complex128, order="F")
    T[np.arange(m), np.arange(m)] = 1.0 + dz[0::2] + 1j * dz[1::2]

    def band(k, col):
        col[max(0, k - 3):k] = 1.0      # rows k-3..k-1 are the first three superdiagonals
        return col

    _fill_strict_upper_complex(T, rng, np.sqrt(0.5 / m), col_fn=band)
    return T


def random_rhs(m: int, n: int, complex_: bool, seed: int):
    """Extra dense right-hand sides for parity tests (N(0,1) entries)."""
    rng = np.random.default_rng([SEED, 100, seed])
    if complex_:
        v = rng.standard_normal((m, 2 * n))
        return np.asfortranarray(v[:, 0::2] + 1j * v[:, 1::2])
    return np.asfortranarray(rng.standard_normal((m, n)))


def random_shifts(n: int, complex_: bool, seed: int, center=0.0, radius=0.5):
    """Shifts uniform in a disk (P:718-719 draws them from the ball B(1.5, 0.5))."""
    rng = np.random.default_rng([SEED, 101, seed])
    if complex_:
        r = radius * np.sqrt(rng.uniform(0, 1, n))
        phi = rng.uniform(0, 2 * np.pi, n)
        return center + r * np.exp(1j * phi)
    return center + rng.uniform(-radius, radius, n)


def e1_hermitian_triangle(m: int, seed: int = 0):
    """P:714-719 generator: Hermitian matrix with eigenvalues U[1,2], strict lower triangle
    deleted (complex).  Q from the QR of a complex Gaussian."""
    rng = np.random.default_rng([SEED, 102, seed])
    G = rng.standard_normal((m, 2 * m))
    Q, _ = np.linalg.qr(G[:, 0::2] + 1j * G[:, 1::2])
    lam = rng.uniform(1.0, 2.0, m)
    H = (Q * lam) @ Q.conj().T
    return np.asfortranarray(np.triu(H))


def g1_pencil(m: int = 4096, complex_: bool = True, seed: int = 0):
    """Generalized stand-in, not a BASELINE config: an upper-triangular pencil
    (T, S) for GeneralizedTriangEig (Alg. 9).  T is Grcar-like as in config 5 (diag 1 + complex
    N(0,1e-3), superdiagonals 1..3 = 1, further entries complex N(0,1)/sqrt(m)), so the safe solve
    rescales heavily; S has diagonal 1 + N(0,1e-3) (real, finite eigenvalues lambda_k =
    T(k,k)/S(k,k) clustered like config 5's) and strictly upper entries N(0, 1/m) (complex circular
    when complex_)."""
    rng = np.random.default_rng([SEED, 103, seed])
    if complex_:
        dz = rng.standard_normal(2 * m) * np.sqrt(0.5e-3)
        T = np.zeros((m, m), dtype=np.complex128, order="F")
        T[np.arange(m), np.arange(m)] = 1.0 + dz[0::2] + 1j * dz[1::2]
    else:
        T = np.zeros((m, m), dtype=np.float64, order="F")
        T[np.arange(m), np.arange(m)] = 1.0 + rng.standard_normal(m) * np.sqrt(1e-3)

    def band(k, col):
        col[max(0, k - 3):k] = 1.0
        return col

    if complex_:
        _fill_strict_upper_complex(T, rng, np.sqrt(0.5 / m), col_fn=band)
        S = np.zeros((m, m), dtype=np.complex128, order="F")
        S[np.arange(m), np.arange(m)] = 1.0 + rng.standard_normal(m) * np.sqrt(1e-3)
        _fill_strict_upper_complex(S, rng, np.sqrt(0.5 / m))
    else:
        _fill_strict_upper_real(T, rng, np.sqrt(1.0 / m))
        for k in range(m):
            T[max(0, k - 3):k, k] = 1.0
        S = np.zeros((m, m), dtype=np.float64, order="F")
        S[np.arange(m), np.arange(m)] = 1.0 + rng.standard_normal(m) * np.sqrt(1e-3)
        _fill_strict_upper_real(S, rng, np.sqrt(1.0 / m))
    return T, S


def schur_pair(m: int, complex_: bool = True, seed: int = 0):
    """Back-transformation stand-in, not a BASELINE config: a Schur pair
    (T, Q) of A = Q T Q^H.  T is the config-3 (complex) or config-2 (real) generator at size m;
    Q is the orthonormal factor of the QR of a Gaussian matrix (complex circular / real)."""
    T = c3_trevc_complex(m) if complex_ else c2_trevc_real(m)
    rng = np.random.default_rng([SEED, 104, seed, m])
    G = rng.standard_normal((m, 2 * m if complex_ else m))
    Q, _ = np.linalg.qr(G[:, 0::2] + 1j * G[:, 1::2] if complex_ else G)
    return T, np.asfortranarray(Q)


def dense_q(m: int, complex_: bool = True, seed: int = 0):
    """A dense m x m stand-in for Q at bench sizes (a QR at m = 8192 would dominate the setup):
    entries N(0, 1/m) (complex circular), so ||Q(:,k)||_2 ~ 1.  Throughput of X = Q Z does not
    depend on Q being unitary."""
    rng = np.random.default_rng([SEED, 105, seed, m])
    if complex_:
        v = rng.standard_normal((m, 2 * m)) * np.sqrt(0.5 / m)
        return np.asfortranarray(v[:, 0::2] + 1j * v[:, 1::2])
    return np.asfortranarray(rng.standard_normal((m, m)) / np.sqrt(m))
