"""Independent reference arithmetic for the pins (long double / mpmath / LAPACK).

Nothing here calls the oracle or the CUDA path; tests compare both against these.
"""
from __future__ import annotations

import numpy as np

LD = np.longdouble
CLD = np.clongdouble
EPS = 2.0 ** -53
OMEGA = 2.0 ** 970


def shifted(U, s):
    A = np.array(U, dtype=np.result_type(U, s), order="F", copy=True)
    A = np.triu(A)
    A[np.arange(A.shape[0]), np.arange(A.shape[0])] -= s
    return A


def residual_ratio(U, s, x, e, b, op="N"):
    """Normwise backward error ||(U - sI)x - c b|| / (||U - sI|| ||x|| + |c| ||b||) in long double,
    inf-norms (op C: ||U - sI||_1 = ||(U - sI)^H||_inf), c = 2^e (never underflows here)."""
    A = shifted(U, s)
    cplx = np.iscomplexobj(A) or np.iscomplexobj(x) or np.iscomplexobj(b)
    T = CLD if cplx else LD
    A = A.astype(T)
    if op == "C":
        A = A.conj().T
    xl = np.asarray(x).astype(T)
    bl = np.asarray(b).astype(T)
    c = np.ldexp(LD(1.0), int(e))
    r = A @ xl - c * bl
    nA = np.max(np.sum(np.abs(A), axis=1))
    den = nA * np.max(np.abs(xl)) + c * np.max(np.abs(bl))
    if den == 0:
        return 0.0
    return float(np.max(np.abs(r)) / den)


def backsub_longdouble(U, s, b, r=None):
    """Unscaled back substitution for (U - sI) x = b in extended precision (x87 long double on
    x86: exponent range 2^+-16382), rows [0, r).  Returns x (long double)."""
    m = U.shape[0]
    r = m if r is None else r
    cplx = np.iscomplexobj(U) or np.iscomplexobj(b) or np.iscomplexobj(s)
    T = CLD if cplx else LD
    A = np.asarray(U)[:r, :r].astype(T)
    x = np.asarray(b)[:r].astype(T).copy()
    sl = T(s)
    for l in range(r - 1, -1, -1):
        x[l] = x[l] / (A[l, l] - sl)
        x[:l] -= x[l] * A[:l, l]
    return x


def normwise_diff_aligned(x_test, e_test, x_ref_ld, e_ref=0):
    """|| 2^(e_ref - e_test) x_test - x_ref || / ||x_ref|| computed in long double."""
    xt = np.asarray(x_test).astype(CLD if np.iscomplexobj(x_test) else LD)
    xt = xt * np.ldexp(LD(1.0), int(e_ref) - int(e_test))
    xr = np.asarray(x_ref_ld)
    den = np.max(np.abs(xr))
    if den == 0:
        return float(np.max(np.abs(xt)))
    return float(np.max(np.abs(xt - xr)) / den)


def log2_absmax(x) -> float:
    a = np.max(np.abs(np.asarray(x)))
    if a == 0:
        return -np.inf
    return float(np.log2(a))
