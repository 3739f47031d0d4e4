"""Helpers for the GPU parity tests (host <-> device marshalling and the R20/R21 comparison)."""
from __future__ import annotations

import numpy as np


def dev(a: np.ndarray):
    """numpy (any order) -> column-major CUDA tensor."""
    import torch
    a = np.asfortranarray(a)
    t = torch.from_numpy(a).cuda()
    if t.dim() == 2:
        assert t.stride(0) == 1
    return t


def host(t) -> np.ndarray:
    return t.cpu().numpy()


def aligned_diff(Xg, eg, Xo, eo):
    """Per-column ||2^(eo-eg) x_gpu - x_orc||_inf / ||x_orc||_inf (R20) and |eg - eo| (R21)."""
    Xg = np.asarray(Xg)
    Xo = np.asarray(Xo)
    n = Xo.shape[1]
    rel = np.zeros(n)
    de = np.abs(np.asarray(eg, dtype=np.int64) - np.asarray(eo, dtype=np.int64))
    for j in range(n):
        xo = Xo[:, j]
        xg = np.ldexp(Xg[:, j].real, int(eo[j]) - int(eg[j]))
        if np.iscomplexobj(Xg):
            xg = xg + 1j * np.ldexp(Xg[:, j].imag, int(eo[j]) - int(eg[j]))
        den = np.max(np.abs(xo))
        if den == 0:
            rel[j] = np.max(np.abs(xg))
        else:
            rel[j] = np.max(np.abs(xg - xo)) / den
    return rel, de


def assert_parity(Xg, eg, Xo, eo, tol=1e-9, what=""):
    rel, de = aligned_diff(Xg, eg, Xo, eo)
    assert np.all(np.isfinite(Xg)), f"{what}: non-finite GPU output"
    assert de.max(initial=0) <= 1, f"{what}: |e_gpu - e_orc| = {de.max()} > 1"
    assert rel.max(initial=0) <= tol, f"{what}: max normwise diff {rel.max():.3e} > {tol:g}"
    return rel, de
