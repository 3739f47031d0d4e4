"""GPU parity of the real path's launch switches (README "Runtime switches"): the
update GEMM's early A issue (`gemm_ws_kernel`, first k-tiles copied before the dependent-launch
wait) forced on for every launch (several tiles per consumer group after the early ones), forced
off, and combined with the diagonal kernel's start trigger; the real update on the persistent
kernel only / the one-tile-per-CTA kernel only (the default picks per launch), which must agree
bit for bit (same k order, same epilogue roundings: a multi-GPU shard may take the other kernel
than the full solve).  Shapes: real TriangEig m = 700 at
n_b = 64 (K = 64: more k-tiles than ring stages) and n_b = 32 (K = 32: fewer), and real safe
solves op N at n_b = 13 (ragged k-tiles in the early copies) and op C at n_b = 32.  The switches
are read once per process, so each variant runs in a subprocess; the comparison against the
oracle (R20/R21) happens here."""
from __future__ import annotations

import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_1607_01477_b200 import inputs
from tests.gpu_util import assert_parity

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, sys.argv[2])
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
from tests.gpu_util import dev, host
from tests.test_gpu_real_launch import solve_inputs
out = {}
T = inputs.c2_trevc_real(m=700)
for nb in (64, 32):
    Z, sc, e = ms.trevc(dev(T), nb=nb)
    torch.cuda.synchronize()
    out[f"Z{nb}"], out[f"e{nb}"] = host(Z), host(e)
U, s, B = solve_inputs()
for op, nb in (("N", 13), ("C", 32)):
    X, sc, e = ms.solve(dev(U), dev(np.ascontiguousarray(s)), dev(B), safe=True, op=op, nb=nb)
    torch.cuda.synchronize()
    out["X" + op], out["e" + op] = host(X), host(e)
np.savez(sys.argv[1], **out)
"""


def solve_inputs(m: int = 530, n: int = 200):
    """Real upper-triangular U with diagonal in [1, 2] and N(0, 1/m) strict upper part, real
    shifts in [-0.4, 0.4], Gaussian right-hand sides; seeded."""
    rng = np.random.default_rng([79, m, n])
    U = np.triu(rng.standard_normal((m, m))) / np.sqrt(m)
    U[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m)
    s = inputs.random_shifts(n, False, m, center=0.0, radius=0.4)
    B = inputs.random_rhs(m, n, False, 6)
    return np.asfortranarray(U), s, B


VARIANTS = {
    "early_a_always": {"MSTRSM_EARLY_A": "1"},
    "early_a_never": {"MSTRSM_EARLY_A": "0"},
    "early_a_with_diag_trigger": {"MSTRSM_EARLY_A": "1", "MSTRSM_DIAGL_TRIGGER": "1"},
    "gemm_real_ws": {"MSTRSM_GEMM_REAL": "ws"},
    "gemm_real_classic": {"MSTRSM_GEMM_REAL": "classic"},
    "both_triggers": {"MSTRSM_GEMM_TRIGGER": "1", "MSTRSM_DIAGL_TRIGGER": "1"},
    "no_gemm_trigger": {"MSTRSM_GEMM_TRIGGER": "0"},
}


@pytest.fixture(scope="module")
def oracle_results():
    T = inputs.c2_trevc_real(m=700)
    res = {nb: oracle.trevc(T, nb=nb) for nb in (64, 32)}
    U, s, B = solve_inputs()
    res["N"] = oracle.mstrsm(U, s, B, safe=True, op="N", nb=13)
    res["C"] = oracle.mstrsm(U, s, B, safe=True, op="C", nb=32)
    return res


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_gpu_real_launch_variant_parity(name, oracle_results, tmp_path):
    path = str(tmp_path / "out.npz")
    env = dict(os.environ, **VARIANTS[name])
    r = subprocess.run([sys.executable, "-c", _SCRIPT, path, ROOT], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(path)
    for nb in (64, 32):
        Zo, eo = oracle_results[nb]
        assert_parity(got[f"Z{nb}"], got[f"e{nb}"], Zo, eo, what=f"{name} real trevc nb={nb}")
    for op in ("N", "C"):
        Xo, eo = oracle_results[op]
        assert_parity(got["X" + op], got["e" + op], Xo, eo, what=f"{name} real op {op} solve")


def _run(tmp_path, name, env_over):
    path = str(tmp_path / f"{name}.npz")
    r = subprocess.run([sys.executable, "-c", _SCRIPT, path, ROOT], env=dict(os.environ, **env_over), cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return np.load(path)


def test_gpu_real_gemm_kernels_bit_identical(tmp_path):
    a = _run(tmp_path, "ws", {"MSTRSM_GEMM_REAL": "ws"})
    b = _run(tmp_path, "classic", {"MSTRSM_GEMM_REAL": "classic"})
    for k in a.files:
        assert np.array_equal(a[k], b[k]), k
