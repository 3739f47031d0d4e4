"""GPU parity of every update-GEMM / diagonal-grid variant the runtime switches select (README
"Runtime switches"): two or three consumer warpgroups, with and without the
staggered start, the unbalanced diagonal grid, look-ahead off.  The switches are read once per
process, so each variant runs in a subprocess that writes its results; the comparison against
the oracle (R20/R21) happens here.  Shapes: TriangEig complex m = 1100 at n_b = 128
(K = 128, a few tiles per CTA, look-ahead active) and n_b = 64 (K = 64), and a complex op C safe
solve (the conjugate-transpose operand path)."""
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
out = {}
T = inputs.c3_trevc_complex(m=1100)
for nb in (128, 64):
    Z, sc, e = ms.trevc(dev(T), nb=nb)
    torch.cuda.synchronize()
    out[f"Z{nb}"], out[f"e{nb}"] = host(Z), host(e)
from tests.test_gpu_gemm_variants import solve_inputs
U, s, B = solve_inputs()
X, sc, e = ms.solve(dev(U), dev(np.ascontiguousarray(s)), dev(B), safe=True, op="C", nb=64)
torch.cuda.synchronize()
out["XC"], out["eC"] = host(X), host(e)
np.savez(sys.argv[1], **out)
"""

def solve_inputs(m: int = 700, n: int = 300):
    """Well-conditioned complex upper-triangular U (diagonal in [1, 2] + small imaginary part),
    shifts in a disc of radius 0.4, Gaussian right-hand sides; seeded."""
    rng = np.random.default_rng([78, m, n])
    U = (np.triu(rng.standard_normal((m, m))) + 1j * np.triu(rng.standard_normal((m, m)))) / np.sqrt(m)
    U[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m) + 1j * rng.uniform(-0.3, 0.3, m)
    s = inputs.random_shifts(n, True, m, center=0.0, radius=0.4)
    B = inputs.random_rhs(m, n, True, 5)
    return np.asfortranarray(U), s, B


VARIANTS = {
    "two_groups_no_stagger": {"MSTRSM_3M_GROUPS": "2", "MSTRSM_3P_PHASE": "0"},
    "two_groups_stagger3": {"MSTRSM_3M_GROUPS": "2", "MSTRSM_3P_PHASE": "3"},
    "three_groups_no_stagger": {"MSTRSM_3M_GROUPS": "3", "MSTRSM_3P_PHASE": "0"},
    "three_groups_stagger1": {"MSTRSM_3M_GROUPS": "3", "MSTRSM_3P_PHASE": "1"},
    "diag_unbalanced": {"MSTRSM_DIAG_BALANCE": "0"},
    "lookahead": {"MSTRSM_LOOKAHEAD": "1"},
}


@pytest.fixture(scope="module")
def oracle_results():
    T = inputs.c3_trevc_complex(m=1100)
    res = {nb: oracle.trevc(T, nb=nb) for nb in (128, 64)}
    U, s, B = solve_inputs()
    res["C"] = oracle.mstrsm(U, s, B, safe=True, op="C", nb=64)
    return res


@pytest.mark.parametrize("name", sorted(VARIANTS))
def test_gpu_gemm_variant_parity(name, oracle_results, tmp_path):
    path = str(tmp_path / "out.npz")
    env = dict(os.environ, **VARIANTS[name])
    r = subprocess.run([sys.executable, "-c", _SCRIPT, path, ROOT], env=env, cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = np.load(path)
    for nb in (128, 64):
        Zo, eo = oracle_results[nb]
        assert_parity(got[f"Z{nb}"], got[f"e{nb}"], Zo, eo, what=f"{name} trevc nb={nb}")
    Xo, eo = oracle_results["C"]
    assert_parity(got["XC"], got["eC"], Xo, eo, what=f"{name} op C solve")
