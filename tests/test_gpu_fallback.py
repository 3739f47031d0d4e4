"""GPU tests (-m gpu) of the diagonal step's synchronous fallback (diag_kernel<FB>, the exact
Alg. 4 order): with MSTRSM_DIAG_FORCE_FALLBACK=1 every guarded column is handed over
by the chunked kernel, so the whole safe path runs through the fallback.  The switch is read when
the library loads, hence a subprocess per case; results are compared with the oracle (R20/R21)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import oracle
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
from tests.gpu_util import aligned_diff
case = {case!r}
if case == "c2":
    T, nb = inputs.c2_trevc_real(), 64
elif case == "c5_1100":
    T, nb = inputs.c5_grcar_like(1100), 128
else:
    T, nb = inputs.c3_trevc_complex(2048), 128
Td = torch.from_numpy(np.asfortranarray(T)).cuda()
Z, sc, e = ms.trevc(Td, nb=nb)
torch.cuda.synchronize()
Z, e = Z.cpu().numpy(), e.cpu().numpy()
Zo, eo = oracle.trevc(T, nb=nb)
rel, de = aligned_diff(Z, e, Zo, eo)
print(json.dumps({{"max_rel": float(rel.max()), "max_de": int(de.max()), "finite": bool(np.isfinite(Z).all()),
                  "rescaled": int((eo < 0).sum()), "launches": int(ms.launch_count(0))}}))
"""


@pytest.mark.parametrize("case", ["c2", "c5_1100", "c3_2048"])
def test_forced_fallback_matches_oracle(case):
    env = dict(os.environ, MSTRSM_DIAG_FORCE_FALLBACK="1")
    out = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT, case=case)], env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["finite"] and r["rescaled"] > 0
    assert r["max_de"] <= 1 and r["max_rel"] <= 1e-9, r


_SCRIPT_IMPL = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import oracle
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
from tests.gpu_util import aligned_diff
case = {case!r}
res = {{}}
if case.startswith("trevc"):
    T, nb = (inputs.c5_grcar_like(700), 64) if case == "trevc_c" else (inputs.c2_trevc_real(2048), 64)
    Z, sc, e = ms.trevc(torch.from_numpy(np.asfortranarray(T)).cuda(), nb=nb)
    torch.cuda.synchronize()
    Zo, eo = oracle.trevc(T, nb=nb)
    rel, de = aligned_diff(Z.cpu().numpy(), e.cpu().numpy(), Zo, eo)
    res = {{"max_rel": float(rel.max()), "max_de": int(de.max()), "rescaled": int((eo < 0).sum())}}
else:
    cp = case == "solve_c"
    m, n = 333, 130
    rng = np.random.default_rng(5)
    U = np.triu(rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cp else 0)) / np.sqrt(m)
    U[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m)
    U = np.asfortranarray(U)
    s = inputs.random_shifts(n, cp, 6, radius=0.5)
    B = inputs.random_rhs(m, n, cp, 7)
    worst, wde = 0.0, 0
    for op in ("N", "C"):
        X, sc, e = ms.solve(torch.from_numpy(U).cuda(), torch.from_numpy(np.ascontiguousarray(s)).cuda(),
                            torch.from_numpy(np.asfortranarray(B)).cuda(), safe=True, op=op, nb=64)
        torch.cuda.synchronize()
        Xo, eo = oracle.mstrsm(U, s, B, safe=True, op=op, nb=64)
        rel, de = aligned_diff(X.cpu().numpy(), e.cpu().numpy(), Xo, eo)
        worst, wde = max(worst, float(rel.max())), max(wde, int(de.max()))
    res = {{"max_rel": worst, "max_de": wde, "rescaled": 1}}
print(json.dumps(res))
"""


@pytest.mark.parametrize("impl", ["tc", "w"])
@pytest.mark.parametrize("case", ["trevc_c", "trevc_r", "solve_c", "solve_r"])
def test_both_diagonal_kernels_match_oracle(impl, case):
    """Both standard-solve diagonal kernels -- the left-looking tensor-pipe one (diag_tc.cuh) and
    the chunked one (diag_fast.cuh) -- whichever the launcher would pick by default, forced by
    MSTRSM_DIAG on real and complex data, op N and op C, n_b = 64 (ragged m)."""
    env = dict(os.environ, MSTRSM_DIAG=impl)
    out = subprocess.run([sys.executable, "-c", _SCRIPT_IMPL.format(root=ROOT, case=case)], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert r["max_de"] <= 1 and r["max_rel"] <= 1e-9 and r["rescaled"] > 0, r
