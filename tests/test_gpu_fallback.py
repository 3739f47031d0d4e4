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
