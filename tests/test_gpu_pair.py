"""GPU tests (-m gpu) of the paired-block update (blocked_solve in csrc/mstrsm.cu, pair_fix in
csrc/diag_kernel.cuh): the update of the rows beyond two consecutive blocks as one
GEMM with K = 2 n_b, the first block's rows rescaled in place when the second rescales.  By
default only complex solves with n_b <= 64 pair; MSTRSM_PAIR=2 forces pairs everywhere and
MSTRSM_PAIR=0 turns them off, so both ways are checked against the oracle (R20/R21) on real and
complex data, op N and op C, with row ends, heavy rescaling and ragged last blocks.  The switch is
read when the library loads, hence a subprocess per setting."""
import json
import os
import subprocess
import sys

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
res = {{}}
def put(name, X, e, Xo, eo):
    rel, de = aligned_diff(X, e, Xo, eo)
    res[name] = [float(rel.max()), int(de.max()), bool(np.isfinite(X).all()), int((eo < 0).sum())]
# TriangEig: heavy rescaling (c5 shape, ragged top block), real (c2 shape), complex n_b = 64 (c4 n_b)
for name, T, nb in (("trevc_c5", inputs.c5_grcar_like(1100), 128), ("trevc_c2", inputs.c2_trevc_real(700), 64),
                    ("trevc_c3", inputs.c3_trevc_complex(1000), 64)):
    Z, sc, e = ms.trevc(torch.from_numpy(np.asfortranarray(T)).cuda(), nb=nb)
    torch.cuda.synchronize()
    Zo, eo = oracle.trevc(T, nb=nb)
    put(name, Z.cpu().numpy(), e.cpu().numpy(), Zo, eo)
    if name == "trevc_c5":   # column subsets (multi-GPU shards) reproduce the full run bit for bit
        Zf, ef = Z.cpu().numpy(), e.cpu().numpy()
        ok = True
        for P, r in ((2, 1), (8, 5)):
            cols = [k for k in range(1100) if (k // 16) % P == r]
            Zs, _, es = ms.trevc(torch.from_numpy(np.asfortranarray(T)).cuda(), nb=nb, cols=cols)
            torch.cuda.synchronize()
            ok = ok and np.array_equal(Zs.cpu().numpy(), Zf[:, cols]) and np.array_equal(es.cpu().numpy(), ef[cols])
        res["subset_bit_identical"] = bool(ok)
# dense right-hand sides, op N (with unsorted row ends) and op C, real and complex, ragged m
for cp in (False, True):
    m, n, nb = 333, 130, 32
    rng = np.random.default_rng(11)
    U = np.triu(rng.standard_normal((m, m)) + (1j * rng.standard_normal((m, m)) if cp else 0)) / np.sqrt(m)
    U[np.arange(m), np.arange(m)] = rng.uniform(0.02, 2, m)
    U = np.asfortranarray(U)
    s = inputs.random_shifts(n, cp, 6, radius=0.8)
    B = inputs.random_rhs(m, n, cp, 7)
    r = rng.integers(0, m + 1, n)
    for op, re_ in (("N", None), ("N", r), ("C", None)):
        X, sc, e = ms.solve(torch.from_numpy(U).cuda(), torch.from_numpy(np.ascontiguousarray(s)).cuda(),
                            torch.from_numpy(np.asfortranarray(B)).cuda(), safe=True, op=op, nb=nb, row_end=re_)
        torch.cuda.synchronize()
        Xo, eo = oracle.mstrsm(U, s, B, safe=True, op=op, nb=nb, row_end=re_)
        put(f"solve_{{'z' if cp else 'd'}}{{op}}{{'_re' if re_ is not None else ''}}", X.cpu().numpy(),
            e.cpu().numpy(), Xo, eo)
print(json.dumps(res))
"""


@pytest.mark.parametrize("mode", ["2", "0"])
def test_paired_and_single_blocks_match_oracle(mode):
    env = dict(os.environ, MSTRSM_PAIR=mode)
    out = subprocess.run([sys.executable, "-c", _SCRIPT.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res.pop("subset_bit_identical"), res
    for name, (rel, de, finite, _rescaled) in res.items():
        assert finite and de <= 1 and rel <= 1e-9, (name, res[name])
    assert res["trevc_c5"][3] > 0                                   # rescaling exercised


def test_odd_block_size_is_never_paired():
    """Odd n_b (the X+ plane cannot hold a pair contiguously and aligned) runs single blocks even
    under MSTRSM_PAIR=2: a complex op N / op C solve at n_b = 7 matches the oracle."""
    script = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import oracle
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
from tests.gpu_util import aligned_diff
m, n, nb = 200, 50, 7
rng = np.random.default_rng(3)
U = np.asfortranarray(np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m))
U[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m)
s = inputs.random_shifts(n, True, 4, radius=0.4)
B = inputs.random_rhs(m, n, True, 5)
worst = 0.0
for op in ("N", "C"):
    for safe in (False, True):
        X, sc, e = ms.solve(torch.from_numpy(U).cuda(), torch.from_numpy(np.ascontiguousarray(s)).cuda(),
                            torch.from_numpy(np.asfortranarray(B)).cuda(), safe=safe, op=op, nb=nb)
        torch.cuda.synchronize()
        Xo, eo = oracle.mstrsm(U, s, B, safe=safe, op=op, nb=nb)
        rel, de = aligned_diff(X.cpu().numpy(), e.cpu().numpy(), Xo, eo)
        worst = max(worst, float(rel.max()) + float(de.max()))
print(json.dumps({{"worst": worst}}))
"""
    env = dict(os.environ, MSTRSM_PAIR="2")
    out = subprocess.run([sys.executable, "-c", script.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1])["worst"] <= 1e-9


def test_adversarial_suite_with_paired_blocks():
    """S:228 safety properties (finite, e <= 0, ||x|| < Omega, c in [0,1], backward error <=
    64 m 2^-53) on the adversarial suite (Jordan blocks, exact zero pivots, graded 10^+-300,
    repeated eigenvalues, tiny pivots with strong coupling) with paired blocks forced
    (MSTRSM_PAIR=2, even n_b), real and complex (the suite's matrices rotated by a unit phase)."""
    script = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, {root!r})
import paper_1607_01477_b200 as ms
from tests.test_oracle_pins import _adversarial_suite
from tests import refmath as R
worst, bad = 0.0, []
for i, (U, s, B, nb) in enumerate(_adversarial_suite()):
    nb = 2 * ((nb + 1) // 2)                                 # even: paired
    for cp in (False, True):
        Uc, sc_, Bc = (U, s, B) if not cp else (U * np.exp(0.3j), s * np.exp(0.3j), B * (1 + 0.5j))
        m = Uc.shape[0]
        X, sc, e = ms.solve(torch.from_numpy(np.asfortranarray(Uc)).cuda(),
                            torch.from_numpy(np.ascontiguousarray(sc_)).cuda(),
                            torch.from_numpy(np.asfortranarray(Bc)).cuda(), safe=True, nb=nb)
        torch.cuda.synchronize()
        X, sc, e = X.cpu().numpy(), sc.cpu().numpy(), e.cpu().numpy()
        ok = np.all(np.isfinite(X)) and np.all(e <= 0) and np.max(np.abs(X)) < R.OMEGA and np.all((sc >= 0) & (sc <= 1))
        unorm = np.max(np.sum(np.abs(np.triu(Uc)), axis=1))
        delta = np.ldexp(unorm, -52) if unorm > 0 else np.finfo(float).tiny
        for j in range(len(sc_)):
            dd = np.diag(Uc) - sc_[j]
            if np.any((dd == 0) & (delta + sc_[j] - sc_[j] != delta)):
                continue
            Ud = np.triu(Uc).copy()
            Ud[np.arange(m), np.arange(m)] = np.where(dd == 0, delta + sc_[j], np.diag(Uc))
            rr = float(R.residual_ratio(Ud, sc_[j], X[:, j], e[j], Bc[:, j]))
            worst = max(worst, rr / (64 * m * 2.0 ** -53))
        if not ok:
            bad.append((i, cp))
print(json.dumps({{"worst": worst, "bad": bad}}))
"""
    env = dict(os.environ, MSTRSM_PAIR="2")
    out = subprocess.run([sys.executable, "-c", script.format(root=ROOT)], env=env, capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    r = json.loads(out.stdout.strip().splitlines()[-1])
    assert not r["bad"] and r["worst"] <= 1.0, r
