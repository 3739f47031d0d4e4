"""Phase timing of the diagonal kernels (experiment build exp/phase/libmstrsm.so, MSTRSM_PHASE_TIMES):
per launch, the median over CTAs of each phase's clock64 delta (µs at the SM clock), CTA spread
and the launch's globaltimer span.  Usage: MSTRSM_LIB=exp/phase/libmstrsm.so python tools/exp_phase.py c5s8|c2|c4|c5"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import dist, inputs
ms.load()
from paper_1607_01477_b200 import _binding as B
lib = B._lib if hasattr(B, "_lib") else B.lib()
cfg = sys.argv[1]
if cfg in ("c5s8", "c5", "c3"):
    m = 16384 if cfg != "c3" else 8192
    T = torch.from_numpy(inputs.c5_grcar_like(m) if cfg != "c3" else inputs.c3_trevc_complex()).cuda()
    cols = dist.shard_cols(m, 8, 0, 16) if cfg == "c5s8" else None
    run = lambda: ms.trevc(T, nb=128, cols=cols) if cols is not None else ms.trevc(T, nb=128)
elif cfg == "c2":
    T = torch.from_numpy(inputs.c2_trevc_real()).cuda()
    run = lambda: ms.trevc(T, nb=64)
else:
    U, z, v0 = inputs.c4_pseudospectra()
    Ud, zd, vd = (torch.from_numpy(x).cuda() for x in (U, z, v0))
    run = lambda: ms.pseudospectra(Ud, zd, vd, iters=1, nb=64)
clk = float(os.environ.get("SM_MHZ", "1965"))
run(); torch.cuda.synchronize()
buf = np.zeros(512 * 256 * 16, dtype=np.int64)
f = lib.mstrsm_phase_read
f.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
f(buf.ctypes.data, 0, 1)
run(); torch.cuda.synchronize()
n = f(buf.ctypes.data, 512, 0)
P = buf.reshape(512, 256, 16)[:min(n, 512)]
names = {2: "prologue", 3: "load y", 4: "precheck", 5: "stage wait", 6: "rows", 7: "done wait", 8: "finish", 9: "to end"}
print("launches", n)
tot = {}
for li in range(P.shape[0]):
    R = P[li]
    act = R[:, 1] != 0
    if not act.any(): continue
    R = R[act]
    span = (R[:, 15].max() - R[:, 0].min()) / 1e3
    row = {"launch": li, "ctas": int(act.sum()), "span_us": round(span, 2)}
    prev = 1
    for k in range(2, 10):
        v = R[:, k]; ok = v != 0
        if not ok.any(): continue
        d = (v[ok] - R[ok, prev]) / clk
        row[names[k]] = round(float(np.median(d)), 2)
        tot[names[k]] = tot.get(names[k], 0.0) + float(np.median(d))
        prev = k
    rep = (R[:, 11] - R[:, 10]) / clk
    row["replay"] = round(float(np.median(rep[R[:, 11] != 0])) if (R[:, 11] != 0).any() else 0, 2)
    tot["span"] = tot.get("span", 0.0) + span
    if li % max(1, P.shape[0] // 12) == 0: print(row)
print("sum over launches (us):", {k: round(v, 1) for k, v in tot.items()})
