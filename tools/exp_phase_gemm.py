"""Phase timing of the update GEMM (gemm_ws3q_kernel; experiment build exp/phase/libmstrsm.so):
per launch, medians over CTAs (µs): pdl wait, first operands of group 0 after the wait, group 0's
first tile (mainloop, epilogue), groups 1/2 first operands, each group's end after the wait, the
spread of CTA ends, and the launch span (first CTA entry to last group end, %globaltimer).
Usage: MSTRSM_LIB=exp/phase/libmstrsm.so python tools/exp_phase_gemm.py c5s8|c5|c4|c3"""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import dist, inputs
ms.load()
from paper_1607_01477_b200 import _binding as B
lib = B._lib
cfg = sys.argv[1]
if cfg in ("c5s8", "c5", "c3"):
    m = 16384 if cfg != "c3" else 8192
    T = torch.from_numpy(inputs.c5_grcar_like(m) if cfg != "c3" else inputs.c3_trevc_complex()).cuda()
    cols = dist.shard_cols(m, 8, 0, 16) if cfg == "c5s8" else None
    run = lambda: ms.trevc(T, nb=128, cols=cols) if cols is not None else ms.trevc(T, nb=128)
else:
    U, z, v0 = inputs.c4_pseudospectra()
    Ud, zd, vd = (torch.from_numpy(x).cuda() for x in (U, z, v0))
    run = lambda: ms.pseudospectra(Ud, zd, vd, iters=1, nb=64)
clk = float(os.environ.get("SM_MHZ", "1965"))
f = lib.mstrsm_phase_read2
f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int]
buf = np.zeros(512 * 256 * 16, dtype=np.int64)
run(); torch.cuda.synchronize()
f(1, buf.ctypes.data, 0, 1)
run(); torch.cuda.synchronize()
n = f(1, buf.ctypes.data, 512, 0)
P = buf.reshape(512, 256, 16)[:min(n, 512)]
print("gemm launches", n)
acc = {}
for li in range(P.shape[0]):
    R = P[li]
    R = R[R[:, 1] != 0]
    if len(R) == 0: continue
    med = lambda a, b: float(np.median((R[:, a] - R[:, b])[(R[:, a] != 0)])) / clk if (R[:, a] != 0).any() else float("nan")
    ends = R[:, 12:15].astype(float); ends[ends == 0] = np.nan
    cta_end = np.nanmax(ends, axis=1)
    row = {"launch": li, "ctas": len(R), "pdl_wait": med(2, 1), "first_ops": med(3, 2), "tile0_main": med(4, 3),
           "tile0_epi": med(5, 4), "g1_first": med(6, 2), "g2_first": med(7, 2),
           "g0_end": med(8, 2), "g1_end": med(9, 2), "g2_end": med(10, 2),
           "cta_end_spread": float(np.nanmax(cta_end) - np.nanmin(cta_end)) / 1e3,
           "span": float(np.nanmax(cta_end) - R[:, 0].min()) / 1e3}
    for k, v in row.items():
        if k not in ("launch", "ctas") and v == v: acc[k] = acc.get(k, 0.0) + v
    if li % max(1, P.shape[0] // 10) == 0: print({k: (round(v, 2) if isinstance(v, float) else v) for k, v in row.items()})
print("sums (us):", {k: round(v, 1) for k, v in acc.items()})
