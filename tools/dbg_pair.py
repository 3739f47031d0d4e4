"""Debug: trevc with paired blocks vs the oracle (run under MSTRSM_PAIR=0/1, MSTRSM_GEMM=...)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
import oracle  # noqa

for cplx in (True, False):
    for m, nb in ((100, 32), (128, 32), (96, 32), (200, 64)):
        T = inputs.c3_trevc_complex(m) if cplx else inputs.c2_trevc_real(m)
        Td = torch.from_numpy(T).cuda()
        Z, sc, e = ms.trevc(Td, nb=nb)
        torch.cuda.synchronize()
        Zg, eg = Z.cpu().numpy(), e.cpu().numpy()
        Zo, eo = oracle.trevc(T, nb=nb)
        nrm = np.maximum(np.abs(Zo).max(axis=0), 1e-300)
        rel = np.abs(Zg - Zo).max(axis=0) / nrm
        bad = np.where(rel > 1e-9)[0]
        print(f"cplx={cplx} m={m} nb={nb}: max rel {rel.max():.2e}, bad cols {len(bad)} {bad[:12]}, de {np.abs(eg - eo).max()}")
        if len(bad):
            j = bad[0]
            rows = np.where(np.abs(Zg[:, j] - Zo[:, j]) > 1e-9 * nrm[j])[0]
            print("   col", j, "bad rows", rows[:20], "...", rows[-5:])
