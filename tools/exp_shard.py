"""Experiment: one rank's TriangEig shard (serpentine block-cyclic, P ranks) at m = 16384, with the
library named by MSTRSM_LIB -- the per-rank solve time of the multi-GPU step."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs, dist
ms.load()
m, P = 16384, int(sys.argv[1]) if len(sys.argv) > 1 else 8
T = torch.from_numpy(inputs.c5_grcar_like(m)).cuda()
for r in (0, P - 1):
    cols = dist.shard_cols(m, P, r, 16)
    for _ in range(2):
        ms.trevc(T, nb=128, cols=cols)
    torch.cuda.synchronize()
    ms.mstrsm_profile(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); ms.trevc(T, nb=128, cols=cols); e1.record(); torch.cuda.synchronize()
    g = ms.mstrsm_profile_read(0); d = ms.mstrsm_profile_read(1); ms.mstrsm_profile(0)
    print(json.dumps({"lib": os.environ.get("MSTRSM_LIB", "default"), "P": P, "rank": r, "ncols": len(cols),
                      "ms": e0.elapsed_time(e1), "gemm_ms": g[0], "diag_ms": d[0]}), flush=True)
