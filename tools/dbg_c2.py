"""Debug: c2 trevc GPU vs oracle, per-column exponent differences (prints worst columns)."""
import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
ms.load()
m = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
nb = int(sys.argv[2]) if len(sys.argv) > 2 else 64
T = inputs.c2_trevc_real(m=m)
Z, sc, e = ms.trevc(torch.from_numpy(T).cuda(), nb=nb)
torch.cuda.synchronize()
e = e.cpu().numpy().astype(int)
Zo, eo = oracle.trevc(T, nb=nb)
de = np.abs(e - eo)
bad = np.nonzero(de > 1)[0]
print("max de", de.max(), "n bad", len(bad), "first bad", bad[:10], flush=True)
for j in bad[:5]:
    print(j, e[j], eo[j])
