import json, sys, os
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
m, nb = 1100, 128
T = torch.from_numpy(np.asfortranarray(inputs.c5_grcar_like(m))).cuda()
ms.comm_init(1, 0)
Z1, s1, e1 = ms.trevc_dist(T, m, nb=nb)
ms.comm_destroy()
Z2, s2, e2 = ms.trevc(T, nb=nb)
torch.cuda.synchronize()
Z1, Z2 = Z1.cpu().numpy(), Z2.cpu().numpy()
d = Z1 != Z2
cols = np.where(d.any(axis=0))[0]
print("bad cols", len(cols), cols[:20])
for j in cols[:4]:
    rows = np.where(d[:, j])[0]
    r = rows[0]
    print("col", j, "rows", rows[:10], "...", rows[-3:], "n", len(rows), "Z1", Z1[r, j], "Z2", Z2[r, j], "ratio", Z1[r, j] / Z2[r, j] if Z2[r, j] != 0 else None)
rb = np.where(d.any(axis=1))[0]
print("bad rows blocks", sorted(set(((m - 1 - rb) // nb).tolist())))
