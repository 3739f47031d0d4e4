import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_1607_01477_b200 as ms
from paper_1607_01477_b200 import inputs
ms.load()
m = int(sys.argv[1]); nb = int(sys.argv[2]); cplx = sys.argv[3] == 'z'
T = inputs.c5_grcar_like(m=m) if cplx else inputs.c2_trevc_real(m=m)
Td = torch.from_numpy(T).cuda()
t0 = time.time()
Z, sc, e = ms.trevc(Td, nb=nb)
torch.cuda.synchronize()
print("ok", m, nb, cplx, time.time() - t0, int(e.min()), flush=True)
