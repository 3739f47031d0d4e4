"""One warm-up solve + one profiled solve (cudaProfilerStart/Stop brackets the second), for
`ncu --profile-from-start off`.  Usage: python tools/profile_run.py --config c5|c3|c4|c2|c5s8|c1"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_1607_01477_b200 as ms  # noqa: E402
from paper_1607_01477_b200 import dist, inputs  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5")
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--iters", type=int, default=15)
    a = ap.parse_args()
    ms.load()
    if a.config in ("c5", "c3"):
        gen = inputs.c5_grcar_like if a.config == "c5" else inputs.c3_trevc_complex
        T = gen(m=a.m) if a.m else gen()
        Td = torch.from_numpy(T).cuda()
        run = lambda: ms.trevc(Td, nb=128)
    elif a.config == "c5s8":                       # rank 0's shard of the 8-GPU c5 step
        m = a.m or 16384
        Td = torch.from_numpy(inputs.c5_grcar_like(m)).cuda()
        cols = dist.shard_cols(m, 8, 0, 16)
        run = lambda: ms.trevc(Td, nb=128, cols=cols)
    elif a.config == "c2":
        Td = torch.from_numpy(inputs.c2_trevc_real()).cuda()
        run = lambda: ms.trevc(Td, nb=64)
    elif a.config == "c1":
        U, s, B = inputs.c1_plain_real()
        Ud, sd, B0 = (torch.from_numpy(x).cuda() for x in (U, s, B))
        Bd = B0.clone()
        run = lambda: (Bd.copy_(B0), ms.solve(Ud, sd, Bd, safe=True, nb=32))
    else:
        U, z, v0 = inputs.c4_pseudospectra(m=a.m or 1024)
        Ud, zd, vd = (torch.from_numpy(x).cuda() for x in (U, z, v0))
        run = lambda: ms.pseudospectra(Ud, zd, vd, iters=a.iters, nb=64)
    run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    run()
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("profile_run done")


if __name__ == "__main__":
    main()
