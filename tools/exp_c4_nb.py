"""c4 (inverse-Lanczos pseudospectra, m = 1024, 16384 shifts, 15 steps) against the block size
n_b: the diagonal solves cost O(m n_b n) and run latency-bound, the update GEMM O(m^2 n) at the
DMMA rate, so n_b trades one against the other.  Usage: python tools/exp_c4_nb.py [nb ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1607_01477_b200 as ms  # noqa: E402
from paper_1607_01477_b200 import inputs  # noqa: E402


def main():
    U, z, v0 = inputs.c4_pseudospectra()
    Ud, zd, vd = (torch.from_numpy(x).cuda() for x in (U, z, v0))
    for nb in [int(v) for v in sys.argv[1:]] or [32, 48, 64, 96, 128]:
        run = lambda: ms.pseudospectra(Ud, zd, vd, iters=15, nb=nb)
        out = run()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            out = run()
        e1.record()
        torch.cuda.synchronize()
        s = out[0] if isinstance(out, tuple) else out
        print(f"nb={nb} ms={e0.elapsed_time(e1) / 3:.2f} smin[0:3]={s.flatten()[:3].tolist()}", flush=True)


if __name__ == "__main__":
    main()
