"""Small hot-path workload for compute-sanitizer (one tool per gpurun call, after a plain run):
a c1-shaped safe solve (op N and op C, real), a c2-shaped TriangEig (real, n_b = 64, the
left-looking tensor-pipe diagonal kernel), a complex m = 1100 TriangEig (n_b = 128, chunked
diagonal kernel with replay warps, look-ahead side stream, 3M update GEMM), a complex op C solve
with the chunked kernel forced onto n_b = 64 columns, and the generalized solve."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1607_01477_b200 as ms  # noqa: E402
from paper_1607_01477_b200 import inputs  # noqa: E402


def main():
    ms.load()
    dev = lambda a: torch.from_numpy(np.asfortranarray(a)).cuda()
    U, s, B = inputs.c1_plain_real()
    for op in ("N", "C"):
        ms.solve(dev(U), dev(np.ascontiguousarray(s)), dev(B), safe=True, op=op, nb=32)
    ms.trevc(dev(inputs.c2_trevc_real(512)), nb=64)
    ms.trevc(dev(inputs.c5_grcar_like(1100)), nb=128)
    m, n = 300, 96
    rng = np.random.default_rng(3)
    Uc = np.triu(rng.standard_normal((m, m)) + 1j * rng.standard_normal((m, m))) / np.sqrt(m)
    Uc[np.arange(m), np.arange(m)] = rng.uniform(1, 2, m)
    sc = inputs.random_shifts(n, True, 4, radius=0.5)
    Bc = inputs.random_rhs(m, n, True, 5)
    ms.solve(dev(Uc), dev(np.ascontiguousarray(sc)), dev(Bc), safe=True, op="C", nb=64)
    V = np.triu(rng.standard_normal((m, m))) / np.sqrt(m) + np.eye(m)
    ms.solve_gen(dev(Uc), dev(V.astype(complex)), dev(np.ascontiguousarray(sc)), dev(Bc), safe=True, nb=64)
    torch.cuda.synchronize()
    print("sanitize_run done")


if __name__ == "__main__":
    main()
