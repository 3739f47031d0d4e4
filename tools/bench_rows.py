"""Measurement of every §8 workload besides the headline (bench.py times config 5): one JSON line
per workload with device-timed throughput (CUDA events on the library stream, warm-up first),
algorithmic GFLOP/s (R18), units/s, and the per-kind kernel time from the live profile.

    python tools/bench_rows.py [--steps 3] [--warmup 2] [--only c3,c4,...]

Workloads: c1 (dense safe solve, real), c2 (TriangEig real), c3 (TriangEig complex), c4 (inverse
Lanczos pseudospectra, 2 x 15 solves over 16384 points), g1 (GeneralizedTriangEig, complex m=4096,
SURVEY §8f row f1), f2 / f2_bt (TriangEig + X = Q Z and the back-transformation alone, complex
m=8192, row f2).  Inputs are seeded synthetic stand-ins."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def eig_flops(m, cplx, products=1):
    k = np.arange(m, dtype=np.float64)
    return float(np.sum(k * k)) * (4.0 if cplx else 1.0) * products


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--only", default="c1,c2,c3,c4,c4d,g1,f2,f4,trsm,c5s8")
    a = ap.parse_args()
    import torch
    import paper_1607_01477_b200 as ms
    from paper_1607_01477_b200 import inputs
    ms.load()
    dev = lambda x: torch.from_numpy(np.asfortranarray(x)).cuda()
    work = {}
    if "c1" in a.only:
        U, s, B = inputs.c1_plain_real()
        Ud, sd, B0 = dev(U), dev(s), dev(B)
        Bd = B0.clone()
        work["c1"] = (lambda: (Bd.copy_(B0), ms.solve(Ud, sd, Bd, safe=True, nb=32)),
                      256.0 ** 2 * 64, 64, "shifts/s", "c1: safe multi-shift solve, real, m=256, n=64, n_b=32")
    if "c2" in a.only:
        T = dev(inputs.c2_trevc_real())
        work["c2"] = (lambda: ms.trevc(T, nb=64), eig_flops(2048, False), 2048, "eigvecs/s",
                      "c2: TriangEig real, m=2048, n_b=64")
    if "c3" in a.only:
        T3 = dev(inputs.c3_trevc_complex())
        work["c3"] = (lambda: ms.trevc(T3, nb=128), eig_flops(8192, True), 8192, "eigvecs/s",
                      "c3: TriangEig complex, m=8192, n_b=128")
    if "c4" in a.only:
        U4, z, v0 = inputs.c4_pseudospectra()
        U4d, zd, vd = dev(U4), dev(z), dev(v0)
        work["c4"] = (lambda: ms.pseudospectra(U4d, zd, vd, iters=15, nb=64),
                      15 * 2 * 4.0 * 1024 ** 2 * z.shape[0], z.shape[0], "points/s",
                      "c4: inverse-Lanczos pseudospectra, complex m=1024, 128x128 grid, 15 steps (30 solves)")
    if "c4d" in a.only or "c4" in a.only.split(","):
        U4, z, v0 = inputs.c4_pseudospectra()
        U4d, zd, vd = dev(U4), dev(z), dev(v0)
        work["c4d"] = (lambda: ms.spectral_cloud(U4d, zd, vd, maxit=15, tol=1e-10, nb=64),
                       15 * 2 * 4.0 * 1024 ** 2 * z.shape[0], z.shape[0], "points/s",
                       "c4d: c4 with SpectralCloud deflation (tol 1e-10, at most 15 steps; SURVEY §8f f3); "
                       "gflops counts the fixed 15-step work, so it is an effective rate")
    if "c5s8" in a.only:
        # one rank's shard of the 8-GPU c5 step (2048 eigenvectors, serpentine block-cyclic), the
        # solve part of what each rank does at N = 8 (the collectives are the driver's to measure)
        from paper_1607_01477_b200 import dist as pdist
        T5 = dev(inputs.c5_grcar_like())
        cols8 = pdist.shard_cols(16384, 8, 0, 16)
        work["c5s8"] = (lambda: ms.trevc(T5, nb=128, cols=cols8), eig_flops(16384, True) / 8, len(cols8),
                        "eigvecs/s", "c5s8: rank 0's shard of the 8-GPU c5 step (2048 eigenvectors), solve only")
    if "trsm" in a.only:
        # SURVEY §8d.5 paper analogue (context only): the multi-shift solve at zero shift against
        # cuBLAS trsm (torch.linalg.solve_triangular) on the same upper-triangular system
        for mt, cx in ((256, False), (4096, True)):
            rng = np.random.default_rng(77)
            Ut = np.triu(rng.standard_normal((mt, mt)) + (1j * rng.standard_normal((mt, mt)) if cx else 0)) / np.sqrt(mt)
            Ut[np.arange(mt), np.arange(mt)] = rng.uniform(1.0, 2.0, mt)
            nt = 64 if mt == 256 else mt
            Bt0 = dev(inputs.random_rhs(mt, nt, cx, 78))
            Utd = dev(Ut)
            zt = dev(np.zeros(nt, dtype=np.complex128 if cx else np.float64))
            Btw = Bt0.clone()
            nbt = 32 if mt == 256 else 128
            fl = (4.0 if cx else 1.0) * mt * mt * nt
            tag = f"{'z' if cx else 'd'}{mt}"
            work[f"trsm_ours_{tag}"] = (lambda U_=Utd, z_=zt, B0=Bt0, Bw=Btw, nb_=nbt: (Bw.copy_(B0),
                                        ms.solve(U_, z_, Bw, safe=False, nb=nb_)), fl, nt, "rhs/s",
                                        f"multi-shift solve at zero shift (plain), {tag}, n={nt}")
            work[f"trsm_cublas_{tag}"] = (lambda U_=Utd, B0=Bt0: torch.linalg.solve_triangular(U_, B0, upper=True),
                                          fl, nt, "rhs/s", f"cuBLAS trsm (torch.linalg.solve_triangular), {tag}, n={nt}")
    if "f4" in a.only:
        m4 = 4096
        rng = np.random.default_rng(44)
        A4 = np.tril(rng.standard_normal((m4, m4)) + 1j * rng.standard_normal((m4, m4))) / np.sqrt(m4)
        A4[np.arange(m4), np.arange(m4)] = rng.uniform(1.0, 2.0, m4)
        A4d = dev(A4)
        s4 = dev(inputs.random_shifts(m4, True, 45, radius=0.5))
        B40 = dev(np.asfortranarray(inputs.random_rhs(m4, m4, True, 46).T))
        B4 = B40.clone()
        work["f4"] = (lambda: (B4.copy_(B40), ms.solve_side(A4d, s4, B4, side="R", uplo="L", safe=True, nb=128)),
                      4.0 * m4 * m4 * m4, m4, "shifts/s",
                      "f4: right-side lower-triangular safe solve x^T (L - s I) = c b^T, complex m=n=4096, n_b=128 "
                      "(transforms + op N solve; SURVEY §8f f4)")
        U4u = dev(np.asfortranarray(A4.T))
        B4u0 = dev(inputs.random_rhs(m4, m4, True, 46))
        B4u = B4u0.clone()
        work["f4_ref"] = (lambda: (B4u.copy_(B4u0), ms.solve(U4u, s4, B4u, safe=True, nb=128)),
                          4.0 * m4 * m4 * m4, m4, "shifts/s",
                          "f4_ref: the same system as a left-upper solve on L^T (no transforms), complex m=n=4096")
    if "g1" in a.only:
        Tg, Sg = inputs.g1_pencil(m=4096)
        Tgd, Sgd = dev(Tg), dev(Sg)
        work["g1"] = (lambda: ms.tgevc(Tgd, Sgd, nb=64), eig_flops(4096, True, products=2), 4096,
                      "eigvecs/s", "g1: GeneralizedTriangEig complex pencil, m=4096, n_b=64 (SURVEY §8f f1)")
    if "f2" in a.only:
        mq = 8192
        Tq = dev(inputs.c3_trevc_complex(mq))
        Qq = dev(inputs.dense_q(mq, True))
        Zq, _, _ = ms.trevc(Tq, nb=128)
        bt_flops = 8.0 * mq * mq * (mq + 1) / 2.0          # X = Q Z, Z upper triangular (complex x4)
        work["f2_bt"] = (lambda: ms.eig_backtransform(Qq, Zq), bt_flops, mq, "eigvecs/s",
                         "f2: back-transformation X = Q Z alone, complex m=8192 (SURVEY §8f f2)")
        work["f2"] = (lambda: ms.trevc_qz(Tq, Qq, nb=128), eig_flops(mq, True) + bt_flops, mq, "eigvecs/s",
                      "f2: TriangEig + back-transformation (Eig's last two steps), complex m=8192, n_b=128")
    if "graph" in a.only:
        # the same c1 / c2 calls captured once into a CUDA graph and replayed (launch overhead and
        # inter-kernel gaps on the device side; the library's launches are stream-capturable)
        for nm in ("c1", "c2"):
            if nm not in work:
                continue
            fn0, flops0, units0, uname0, desc0 = work[nm]
            for _ in range(2):
                fn0()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            s_cap = torch.cuda.Stream()
            s_cap.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s_cap):
                with torch.cuda.graph(g, stream=s_cap):
                    fn0()
            torch.cuda.current_stream().wait_stream(s_cap)
            torch.cuda.synchronize()
            work[nm + "_graph"] = (lambda g_=g: g_.replay(), flops0, units0, uname0, desc0 + " (CUDA graph replay)")
    for name, (fn, flops, units, uname, desc) in work.items():
        for _ in range(a.warmup):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        t0 = time.perf_counter()
        for _ in range(a.steps):
            fn()
        t_host = (time.perf_counter() - t0) * 1e3 / a.steps    # host time to enqueue one step
        e1.record()
        torch.cuda.synchronize()
        ms_step = e0.elapsed_time(e1) / a.steps
        ms.mstrsm_profile(1)                     # one more step for the per-kind breakdown
        fn()
        torch.cuda.synchronize()
        gm, gn, _ = ms.mstrsm_profile_read(0)
        dm, dn, _ = ms.mstrsm_profile_read(1)
        ms.mstrsm_profile(0)
        print(json.dumps({"workload": desc, "config": name, "ms_per_step": ms_step,
                          "gflops_algorithmic": flops / (ms_step * 1e-3) / 1e9,
                          uname: units / (ms_step * 1e-3), "steps": a.steps, "warmup": a.warmup,
                          "gemm_ms_profiled_step": gm, "diag_ms_profiled_step": dm,
                          "host_enqueue_ms_per_step": t_host,
                          "timing": "CUDA events around the timed steps (no per-launch events); the "
                                    "per-kind split comes from one extra step with per-launch events; "
                                    "host_enqueue_ms_per_step = wall time of the host calls alone (below "
                                    "ms_per_step: the host stays ahead, launch overhead is hidden)"}),
              flush=True)


if __name__ == "__main__":
    main()
