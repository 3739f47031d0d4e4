#!/usr/bin/env python
"""Benchmark: the blocked safe multi-shift triangular solve of arXiv 1607.01477 on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl cuda|reference] [--config c5]

Workload (BASELINE.json config 5, the config the metric's 1/2/4/8-GPU scaling is quoted on):
triangular eigenvectors of an m = 16384 complex Grcar-like upper-triangular T (all 16384 shifts
taken from diag(T), RHS -T(1:k-1,k), safe solve with n_b = 128; TriangEig, Alg. 6).  One step =
one whole pass of the hot path: a.1 init, a.2 norm pass, the 128 blocked steps (a.3 diagonal
solve + a.4 bound + a.5 DMMA update GEMM), a.6 finalize.  Inputs are resident in HBM when the
timed region starts; T (4.3 GB) and Z are far larger than the 126 MB L2, so no flush is needed.

N > 1 (torchrun, one process per GPU, NCCL): shifts/columns are sharded block-cyclically (groups
of 16 columns); a step is NCCL broadcast of T from rank 0 + the local solve + NCCL all-gather of
the local eigenvectors (the only collectives, BASELINE north star).  Strong scaling (fixed
problem).  Timing: CUDA events on the launching stream, barrier + synchronize on both sides,
max over ranks.

Flop convention (R18): the paper's "~m^2 flops" per triangular solve,
complex x4, applied to the rows the eigen shortcut actually solves: eigenvector k (0-based) is a
k x k solve -> k^2 (real) / 4 k^2 (complex) flops; c5 total = 4 sum_k k^2 = 5.86e12.  BASELINE's
nominal m^2 n figure (3x larger for the eigen shortcut) is printed as gflops_nominal_m2n.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "multi-shift TRSM fp64 GFLOP/s & % FP64 TC peak at 1/2/4/8 GPU; eigvecs/s"

CONFIGS = {
    # name: (m, nb, generator, complex)
    "c5": dict(m=16384, nb=128, gen="c5_grcar_like", cplx=True,
               workload="c5: TriangEig (safe multi-shift, eigen shortcut), complex fp64 Grcar-like T, "
                        "m=n=16384, n_b=128 (BASELINE config 5)"),
    "c3": dict(m=8192, nb=128, gen="c3_trevc_complex", cplx=True,
               workload="c3: TriangEig complex fp64, m=n=8192, n_b=128 (BASELINE config 3)"),
    "c2": dict(m=2048, nb=64, gen="c2_trevc_real", cplx=False,
               workload="c2: TriangEig real fp64, m=n=2048, n_b=64 (BASELINE config 2)"),
}


def algorithmic_flops_cols(cols, cplx: bool) -> float:
    """Eigen shortcut (R11/R18): column k (0-based) is a k x k shifted triangular solve:
    k^2 flops real, 4 k^2 complex (the paper's m^2 convention on the active rows)."""
    k = np.asarray(cols, dtype=np.float64)
    return float(np.sum(k * k)) * (4.0 if cplx else 1.0)


def nominal_flops(m: int, n: int, cplx: bool) -> float:
    return float(m) * m * n * (4.0 if cplx else 1.0)


# ----------------------------------------------------------------------------- clocks sampler
class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region (B200_PROFILING.md)."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([v.strip() for v in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        pw = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "power_w_max": max(pw) if pw else None, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def generate(cfgname: str):
    from paper_1607_01477_b200 import inputs
    c = CONFIGS[cfgname]
    return getattr(inputs, c["gen"])(m=c["m"])


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def ncu_traffic(kernel: str = "gemm_ws_kernel"):
    """dram bytes per launch of the GEMM from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_gemm_traffic.json")
    try:
        d = json.load(open(p))
        return d.get("dram_bytes_per_launch"), d
    except Exception:
        return None, None


# ----------------------------------------------------------------------------- CPU baseline
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cublas_fp64_ceiling(n: int = 8192):
    """SURVEY §8d.5's third peak figure: cuBLAS DGEMM / ZGEMM via torch.matmul at n^3, best of 3
    (context for the roofline; the denominator stays the DMMA microbenchmark)."""
    import torch
    out = {}
    for name, dt, fl in (("dgemm", torch.float64, 2.0), ("zgemm", torch.complex128, 8.0)):
        a = torch.randn(n, n, dtype=dt, device="cuda")
        b = torch.randn(n, n, dtype=dt, device="cuda")
        torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e30
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            torch.matmul(a, b)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[name + "_tflops"] = fl * n ** 3 / (best * 1e-3) / 1e12
        del a, b
    torch.cuda.empty_cache()
    out["note"] = f"torch.matmul {n}^3 (cuBLAS), best of 3; zgemm counted at 8 n^3 (4 real products)"
    return out


def cpu_baseline(T: np.ndarray, cfg: dict, budget_s: float = 15.0):
    """The oracle, as it stands, on a bounded sample of the same workload's columns (the oracle
    is never tuned for this).  Columns are independent, so the sample is exact per column."""
    import oracle
    m, nb, cplx = cfg["m"], cfg["nb"], cfg["cplx"]
    threads = oracle.default_threads()
    # probe the rate on a small sample, then size the timed sample to ~budget_s
    probe = np.linspace(m // 8, m // 4, 4).astype(np.int64)
    t0 = time.perf_counter()
    oracle.trevc(T, nb=nb, cols=probe, nthreads=threads)
    tp = time.perf_counter() - t0
    rate = algorithmic_flops_cols(probe, cplx) / max(tp, 1e-6)     # flops/s, rough
    target = rate * budget_s
    # evenly spread columns (a weighted sample of the whole triangle), at least 8 per thread so
    # that the oracle's dynamic column queue keeps every core busy (the heaviest column is a small
    # part of one thread's share) -- the rate is then the host's, not one column's
    ncol = 8 * threads
    while True:
        cols = np.unique(np.linspace(1, m - 1, ncol).astype(np.int64))
        if algorithmic_flops_cols(cols, cplx) >= target or ncol >= m:
            break
        ncol *= 2
    ncol = max(8 * threads, ncol // 2)
    cols = np.unique(np.linspace(1, m - 1, min(ncol, m - 1)).astype(np.int64))
    t0 = time.perf_counter()
    oracle.trevc(T, nb=nb, cols=cols, nthreads=threads)
    dt = time.perf_counter() - t0
    fl = algorithmic_flops_cols(cols, cplx)
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "per_core_gflops": fl / dt / 1e9 / threads,
            "sample": f"{len(cols)} of {m} eigenvectors (evenly spaced k in [1, {m - 1}], "
                      f"{len(cols) / threads:.0f} per thread, {fl:.3e} algorithmic flops) in {dt:.1f} s",
            "note": "plain C oracle (scalar fp64, no FMA, no BLAS), never tuned; the heavily rescaled "
                    "c5 columns carry subnormal intermediates, which slow it further",
            "eigvecs_per_s_sample": len(cols) / dt, "seconds": dt}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, cfgname):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = CONFIGS[cfgname]
    import oracle
    T = generate(cfgname)
    threads = oracle.default_threads()
    m, nb, cplx = cfg["m"], cfg["nb"], cfg["cplx"]
    # each step: a bounded sample of the workload (so W + K steps finish in minutes)
    # >= 8 columns per thread (the oracle's dynamic column queue balances them)
    cols = np.unique(np.linspace(1, m - 1, min(m - 1, 8 * max(threads, 2))).astype(np.int64))
    for _ in range(args.warmup):
        oracle.trevc(T, nb=nb, cols=cols[: max(1, len(cols) // 4)], nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.trevc(T, nb=nb, cols=cols, nthreads=threads)
        times.append(time.perf_counter() - t0)
    fl = algorithmic_flops_cols(cols, cplx)
    dt = float(np.mean(times))
    val = fl / dt / 1e9
    line = {"metric": METRIC, "value": val, "unit": "GFLOP/s", "impl": "reference", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64" if not cplx else "c128 (f64)",
            "data": "synthetic (seeded, inputs.py)",
            "config": {"workload": cfg["workload"], "m": m, "n": m, "nb": nb,
                       "sample_per_step": f"{len(cols)} evenly spaced eigenvectors"},
            "eigvecs_per_s": len(cols) / dt,
            "cpu_baseline": {"value": val, "unit": "GFLOP/s", "cores": threads, "kind": "oracle",
                             "cpu_model": cpu_model(), "per_core_gflops": val / threads,
                             "sample": f"{len(cols)} of {m} eigenvectors per step "
                                       f"(evenly spaced k, {len(cols) / threads:.0f} per thread)"},
            "e2e": {"value": val, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------------- CUDA arm
def run_cuda(args, cfgname):
    import torch
    import paper_1607_01477_b200 as ms
    from paper_1607_01477_b200 import dist as pdist

    ws, rank, local = dist_env()
    cfg = CONFIGS[cfgname]
    m, nb, cplx = cfg["m"], cfg["nb"], cfg["cplx"]
    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ms.load()
    dtype = torch.complex128 if cplx else torch.float64
    stream = torch.cuda.current_stream()

    # ---- inputs (host, seeded) -> HBM
    T_host = generate(cfgname) if rank == 0 else None
    Td = torch.empty((m, m), dtype=dtype, device="cuda").t()          # column-major
    if rank == 0:
        Td.copy_(torch.from_numpy(T_host))
    cols = pdist.shard_cols(m, ws, rank)
    ncols = len(cols)
    scales = torch.empty(ncols, dtype=torch.float64, device="cuda")
    exps = torch.empty(ncols, dtype=torch.int32, device="cuda")

    solve_evs = []          # (start, end) CUDA events around the local solve of each timed step

    def solve_cols(T, c, out):
        fn = ms.trevc_z_cols if cplx else ms.trevc_d_cols
        if timing["on"]:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        fn(T, m, m, c, len(c), out, m, scales, exps, nb)
        if timing["on"]:
            e1.record(stream)
            solve_evs.append((e0, e1))
        return exps

    timing = {"on": False}

    last = {}

    # N > 1: the library's native NCCL path (torch only bootstraps the process group and hands the
    # NCCL id over): delta + T's panels streamed right to left overlapping the shard solve, status
    # all-reduce, triangular all-gather, unpack (trevc_*_dist, csrc/mstrsm.cu).  MSTRSM_DIST_IMPL=torch
    # selects the torch.distributed mirror of the same sequence (paper_1607_01477_b200/dist.py).
    native = ws > 1 and os.environ.get("MSTRSM_DIST_IMPL", "native") == "native"
    if native:
        ms.comm_init(ws, rank)

    def step():
        if native:
            Z, _, e = ms.trevc_dist(Td if rank == 0 else None, m, nb=nb, root=0)
            last["Z"], last["e"] = Z, e
        else:
            # N = 1: the local solve; torch mirror for N > 1 (paper_1607_01477_b200/dist.py)
            last["Z"], last["e"] = pdist.trevc_sharded(Td, m, solve_cols, rank=rank, world=ws)

    # ---- FP64 roofline denominators (measured on this GPU, before timing)
    dmma_tf, dfma_tf = ms.fp64_peak(100.0)
    cublas = cublas_fp64_ceiling() if rank == 0 else None

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()

    ms.launch_count(1)
    ms.mstrsm_profile(1)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    sampler = ClockSampler(local)
    timing["on"] = True
    with sampler:
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            evs[i][0].record(stream)
            step()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        t_wall = time.perf_counter() - t_wall0
    timing["on"] = False
    if dist:
        dist.barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    solve_ms = float(np.sum([a.elapsed_time(b) for a, b in solve_evs]))
    launches = ms.launch_count(0)
    g_ms, g_n, g_fl = ms.mstrsm_profile_read(0)
    d_ms, d_n, d_fl = ms.mstrsm_profile_read(1)
    o_ms, o_n, _ = ms.mstrsm_profile_read(2)
    ms.mstrsm_profile(0)
    total_ms = float(np.sum(step_ms))
    if dist:
        t = torch.tensor([total_ms, solve_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms, solve_ms = float(t[0].item()), float(t[1].item())
    ms_per_step = total_ms / args.steps

    # correctness spot check of the timed output (cheap, outside the timed region)
    Zlast = last["Z"]
    ok_finite = bool(torch.isfinite(torch.view_as_real(Zlast) if cplx else Zlast).all().item())

    fl_step = algorithmic_flops_cols(np.arange(m), cplx)                # whole job, all ranks
    value = fl_step / (ms_per_step * 1e-3) / 1e9
    eig_per_s = m / (ms_per_step * 1e-3)

    if rank != 0:
        if native:
            ms.comm_destroy()
        if dist:
            dist.destroy_process_group()
        return 0

    # ---- roofline of the dominant kernel (the DMMA update GEMM), measured live.  `achieved` counts
    #      the real DMMA flops the kernel executes: the complex GEMM runs 3 real products per
    #      complex multiply-add (3M), i.e. 3/4 of the algorithmic 8MNK.
    prods = ms.gemm_real_products() if cplx else 4
    gemm_tf = (g_fl * prods / 4.0 / (g_ms * 1e-3) / 1e12) if g_ms > 0 else None
    gemm_alg_tf = (g_fl / (g_ms * 1e-3) / 1e12) if g_ms > 0 else None
    peak_tf = dmma_tf
    traffic, _ = ncu_traffic()
    roofline = {"bound": "tensor", "achieved": gemm_tf, "peak": peak_tf, "unit": "TFLOP/s",
                "frac": (gemm_tf / peak_tf) if gemm_tf else None, "traffic": traffic,
                "kernel": ((("gemm_ws3p_kernel (two" if os.environ.get("MSTRSM_3M_GROUPS") == "2" or nb < 96 else
                             "gemm_ws3q_kernel (three") +
                            " staggered consumer warpgroups; persistent warp-specialised, complex as 3 real "
                            "products with precomputed operand sums, TMA/bulk-copy producer, mma.sync m8n8k4 "
                            "f64 -> DMMA)")
                           if os.environ.get("MSTRSM_3M_PRESUM", "1") != "0" else
                           "gemm_ws3m_kernel<false> (persistent warp-specialised, complex as 3 real products, "
                           "mma.sync m8n8k4 f64 -> DMMA)") if (cplx and prods == 3) else
                          "gemm_ws_kernel (persistent warp-specialised, mma.sync m8n8k4 f64 -> DMMA)",
                "achieved_counts": f"executed real DMMA flops ({prods} real products per complex MAC)",
                "gemm_algorithmic_tflops": gemm_alg_tf,
                "peak_source": "measured: register-resident DMMA loop on all SMs (mstrsm_fp64_peak), "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "dfma_peak": dfma_tf,
                "derived_peak_tflops_at_max_clock": 148 * 64 * 2 * 1.965e9 / 1e12,
                "cublas_fp64": cublas,
                "gemm_launches": g_n, "gemm_ms_per_step": g_ms / args.steps,
                "gemm_share_of_step": (g_ms / args.steps) / ms_per_step,
                "diag_ms_per_step": d_ms / args.steps, "other_ms_per_step": o_ms / args.steps,
                "gemm_flops_per_launch": g_fl / max(g_n, 1)}

    clocks = sampler.summary()
    line = {"metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "c128 (f64)" if cplx else "f64",
            "data": "synthetic (seeded numpy generators, paper_1607_01477_b200/inputs.py)",
            "config": {"workload": cfg["workload"], "m": m, "n": m, "nb": nb,
                       "parallelism": f"shift-sharded x{ws} (serpentine block-cyclic, 16 cols)" +
                                      ("; native NCCL: delta + panel-streamed broadcast overlapping the "
                                       "shard solve, status all-reduce, triangular all-gather" if native else ""),
                       "l2": "inputs (4.3 GB T, 4.3 GB Z) >> 126 MB L2; no flush needed"},
            "eigvecs_per_s": eig_per_s,
            "pct_fp64_peak": 100.0 * value / 1e3 / (peak_tf * ws) if peak_tf else None,
            "pct_fp64_peak_note": "algorithmic flops (R18: 8 real flops per complex MAC) / measured DMMA "
                                  "peak x N; the 3M update executes 3/4 of those flops, so this is the "
                                  "metric's figure, not hardware utilisation (roofline.frac is)",
            "gflops_nominal_m2n": nominal_flops(m, m, cplx) / (ms_per_step * 1e-3) / 1e9,
            "roofline": roofline, "clocks": clocks, "gpu_launches": launches,
            "wall_s_timed": t_wall, "output_finite": ok_finite,
            "solve_only_ms_per_step": (solve_ms / args.steps) if not native else None,
            "solve_only_note": "the local trevc_*_cols call alone (CUDA events, max over ranks); ms_per_step "
                               "is end to end: broadcast + solve + all-gather + unpack (SURVEY §8d.5)"}

    if ws == 1 and cplx and not args.no_e2e:
        line["e2e"] = e2e_host(ms, T_host, m, nb, args)
    else:
        line["e2e"] = None
    if ws == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(T_host, cfg, budget_s=args.cpu_budget)
    print(json.dumps(line), flush=True)
    if native:
        ms.comm_destroy()
    if dist:
        dist.destroy_process_group()
    return 0


def e2e_host(ms, T_host, m, nb, args):
    """Same metric through the C-ABI host-buffer entries, every step's H2D of T (upper triangle,
    pinned host memory) and D2H of Z, scales and exponents inside the timed region:
      - headline: trevc_z_host_batch over K = max(steps, 3) problems (problem k+1's upload and k-1's
        download overlap problem k's solve; pipeline fill and drain included), time / K;
      - `single`: trevc_z_host one problem at a time (copies not overlapped)."""
    import torch
    Tp = torch.empty((m, m), dtype=torch.complex128, pin_memory=True).t()
    Tp.copy_(torch.from_numpy(T_host))
    Zp = torch.empty((m, m), dtype=torch.complex128, pin_memory=True).t()
    sp = torch.empty(m, dtype=torch.float64, pin_memory=True)
    ep = torch.empty(m, dtype=torch.int32, pin_memory=True)
    Tn, Zn, sn, en = Tp.numpy(), Zp.numpy(), sp.numpy(), ep.numpy()
    fl = algorithmic_flops_cols(np.arange(m), True)
    # the upper triangle of T is uploaded by 128-column panels (rows 0 .. panel end); Z comes back
    # the same way (rows 0..k of eigenvector k, R37), plus the scales (8 B) and exponents (4 B)
    h2d = sum(min(m, c0 + 128) * (min(m, c0 + 128) - c0) for c0 in range(0, m, 128)) * 16
    d2h = int(h2d) + m * 12
    ms.trevc_z_host(Tn, m, Zn, sn, en, nb)                              # warm-up
    single = []
    for _ in range(max(1, min(args.steps, 2))):
        t0 = time.perf_counter()
        ms.trevc_z_host(Tn, m, Zn, sn, en, nb)
        single.append(time.perf_counter() - t0)
    K = max(3, args.steps)
    ms.trevc_z_host_batch([Tn] * 2, m, [Zn] * 2, [sn] * 2, [en] * 2, nb)   # warm-up (streams, pools)
    t0 = time.perf_counter()
    ms.trevc_z_host_batch([Tn] * K, m, [Zn] * K, [sn] * K, [en] * K, nb)
    dt = (time.perf_counter() - t0) / K
    ds = float(np.mean(single))
    return {"value": fl / dt / 1e9, "unit": "GFLOP/s", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": d2h, "ms_per_step": dt * 1e3, "eigvecs_per_s": m / dt, "steps": K,
            "api": "trevc_z_host_batch (C ABI, pinned host buffers; uploads/downloads of neighbouring "
                   "problems overlap the solve; wall clock incl. pipeline fill and drain) / K",
            "single": {"value": fl / ds / 1e9, "ms_per_step": ds * 1e3, "steps": len(single),
                       "api": "trevc_z_host (one problem per call, copies not overlapped)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args, args.config)
    return run_cuda(args, args.config)


if __name__ == "__main__":
    sys.exit(main())
