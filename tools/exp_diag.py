"""Experiment driver: time one c5-shaped TriangEig with the library named by MSTRSM_LIB and report
the per-kind kernel time (live CUDA-event profile) and, with --handed, the fallback counts."""
import os, subprocess, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) > 1 and sys.argv[1] == "--child":
    import torch
    import paper_1607_01477_b200 as ms
    from paper_1607_01477_b200 import inputs
    ms.load()
    m = int(sys.argv[2])
    nb = int(os.environ.get("EXP_NB", "128"))
    T = inputs.c5_grcar_like(m=m)
    Td = torch.from_numpy(T).cuda()
    ms.trevc(Td, nb=nb); torch.cuda.synchronize()
    ms.mstrsm_profile(1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); Z, sc, e = ms.trevc(Td, nb=nb); e1.record(); torch.cuda.synchronize()
    g = ms.mstrsm_profile_read(0); d = ms.mstrsm_profile_read(1)
    ms.mstrsm_profile(0)
    print(json.dumps({"lib": os.environ.get("MSTRSM_LIB", "default"), "m": m, "nb": nb, "total_ms": e0.elapsed_time(e1),
                      "gemm_ms": g[0], "diag_ms": d[0], "emin": int(e.min().item())}), flush=True)
    sys.exit(0)
m = sys.argv[1] if len(sys.argv) > 1 else "16384"
for lib in sys.argv[2:]:
    env = dict(os.environ, MSTRSM_LIB=os.path.abspath(lib))
    subprocess.run([sys.executable, __file__, "--child", m], env=env, timeout=300)
    if os.environ.get("EXP_NOHANDED"):
        continue
    env["MSTRSM_DEBUG_SYNC"] = "1"
    r = subprocess.run([sys.executable, __file__, "--child", m], env=env, timeout=300, capture_output=True, text=True)
    handed = sum(int(l.split()[-1]) for l in r.stderr.splitlines() if "main done" in l)
    print(json.dumps({"lib": lib, "handed_total": handed}), flush=True)
