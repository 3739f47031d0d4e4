"""Summarise one `ncu --set full` capture of the update GEMM into profiles/ncu_gemm_traffic.json
(the `traffic` field of bench.py's roofline).

    python tools/ncu_traffic.py <report.ncu-rep> <raw-csv-out> "<launch description>" M N K [planes]

`planes` = 1 when the kernel also reads the operand-sum planes (gemm_ws3p_kernel)."""
import csv
import json
import subprocess
import sys


def main():
    rep, raw_out, desc = sys.argv[1], sys.argv[2], sys.argv[3]
    M, N, K = (int(v) for v in sys.argv[4:7])
    planes = len(sys.argv) > 7 and sys.argv[7] == "1"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    open(raw_out, "w").write(raw)
    rows = list(csv.reader(raw.splitlines()))
    h, units, v = rows[0], rows[1], rows[2]
    get = lambda name: float(v[h.index(name)].replace(",", ""))
    unit = lambda name: units[h.index(name)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = get("dram__bytes_read.sum") * scale[unit("dram__bytes_read.sum")]
    wr = get("dram__bytes_write.sum") * scale[unit("dram__bytes_write.sum")]
    dur = get("gpu__time_duration.sum") * {"ns": 1e-6, "us": 1e-3, "ms": 1.0}[unit("gpu__time_duration.sum")]
    alg = M * K * 16 + K * N * 16 + 2 * M * N * 16 + ((M * K + K * N) * 8 if planes else 0)
    out = {"source": f"{raw_out} (ncu --set full --clock-control none, {desc})",
           "dram_bytes_per_launch": int(rd + wr), "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
           "algorithmic_bytes_this_launch": alg,
           "dmma_active_pct": get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
           "duration_ms": dur,
           "note": "algorithmic = A (M*K*16) + X (K*N*16) + C read+write (2*M*N*16)"
                   + (" + operand-sum planes A+ (M*K*8), X+ (K*N*8)" if planes else "")}
    json.dump(out, open("profiles/ncu_gemm_traffic.json", "w"), indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
