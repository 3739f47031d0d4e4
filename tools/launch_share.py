"""Per-kernel share of one c5 step from an ncu launch list (gpu__time_duration.sum csv).

    python tools/launch_share.py <launches.csv> "<command description>" > profiles/r01/launch_share_<tag>.txt

Steps are delimited by the first kernel of a TriangEig (trevc_prepass_kernel, or the norm pass); the last step is reported (libmstrsm kernels only)."""
import collections
import csv
import sys


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    start = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[start]
    I = h.index
    launches = []
    for r in rows[start + 1:]:
        if len(r) < len(h) or r[I("Metric Name")] != "gpu__time_duration.sum":
            continue
        launches.append((r[I("Kernel Name")].split("(")[0], float(r[I("Metric Value")].replace(",", "")) / 1e6))
    begins = []
    for marker in ("trevc_prepass_kernel", "norm_cols_n_kernel", "init_trevc_kernel"):
        begins = [i for i, (n, _) in enumerate(launches) if marker in n]
        if begins:
            break
    step = [x for x in launches[begins[-1]:] if "mstrsm::" in x[0]]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in step:
        agg[n][0] += 1
        agg[n][1] += v
    tot = sum(v for _, v in agg.values())
    print("ncu launch list (gpu__time_duration.sum, --clock-control none, serialised, cold-cache) of the")
    print(f"last timed step of: {sys.argv[2]}")
    for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{n[:60]:60s} launches {c:4d} {v:10.2f} ms  share {100 * v / tot:5.1f}%")
    print(f"total libmstrsm kernel time {tot:.2f} ms")


if __name__ == "__main__":
    main()
