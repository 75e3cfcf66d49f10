"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes) per kernel.

    python scripts/launch_summary.py gpurun_out/launches.csv [--skip-gen]
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        lid = r[0]
        names[lid] = r[ki].split("(")[0].replace("void ", "")
        v = float(r[vi].replace(",", ""))
        u = r[ui]
        scale = {"nsecond": 1e-6, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "usecond": 1e-3, "msecond": 1.0,
                 "second": 1e3, "byte": 1.0, "Kbyte": 1e3,
                 "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1.0)
        per[lid][r[mi]] = v * scale
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for lid, m in per.items():
        a = agg[names[lid]]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':34s} {'n':>5s} {'total ms':>10s} {'avg ms':>9s} {'share':>6s} {'GB/launch':>10s} {'GB/s':>8s}")
    for k, (n, ms, by) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:34s} {n:5d} {ms:10.3f} {ms / n:9.4f} {100 * ms / tot:5.1f}% {by / n / 1e9:10.4f} "
              f"{(by / 1e9) / (ms / 1e3) if ms else 0:8.0f}")
    print(f"total {tot:.3f} ms over {sum(v[0] for v in agg.values())} launches")


if __name__ == "__main__":
    main(sys.argv[1])
