"""Opcode mix and top stall sites of one kernel from `ncu --page source --print-source sass --csv`.

    ncu -i prof.ncu-rep --page source --csv --kernel-name regex:NAME --print-source sass > sass.csv
    python scripts/sass_hotspots.py sass.csv
"""
import collections
import csv
import sys


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return None


def main(path):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    ai, si, ie, ws = (h.index(k) for k in ("Address", "Source", "Instructions Executed",
                                            "Warp Stall Sampling (All Samples)"))
    data = [r for r in rows[2:] if len(r) == len(h) and num(r[ie]) is not None]
    tot = sum(num(r[ie]) for r in data)
    totst = sum(num(r[ws]) or 0 for r in data)
    print(f"instructions {tot:.4g}  stall samples {totst:.4g}")
    op, opst = collections.Counter(), collections.Counter()
    for r in data:
        t = r[si].split()
        if not t:
            continue
        o = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        op[o] += num(r[ie])
        opst[o] += num(r[ws]) or 0
    for k, v in op.most_common(24):
        print(f"  {k:10s} {100 * v / tot:6.2f}% inst  {100 * opst[k] / max(totst, 1):6.2f}% stall samples")
    print("top stall sites:")
    for r in sorted(data, key=lambda r: -(num(r[ws]) or 0))[:14]:
        print(f"  {r[ai]} {r[si][:70]:70s} stalls={r[ws]} inst={r[ie]}")


if __name__ == "__main__":
    main(sys.argv[1])
