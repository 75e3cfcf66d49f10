"""Print the key metrics + top stall reasons of every kernel in an .ncu-rep.

    python scripts/ncu_summary.py gpurun_out/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "smsp__inst_executed.sum",
        "lts__t_sectors_srcunit_tex_op_red.sum", "l1tex__t_sector_hit_rate.pct"]


def main(path):
    if path.endswith(".csv"):  # an exported `--page raw --csv` table
        out = open(path).read()
    else:
        out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    for r in rows[2:]:
        print("----", r[h.index("Kernel Name")][:90])
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"   {k:58s} {r[i]} {units[i]}")
        st = [(h[i], r[i]) for i in range(len(h))
              if h[i].startswith("smsp__average_warps_issue_stalled") and h[i].endswith("per_issue_active.ratio")]
        st = sorted(st, key=lambda x: -float(x[1] or 0))[:5]
        print("   stalls:", ", ".join(f"{k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')}={float(v):.2f}" for k, v in st))


if __name__ == "__main__":
    main(sys.argv[1])
