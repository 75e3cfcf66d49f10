"""Per-launch DRAM / L2 traffic of the bench's dominant kernels from one ncu capture.

    python scripts/roofline.py gpurun_out/roofline.raw.csv > profiles/traffic.json

The capture (scripts/profile_round.sh) holds `ncu --set full` rows for the two
launches of one K3 walk (merged nonzeros + zero stratum, k_walk_tma<2, 0, *>)
and one weight-gradient walk (k_wgrad).  Output: time, DRAM bytes and L2 bytes
per walk (sum over its launches), which bench.py turns into dram_frac / l2_frac.
"""
import csv
import io
import json
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "sector": 1.0,
        "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main(path):
    rows = list(csv.reader(io.StringIO(open(path).read())))
    h, units = rows[0], rows[1]

    def val(r, name):
        if name not in h:
            return None
        i = h.index(name)
        try:
            return float(r[i].replace(",", "")) * UNIT.get(units[i], 1.0)
        except ValueError:
            return None

    walks = {}
    for r in rows[2:]:
        name = r[h.index("Kernel Name")]
        key = "k3" if "k_walk_tma" in name and "<2, 0" in name else ("k3" if "k_sgrad" in name else
                                                                    ("k2w" if "wgrad" in name else None))
        if key is None:
            continue
        w = walks.setdefault(key, {"launches": [], "time_ms": 0.0, "dram_bytes": 0.0, "l2_bytes": 0.0})
        t = val(r, "gpu__time_duration.sum")
        dr = (val(r, "dram__bytes_read.sum") or 0.0) + (val(r, "dram__bytes_write.sum") or 0.0)
        sec = val(r, "lts__t_sectors.sum")
        l2 = sec * 32.0 if sec is not None else (val(r, "lts__t_bytes.sum") or 0.0)
        w["launches"].append({"kernel": name.split("(")[0], "time_ms": t, "dram_bytes": dr, "l2_bytes": l2,
                              "lts_pct": val(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
                              "red_sectors": val(r, "lts__t_sectors_srcunit_tex_op_red.sum")})
        w["time_ms"] += t or 0.0
        w["dram_bytes"] += dr
        w["l2_bytes"] += l2
    json.dump({"source": path, "walks": walks}, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
