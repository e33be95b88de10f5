"""Per-kernel HBM roofline table from an ncu launch list captured with
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none --profile-from-start off --csv --log-file L.csv \
      python tools/warm_step.py 256
(one warm 256^3 step).  GB/s = measured DRAM bytes / kernel duration (ncu,
serialised, one replay per metric group), fraction of the measured copy
peak (MEASURED_PEAKS.json).  Usage: python tools/roofline_table.py L.csv [top]"""
import collections
import csv
import json
import os
import sys

UNIT_T = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
UNIT_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, top=25):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ii, ki = hdr.index("ID"), hdr.index("Kernel Name")
    mi, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    launch = collections.defaultdict(dict)
    for r in rows:
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            v *= UNIT_T[r[ui]]
        else:
            v *= UNIT_B.get(r[ui], 1.0)
        launch[(r[ii], r[ki])][r[mi]] = v
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for (_, k), m in launch.items():
        name = k.split("(")[0].replace("void ", "").replace("flip::", "")[:52]
        a = agg[name]
        a[0] += 1
        a[1] += m.get("gpu__time_duration.sum", 0.0)
        a[2] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    try:
        peak = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))["hbm_gbs"]
    except Exception:
        peak = 6552.6
    tot = sum(a[1] for a in agg.values())
    print(f"{sum(a[0] for a in agg.values())} launches, {tot / 1e3:.2f} ms kernel time; peak {peak} GB/s")
    print("| kernel | launches | avg us | share | DRAM MB / launch | GB/s | HBM frac |")
    print("|---|---|---|---|---|---|---|")
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        gbs = b / (t * 1e-6) / 1e9 if t else 0.0
        print(f"| `{k}` | {n} | {t / n:.1f} | {100 * t / tot:.1f}% | {b / n / 1e6:.1f} | "
              f"{gbs:.0f} | {gbs / peak:.1%} |")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
