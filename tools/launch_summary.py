"""Per-kernel totals from an ncu `--metrics gpu__time_duration.sum --csv`
launch list: python tools/launch_summary.py launches.csv [top]."""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3,
        "second": 1e6, "s": 1e6}


def main(path, top=30):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, rows = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows:
        us = float(r[vi].replace(",", "")) * UNIT[r[ui]]
        name = r[ki].split("(")[0][:58]
        agg[name][0] += 1
        agg[name][1] += us
    tot = sum(t for _, t in agg.values())
    print(f"{len(rows)} launches, {tot / 1e3:.2f} ms of kernel time")
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{k:58s} {n:5d} {t / n:9.1f} us {t / 1e3:8.2f} ms {100 * t / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
