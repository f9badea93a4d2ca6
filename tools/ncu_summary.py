"""Summarise an ncu --csv launch list (gpu__time_duration + optional byte metrics) per kernel."""
import csv
import sys
from collections import OrderedDict


def main(path, last=0):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    H = rows[hdr]
    ki, mi, vi, idi = H.index("Kernel Name"), H.index("Metric Name"), H.index("Metric Value"), H.index("ID")
    d = OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            d.setdefault((int(r[idi]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    items = list(d.items())
    if last:
        items = items[-last:]
    agg = OrderedDict()
    for (_, k), v in items:
        a = agg.setdefault(k[:70], {"n": 0, "us": 0.0, "rd": 0.0, "wr": 0.0})
        a["n"] += 1
        a["us"] += v.get("gpu__time_duration.sum", 0) / 1e3
        a["rd"] += v.get("dram__bytes_read.sum", 0)
        a["wr"] += v.get("dram__bytes_write.sum", 0)
    tot = sum(a["us"] for a in agg.values())
    print(f"{'n':>5} {'total_us':>10} {'avg_us':>9} {'share':>6} {'rdMB/l':>8} {'wrMB/l':>8}  kernel")
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        print(f"{a['n']:5d} {a['us']:10.1f} {a['us'] / a['n']:9.2f} {100 * a['us'] / tot:5.1f}% "
              f"{a['rd'] / a['n'] / 1e6:8.1f} {a['wr'] / a['n'] / 1e6:8.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 0)
