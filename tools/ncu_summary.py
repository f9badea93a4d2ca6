"""Summarise an ncu --csv launch list: per-kernel count, total/avg time, DRAM bytes."""
import collections
import csv
import sys


def main(path, top=20):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    idx = {h: j for j, h in enumerate(hdr)}
    by = collections.defaultdict(dict)
    names = {}
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        i = int(r[idx["ID"]])
        names[i] = r[idx["Kernel Name"]]
        by[i][r[idx["Metric Name"]]] = float(r[idx["Metric Value"]].replace(",", ""))
    tot = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for i, d in by.items():
        t = tot[names[i][:90]]
        t[0] += 1
        t[1] += d.get("gpu__time_duration.sum", 0.0)
        t[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    grand = sum(t[1] for t in tot.values())
    print(f"{'n':>5} {'total_us':>10} {'avg_us':>9} {'share':>6} {'MB/launch':>10}  kernel")
    for n, t in sorted(tot.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{t[0]:5d} {t[1] / 1e3:10.1f} {t[1] / 1e3 / t[0]:9.2f} {t[1] / grand:6.1%} {t[2] / 1e6 / t[0]:10.2f}  {n}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 20)
