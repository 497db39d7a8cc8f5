"""Summarise an ncu --csv launch list (gpu__time_duration.sum) per kernel."""
import collections
import csv
import sys


def summarise(path, out=sys.stdout):
    rows = list(csv.reader(open(path)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[start + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        v *= {"nsecond": 1.0, "usecond": 1e3, "msecond": 1e6, "second": 1e9}.get(r[ui], 1.0)
        name = r[ki].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(a[1] for a in agg.values())
    out.write(f"{'kernel':58s} {'launches':>8s} {'total ms':>10s} {'us/launch':>10s} {'share':>6s}\n")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.write(f"{k[:58]:58s} {c:8d} {t / 1e6:10.3f} {t / c / 1e3:10.1f} {100 * t / tot:5.1f}%\n")
    out.write(f"{'TOTAL':58s} {sum(a[0] for a in agg.values()):8d} {tot / 1e6:10.3f}\n")


if __name__ == "__main__":
    summarise(sys.argv[1])
