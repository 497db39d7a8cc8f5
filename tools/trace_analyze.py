"""Analyse a tools/chol_trace.py timeline: per-phase span, small/large split,
critical path (chain of fronts whose completion gated the root)."""
import sys

import numpy as np


def analyse(path):
    d = np.load(path)
    tr, nrows, ncols, parent, order = d["trace"], d["nrows"], d["ncols"], d["parent"], d["order"]
    nfs = int(d["nf_small"])
    small = np.zeros(len(nrows), bool)
    small[order[:nfs]] = True
    if "panels" in d:
        fb = d["panels"].astype(np.float64)[32:]
        ok = fb[:, 0] > 0
        if ok.any():
            b0 = fb[ok][0, 0]
            print("forward blocks of the last front (us): start  diag-solve  gemv")
            for row in fb[ok]:
                print("   %8.1f %6.1f %6.1f" % ((row[0] - b0) / 1e3, (row[1] - row[0]) / 1e3, (row[2] - row[1]) / 1e3))
    for ph, name in enumerate(("factor", "forward", "backward")):
        t = tr[ph].astype(np.float64)
        t0 = t[:, 0][t[:, 0] > 0].min()
        t = np.where(t > 0, t - t0, np.nan)
        span = np.nanmax(t[:, 3])
        print(f"== {name}: span {span / 1e3:.1f} us")
        for lab, mk in (("small", small), ("large", ~small)):
            if mk.sum() == 0:
                continue
            dur = t[mk, 3] - t[mk, 1]
            wait = t[mk, 1] - t[mk, 0]
            print(f"  {lab:5s} n={mk.sum():6d} end {np.nanmax(t[mk, 3]) / 1e3:8.1f} us  "
                  f"work mean {np.nanmean(dur) / 1e3:7.2f} us max {np.nanmax(dur) / 1e3:7.1f}  "
                  f"wait mean {np.nanmean(wait) / 1e3:7.2f} us  sum work {np.nansum(dur) / 1e3:9.0f} us")
        if ph == 2:
            # backward: the last-finishing front and its chain of parents
            J = int(np.nanargmax(t[:, 3]))
            chain = []
            while J >= 0 and J < len(parent):
                chain.append(J)
                pj = int(parent[J])
                if pj == J or pj < 0:
                    break
                J = pj
            print("  backward critical chain (last front first): front w s  start, wait, work us")
            for J in chain[:60]:
                a = t[J]
                print(f"   {J:6d} w={ncols[J]:4d} s={nrows[J]:4d} {'S' if small[J] else 'L'} "
                      f"start {a[0] / 1e3:8.1f} wait {(a[1] - a[0]) / 1e3:7.1f} work {(a[3] - a[1]) / 1e3:7.1f}")
        if ph in (0, 1):
            # critical path backwards from the last-finishing root
            J = int(np.nanargmax(t[:, 3]))
            chain = []
            children = {}
            for c, p in enumerate(parent):
                children.setdefault(int(p), []).append(c)
            while True:
                chain.append(J)
                ch = children.get(J, [])
                if not ch:
                    break
                J = max(ch, key=lambda c: t[c, 3])
            tot = 0.0
            print("  critical chain (root first): front w s  [wait->deps, deps->asm, asm->done] us")
            if ph == 0 and "panels" in d:
                pt = d["panels"].astype(np.float64)[:32]
                ok = pt[:, 0] > 0
                if ok.any():
                    p0 = pt[ok]
                    base = p0[0, 0]
                    print("  last front panels (us): start  load  diag  trsm  update")
                    for row in p0:
                        print("   %8.1f %6.1f %6.1f %6.1f %6.1f" % ((row[0] - base) / 1e3, *(np.diff(row) / 1e3)))
            for J in chain[:40]:
                a = t[J]
                print(f"   {J:6d} w={ncols[J]:4d} s={nrows[J]:4d} {'S' if small[J] else 'L'} "
                      f"start {a[0] / 1e3:8.1f} deps {(a[1] - a[0]) / 1e3:7.1f} "
                      f"asm {(a[2] - a[1]) / 1e3 if not np.isnan(a[2]) else float('nan'):7.1f} "
                      f"done {(a[3] - (a[2] if not np.isnan(a[2]) else a[1])) / 1e3:7.1f}")


if __name__ == "__main__":
    analyse(sys.argv[1])
