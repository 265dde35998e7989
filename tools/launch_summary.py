"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per kernel share)."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[hdr]
    ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
    mult = {'ns': 1e-3, 'nsecond': 1e-3, 'us': 1.0, 'usecond': 1.0, 'ms': 1e3, 'msecond': 1e3}
    agg = collections.defaultdict(lambda: [0, 0.0])
    tot = 0.0
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(',', '')) * mult[r[ui]]
        name = r[ki].split('(')[0].replace('void ', '').replace('mg::', '')[:60]
        agg[name][0] += 1
        agg[name][1] += v
        tot += v
    n = sum(c for c, _ in agg.values())
    print(f"{n} launches, {tot/1e3:.1f} ms total kernel time (ncu-serialised, cold cache)")
    print(f"{'share':>6} {'ms':>9} {'launches':>8} {'avg us':>9}  kernel")
    for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{100*t/tot:5.1f}% {t/1e3:9.2f} {c:8d} {t/c:9.1f}  {k}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
