"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-kernel totals.

usage: python tools/launch_sum.py launches.csv [--second-half] [--top N]
--second-half keeps only the launches after the midpoint (the warm repetition
when the captured program ran the same phase twice).
"""
import collections
import csv
import re
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    hdr, data = None, []
    for r in csv.reader(open(path)):
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    if "--second-half" in sys.argv:
        data = data[len(data) // 2:]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        n = re.sub(r"\(.*", "", d["Kernel Name"]).replace("void ", "").replace("mg::", "")
        agg[n][0] += 1
        agg[n][1] += float(d["Metric Value"]) / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"{len(data)} launches, {tot / 1e3:.2f} ms kernel time (cold-cache, serialised: compare SHARES)")
    print(" share       ms launches   avg us  kernel")
    for n, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        print(f"{100 * s / tot:5.1f}% {s / 1e3:8.2f} {c:8d} {s / c:8.1f}  {n[:80]}")


if __name__ == "__main__":
    main()
