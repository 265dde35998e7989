"""Summarise an MG_TRACE log (tools/setup_trace.py): per-AMG-level setup time and phase totals."""
import re
import sys
from collections import defaultdict


def main(path):
    lines = open(path).read().split("==== setup 1")[-1].splitlines()
    lvl, hier, out, phase = None, 0, [], defaultdict(float)
    for ln in lines:
        m = re.match(r"\[mg\] (.*?)\s+([\d.]+) ms\s+(\d+) syncs\s+(\d+) launches", ln)
        if not m:
            continue
        what, ms, sy, la = m.group(1).strip(), float(m.group(2)), int(m.group(3)), int(m.group(4))
        mm = re.match(r"amg level (\d+) start n=(\d+) nnz=(\d+)", what)
        if mm:
            if int(mm.group(1)) == 0:
                hier += 1
            lvl = [hier, int(mm.group(1)), int(mm.group(2)), int(mm.group(3)), 0.0, 0, 0]
            out.append(lvl)
            continue
        phase[what] += ms
        if what.startswith("mgr:"):
            lvl = None
        elif lvl is not None:
            lvl[4] += ms
            lvl[5] += sy
            lvl[6] += la
    print("hier level        n        nnz     ms  syncs launches")
    for h, l, n, nnz, ms, sy, la in out:
        print(f"{h:4d} {l:5d} {n:8d} {nnz:10d} {ms:6.2f} {sy:6d} {la:8d}")
    print("phase totals (ms):", {k: round(v, 2) for k, v in sorted(phase.items(), key=lambda x: -x[1])})
    print("total ms", round(sum(phase.values()), 2))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/trace.log")
