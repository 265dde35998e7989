"""Per-kernel HBM bandwidth on the config-3 hierarchy (CUDA events, warm, many reps).

Bytes are the stored format's (column indices at the plan's 4 / 2 / 1 B per entry).

usage: python tools/kbench.py [CFG] [EDGE] [reps]
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402


def devbuf(ctx, n, fill=None):
    p = _lib.P()
    ctx.call("mg_dev_alloc", 8 * n, ctypes.byref(p))
    v = np.random.default_rng(0).standard_normal(n) if fill is None else np.full(n, fill)
    ctx.call("mg_memcpy_h2d", p, _lib.ptr(v), 8 * n)
    return p


def time_spmv(ctx, m, reps):
    nr, nc = m.nrows, m.ncols
    x, y = devbuf(ctx, nc), devbuf(ctx, nr)
    for _ in range(3):
        ctx.call("mg_spmv_dev", m.h, x, y)
    ctx.call("mg_timer_start")
    for _ in range(reps):
        ctx.call("mg_spmv_dev", m.h, x, y)
    v = ctypes.c_double()
    ctx.call("mg_timer_stop", ctypes.byref(v))
    ms = v.value / reps
    _, _, nnz, b = m._load_info()
    nbr = nr // b
    _, ib, _ = m.spmv_layout()  # stored bytes per column index (4 / 2 / 1)
    byt = nnz * (8.0 * b * b + ib) + 4 * (nbr + 1) + 8.0 * nc + 8.0 * nr
    ctx.call("mg_dev_free", x)
    ctx.call("mg_dev_free", y)
    return ms, byt


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    edge = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    ctx = _lib.ctx()
    s = synth.make_config(cfg, edge)
    solver = pipeline.SyntheticSolver()
    a = solver.upload(s)
    h = solver.setup()
    peak = 6538.9
    rows = [("BCSR A", a)]
    rows.append(("MGR A_hat (level 0)", h.level_matrix(0, "a")))
    rows.append(("MGR R", h.level_matrix(0, "r")))
    rows.append(("MGR P", h.level_matrix(0, "p")))
    rows.append(("MGR A_ff", h.level_matrix(0, "a_ff")))
    camg = h.amg(-1)
    for k in range(camg.nlevels):
        if camg.levels[k].a.nrows >= 10000:
            rows.append((f"coarse AMG A_{k}", camg.levels[k].a))
    famg = h.amg(0)
    for k in range(famg.nlevels):
        if famg.levels[k].a.nrows >= 10000:
            rows.append((f"F-relax AMG A_{k}", famg.levels[k].a))
    for nm, hh in (("coarse", camg), ("F-relax", famg)):
        for k in range(min(2, hh.nlevels - 1)):
            pk = hh.levels[k].p
            rows.append((f"{nm} AMG P_{k}", pk))
            rows.append((f"{nm} AMG R_{k}", pk.transpose()))
    for name, m in rows:
        ms, byt = time_spmv(ctx, m, reps)
        sell, ib, srt = m.spmv_layout()
        lay = ("SELL-s" if srt else "SELL") if sell else "CSR"
        print(f"{name:22s} {lay:6s} idx {ib}B rows={m.nrows:9d} nnz={m.nnz:10d} nnz/row={m.nnz/max(m.nrows,1)*(m.block_size**2)/m.block_size:6.1f} "
              f"{ms*1e3:9.1f} us  {byt/ms/1e6:8.1f} GB/s  {byt/ms/1e6/peak*100:5.1f}% of {peak}", flush=True)


if __name__ == "__main__":
    main()
