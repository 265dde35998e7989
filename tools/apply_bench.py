"""Graph-replayed MGR applies at 128^3 config 3: device time per apply (CUDA events
on the library stream), for comparison with the per-kernel durations of the same
applies from an ncu launch list (the difference is launch / dependency overhead).

    python tools/apply_bench.py [CFG EDGE REPS]
"""
import ctypes
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402


def main():
    cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    edge = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
    s = synth.make_config(cfg, edge)
    ctx = _lib.ctx()
    solver = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx)
    solver.upload(s)
    solver.setup()
    n = s.n
    r, e = _lib.P(), _lib.P()
    ctx.call("mg_dev_alloc", 8 * n, ctypes.byref(r))
    ctx.call("mg_dev_alloc", 8 * n, ctypes.byref(e))
    rh = np.random.default_rng(0).standard_normal(n)
    ctx.call("mg_memcpy_h2d", r, _lib.ptr(rh), 8 * n)
    import time
    ctx.sync()
    t0 = time.perf_counter()
    ctx.call("mg_mgr_apply_dev", solver.hier.h, r, e)  # first apply: graph capture + instantiate
    ctx.sync()
    t1 = time.perf_counter()
    ctx.call("mg_mgr_apply_dev", solver.hier.h, r, e)
    ctx.sync()
    t2 = time.perf_counter()
    print(f"first apply (capture + instantiate + run) {1e3 * (t1 - t0):.2f} ms, second {1e3 * (t2 - t1):.2f} ms",
          flush=True)
    for _ in range(5):
        ctx.call("mg_mgr_apply_dev", solver.hier.h, r, e)
    ctx.sync()
    ctx.call("mg_timer_start")
    for _ in range(reps):
        ctx.call("mg_mgr_apply_dev", solver.hier.h, r, e)
    ms = ctypes.c_double()
    ctx.call("mg_timer_stop", ctypes.byref(ms))
    print(f"config {cfg} {edge}^3: {ms.value / reps * 1e3:.1f} us per graph-replayed MGR apply ({reps} reps), "
          f"F-AMG {solver.hier.amg(0).level_sizes()} coarse {solver.hier.amg(-1).level_sizes()}", flush=True)


if __name__ == "__main__":
    main()
