"""Diagnose per-step timing: device-resident steps with / without the nvidia-smi sampler."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_1801_08464_b200 import _lib, synth  # noqa: E402
from paper_1801_08464_b200.pipeline import SyntheticSolver  # noqa: E402


def main():
    ctx = _lib.ctx()
    s = synth.make_config(3, int(sys.argv[1]) if len(sys.argv) > 1 else 128)
    solver = SyntheticSolver(ctx=ctx)
    a = solver.upload(s)
    b_dev, x_dev = _lib.P(), _lib.P()
    ctx.call("mg_dev_alloc", 8 * s.n, _lib.ctypes.byref(b_dev))
    ctx.call("mg_dev_alloc", 8 * s.n, _lib.ctypes.byref(x_dev))
    rhs = np.ascontiguousarray(s.rhs)
    ctx.call("mg_memcpy_h2d", b_dev, _lib.ptr(rhs), 8 * s.n)
    g = solver.gopts.to_c()
    res = _lib.GmresRes()

    def step():
        t0 = time.perf_counter()
        solver.setup()
        ctx.sync()
        t1 = time.perf_counter()
        ctx.call("mg_gmres_dev", a.h, solver.hier.h, b_dev, x_dev, _lib.ctypes.byref(g), -1.0, _lib.ctypes.byref(res))
        ctx.sync()
        t2 = time.perf_counter()
        t = ctx.timing()
        return (t1 - t0) * 1e3, (t2 - t1) * 1e3, t.setup_ms, t.solve_ms

    for tag in ("plain", "plain", "sampler", "plain"):
        clk = bench.ClockSampler(0) if tag == "sampler" else None
        if clk:
            clk.start()
        r = [step() for _ in range(3)]
        if clk:
            print(clk.stop())
        for x in r:
            print(tag, "setup wall %.1f (mgr %.1f)  solve wall %.1f (dev %.1f)" % (x[0], x[2], x[1], x[3]), flush=True)


if __name__ == "__main__":
    main()
