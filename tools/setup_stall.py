"""Host-side timing of each call of the benchmark's device step (stall hunting).

usage: python tools/setup_stall.py [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402
from paper_1801_08464_b200.mgr import setup_from_matrix  # noqa: E402
from paper_1801_08464_b200.sparse import block_scale  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 12
s = synth.make_config(3, 128)
solver = pipeline.SyntheticSolver(rel_tol=1e-8)
a = solver.upload(s)
ctx = solver.ctx if hasattr(solver, "ctx") else _lib.ctx()
import numpy as np  # noqa: E402

b_dev = ctx.lib.mg_malloc if False else None
solver.setup()
xs = np.zeros(s.n)
for k in range(steps):
    T = [time.perf_counter()]
    if solver.hier is not None:
        solver.hier.free()
        solver.hier = None
    for m in (solver.dinv, solver.ahat):
        if m is not None:
            m.free()
    T.append(time.perf_counter())
    solver.dinv, solver.ahat = block_scale(solver.a)
    T.append(time.perf_counter())
    solver.hier = setup_from_matrix(solver.ahat, solver._plan[1], solver.amg_opts)
    T.append(time.perf_counter())
    solver.hier.set_prescale(solver.dinv)
    solver.ahat.free()
    solver.ahat = None
    T.append(time.perf_counter())
    res = solver.solve(s.rhs)
    T.append(time.perf_counter())
    t = ctx.timing()
    d = [1e3 * (T[i + 1] - T[i]) for i in range(len(T) - 1)]
    print(f"step {k}: free {d[0]:.1f} block_scale {d[1]:.1f} mgr_setup {d[2]:.1f} (dev {t.setup_ms:.1f}) "
          f"prescale {d[3]:.1f} solve {d[4]:.1f} its {res.iterations}", flush=True)
