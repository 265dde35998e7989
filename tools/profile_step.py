"""One block-scale + MGR setup + GMRES solve, for ncu launch lists.

usage: python tools/profile_step.py CFG EDGE [reps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402


def main():
    cfg, edge = int(sys.argv[1]), int(sys.argv[2])
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    s = synth.make_config(cfg, edge)
    ctx = _lib.ctx()
    solver = pipeline.SyntheticSolver(rel_tol=1e-8)
    solver.upload(s)
    for r in range(reps):
        ctx.sync()
        t0 = time.perf_counter()
        solver.setup()
        ctx.sync()
        t1 = time.perf_counter()
        res = solver.solve(s.rhs)
        t2 = time.perf_counter()
        tm = ctx.timing()
        print(f"rep {r}: setup {1e3*(t1-t0):.1f} ms (mgr_setup dev {tm.setup_ms:.1f}) solve {1e3*(t2-t1):.1f} ms "
              f"(dev {tm.solve_ms:.1f}) its {res.iterations} launches {ctx.launches}", flush=True)


if __name__ == "__main__":
    main()
