"""Per-phase device time of one warm solve (mg_set_profiling)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402

NAMES = ["BCSR SpMV", "coarse AMG", "F-relax AMG", "GMRES ortho", "MGR transfers", "prescale", "D2H sync", "-"]


def main():
    cfg, edge = int(sys.argv[1]), int(sys.argv[2])
    s = synth.make_config(cfg, edge)
    ctx = _lib.ctx()
    solver = pipeline.SyntheticSolver(rel_tol=1e-8)
    solver.upload(s)
    for rep in range(3):
        solver.setup()
        ctx.set_profiling(rep == 2)
        t0 = time.perf_counter()
        res = solver.solve(s.rhs)
        t1 = time.perf_counter()
    ctx.set_profiling(False)
    t = ctx.timing()
    tot = t.solve_ms
    print(f"solve {tot:.1f} ms (wall {1e3*(t1-t0):.1f}), its {res.iterations}")
    acc = 0.0
    for k in range(7):
        acc += t.phase_ms[k]
        print(f"  {NAMES[k]:14s} {t.phase_ms[k]:8.2f} ms  {100*t.phase_ms[k]/tot:5.1f}%")
    print(f"  {'unaccounted':14s} {tot-acc:8.2f} ms  {100*(tot-acc)/tot:5.1f}%")


if __name__ == "__main__":
    main()
