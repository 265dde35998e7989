"""Option exploration on one synthetic config (GPU): setup / solve ms, iterations
and hierarchy shapes for variants of the AMG options and the MGR plan.

    python tools/explore_opts.py CFG EDGE 'label:key=val,key=val' ...
keys: any AmgOptions field (e.g. coarse_size_cutoff=2000), gr=1 (global block
relaxation on every MGR level), frpre / frpost (F-relaxation AMG sweeps),
fr=jacobi|gauss_seidel|amg and frsweeps=N (the F-relaxation kind, mgr.py:159-209),
rp=injective|noninjective|injection (RpKind of every MGR level, mgr.py:47-51),
post=1 (MGR post-smoothing: the F-relaxation again after the coarse correction), frmax=N (FRelax.max_levels).
"""
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402
from paper_1801_08464_b200.mgr import FRelax, RpKind  # noqa: E402


def run(ctx, s, label, kv, reps=3, warm=2):
    amg_kw = dict(pipeline.DEFAULT_AMG)
    fr_kw = dict(pipeline.DEFAULT_FRELAX)
    gr = False
    fr_kind, fr_sweeps = "amg", 1
    rp = None
    post = None
    for k, v in kv.items():
        if k == "gr":
            gr = bool(int(v))
        elif k == "fr":
            fr_kind = v
        elif k == "rp":
            rp = RpKind[v.upper()]
        elif k == "post":
            post = bool(int(v))
        elif k == "frmax":
            fr_kw["max_levels"] = int(v)
        elif k == "frsweeps":
            fr_sweeps = int(v)
        elif k in ("frpre", "frpost"):
            fr_kw["pre" if k == "frpre" else "post"] = int(v)
        else:
            amg_kw[k] = type(pipeline.DEFAULT_AMG.get(k, 0))(v) if k in pipeline.DEFAULT_AMG else int(v)
    solver = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx, amg_opts=pipeline.default_amg_options(**amg_kw),
                                      frelax=FRelax("amg", **fr_kw) if fr_kind == "amg" else FRelax(fr_kind, sweeps=fr_sweeps),
                                      global_relax=gr, rp=rp, post_smoothing=post)
    solver.upload(s)
    rows = []
    for r in range(warm + reps):
        solver.setup()
        t_set = ctx.timing().setup_ms
        res = solver.solve(s.rhs)
        t = ctx.timing()
        if r >= warm:
            rows.append((t_set, t.solve_ms, res.iterations))
    h = solver.hier
    su = statistics.median(x[0] for x in rows)
    so = statistics.median(x[1] for x in rows)
    print(f"{label:28s} its {rows[-1][2]:4d} setup {su:7.1f} solve {so:7.1f} ms  {s.n / ((su + so) / 1e3) / 1e6:6.2f} "
          f"MDOF/s  F-AMG {h.amg(0).level_sizes() if fr_kind == 'amg' else fr_kind} coarse {h.amg(-1).level_sizes()}",
          flush=True)
    solver.hier.free()
    solver.a.free()


def main():
    cfg, edge = int(sys.argv[1]), int(sys.argv[2])
    ctx = _lib.ctx()
    s = synth.make_config(cfg, edge)
    for spec in sys.argv[3:]:
        label, _, kvs = spec.partition(":")
        kv = dict(x.split("=") for x in kvs.split(",") if x)
        run(ctx, s, label, kv)


if __name__ == "__main__":
    main()
