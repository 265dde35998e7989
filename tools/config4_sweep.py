"""Config 4 (b=3, 3-level MGR: S, then rho, then AMG on p): iterations versus size.

    python tools/config4_sweep.py gpu [EDGES]      # GPU: default plan and global relaxation
    python tools/config4_sweep.py oracle [EDGES]   # CPU oracle: default plan, and every
                                                   # F-relaxation / the coarse solve exact
Each line is one JSON record (rtol 1e-8, GMRES(30)).
"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_1801_08464_b200 import pipeline, synth  # noqa: E402


def gpu(edges):
    from paper_1801_08464_b200 import _lib
    ctx = _lib.ctx()
    for e in edges:
        s = synth.make_config(4, e)
        for gr in (False, True):
            solver = pipeline.SyntheticSolver(rel_tol=1e-8, ctx=ctx, global_relax=gr)
            solver.upload(s)
            rows = []
            for r in range(4):
                solver.setup()
                t_set = ctx.timing().setup_ms
                res = solver.solve(s.rhs)
                if r >= 1:
                    rows.append((t_set, ctx.timing().solve_ms, res.iterations, res.converged))
            su = statistics.median(x[0] for x in rows)
            so = statistics.median(x[1] for x in rows)
            print(json.dumps(dict(where="gpu", edge=e, dofs=s.n, global_relax=gr, iterations=rows[-1][2],
                                  converged=rows[-1][3], setup_ms=round(su, 2), solve_ms=round(so, 2),
                                  dofs_per_s=s.n / ((su + so) / 1e3))), flush=True)
            solver.hier.free()
            solver.a.free()


def oracle(edges):
    import numpy as np
    from oracle import amg as oamg, blockscale, krylov, mgr as omgr, pipeline as opipe
    for e in edges:
        s = synth.make_config(4, e)
        a = opipe.scalar_a(s)
        dinv, ahat = blockscale.block_scale(s)
        fsets = synth.mgr_f_indices(s.b, s.n_cells, order="cell")
        variants = [("default", "amg", "amg", False)]
        if e <= 32:
            variants.append(("all exact", "exact", "exact", False))
            variants.append(("all exact + global relax", "exact", "exact", True))
        for name, fr_kind, coarse, gr in variants:
            fr = omgr.FRelax(fr_kind, **(pipeline.DEFAULT_FRELAX if fr_kind == "amg" else {}))
            plan = [(f, omgr.MgrLevelSpec((), omgr.RpKind.INJECTIVE, fr, global_relax=gr)) for f in fsets]
            cells = np.repeat(np.arange(s.n_cells), s.b) if gr else None
            t0 = time.perf_counter()
            hier = omgr.setup_from_matrix(ahat, plan, oamg.AmgOptions(**pipeline.DEFAULT_AMG),
                                          coarse="exact" if coarse == "exact" else "amg", cells=cells)
            res = krylov.gmres(lambda v: a @ v, lambda v: omgr.mgr_apply(hier, blockscale.prescale(dinv, v)),
                               s.rhs, krylov.GmresOptions(rel_tol=1e-8, restart=30, max_iter=600))
            print(json.dumps(dict(where="oracle", edge=e, dofs=s.n, variant=name, iterations=res.iterations,
                                  converged=bool(res.converged), seconds=round(time.perf_counter() - t0, 1))),
                  flush=True)


if __name__ == "__main__":
    mode = sys.argv[1]
    edges = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8, 12, 16, 24, 32, 48, 64, 96]
    (gpu if mode == "gpu" else oracle)(edges)
