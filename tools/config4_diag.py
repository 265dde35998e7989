"""Config-4 convergence diagnosis on the CPU oracle: which component of the
3-level MGR (S, then rho, then AMG on p) loses mesh independence.

    python tools/config4_diag.py EDGE [EDGE ...]
Variants: exact (sparse LU) solves substituted for the F-relaxation AMG of
level 1 / level 2 and for the coarse AMG, one at a time and all together.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from oracle import amg as oamg, blockscale, krylov, mgr as omgr, pipeline as opipe  # noqa: E402
from paper_1801_08464_b200 import pipeline as gpipe, synth  # noqa: E402


def run(s, label, fr_kinds=("amg", "amg"), coarse="amg", amg_kw=None, rtol=1e-8, gr=False):
    a = opipe.scalar_a(s)
    dinv, ahat = blockscale.block_scale(s)
    fsets = synth.mgr_f_indices(s.b, s.n_cells, order="cell")
    plan = []
    for f, k in zip(fsets, fr_kinds):
        fr = omgr.FRelax(k, **(gpipe.DEFAULT_FRELAX if k == "amg" else {}))
        plan.append((f, omgr.MgrLevelSpec((), omgr.RpKind.INJECTIVE if s.b == 3 else omgr.RpKind.NONINJECTIVE, fr,
                                          global_relax=gr)))
    opts = oamg.AmgOptions(**dict(gpipe.DEFAULT_AMG, **(amg_kw or {})))
    t0 = time.perf_counter()
    cells = np.repeat(np.arange(s.n_cells), s.b) if gr else None
    hier = omgr.setup_from_matrix(ahat, plan, opts, coarse=coarse, cells=cells)
    t1 = time.perf_counter()
    res = krylov.gmres(lambda v: a @ v, lambda v: omgr.mgr_apply(hier, blockscale.prescale(dinv, v)), s.rhs,
                       krylov.GmresOptions(rel_tol=rtol, restart=30, max_iter=600))
    t2 = time.perf_counter()
    print(f"{s.nx:3d}^3 {label:18s} its {res.iterations:4d} conv {res.converged} dims {hier.level_dims()} "
          f"setup {t1 - t0:5.1f}s solve {t2 - t1:5.1f}s", flush=True)
    return res.iterations


def main():
    for e in [int(x) for x in sys.argv[1:]]:
        s = synth.make_config(4, e)
        run(s, "base")
        run(s, "coarse exact", coarse="exact")
        run(s, "F1 exact", fr_kinds=("exact", "amg"))
        run(s, "F2 exact", fr_kinds=("amg", "exact"))
        run(s, "F1,F2 exact", fr_kinds=("exact", "exact"))
        run(s, "all exact", fr_kinds=("exact", "exact"), coarse="exact")
        run(s, "coarse V(1,1)", amg_kw=dict(pre_sweeps=1, post_sweeps=1))
        run(s, "global relax", gr=True)


if __name__ == "__main__":
    main()
