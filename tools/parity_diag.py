"""GPU-vs-oracle diagnostics on one synthetic system (parity investigations).

    python tools/parity_diag.py CFG EDGE

Reports the normwise / elementwise differences of the preconditioner apply
(M^-1 v = MGR_Â(D^-1 v)) and of A·v between the GPU and the oracle, the GPU's
determinism and linearity defect, and the GMRES iteration counts.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402


def main():
    cfg, edge = int(sys.argv[1]), int(sys.argv[2])
    from oracle import amg as oamg, blockscale, mgr as omgr, pipeline as opipe
    from paper_1801_08464_b200 import pipeline as gpipe, synth, sparse as gsp, mgr as gmgr
    s = synth.make_config(cfg, edge)
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    (a, dinv, hier), _ = opipe.setup_synthetic(s, amg_opts=oamg.AmgOptions(**gpipe.DEFAULT_AMG), plan=plan)
    sol = gpipe.SyntheticSolver(rel_tol=1e-10)
    d = sol.upload(s)
    sol.setup()
    h = sol.hier
    rng = np.random.default_rng(0)
    for t in range(3):
        v = rng.standard_normal(s.n)
        mo = omgr.mgr_apply(hier, blockscale.prescale(dinv, v))
        mg = gmgr.mgr_apply(h, v)
        mg2 = gmgr.mgr_apply(h, v)
        rel = np.linalg.norm(mg - mo) / np.linalg.norm(mo)
        el = np.max(np.abs(mg - mo) / np.maximum(np.abs(mo), 1e-300 + np.max(np.abs(mo)) * 1e-6))
        ao, ag = a @ v, gsp.spmv(d, v)
        print(f"M^-1: normwise {rel:.2e} elementwise(max, floored) {el:.2e} deterministic {np.array_equal(mg, mg2)}; "
              f"A v: normwise {np.linalg.norm(ag - ao) / np.linalg.norm(ao):.2e} bitwise {np.array_equal(ag, ao)}")
        w = rng.standard_normal(s.n)
        lin = gmgr.mgr_apply(h, v + w) - gmgr.mgr_apply(h, v) - gmgr.mgr_apply(h, w)
        lino = omgr.mgr_apply(hier, blockscale.prescale(dinv, v + w)) - mo - omgr.mgr_apply(hier, blockscale.prescale(dinv, w))
        print(f"  linearity defect GPU {np.linalg.norm(lin) / np.linalg.norm(mg):.2e} oracle {np.linalg.norm(lino) / np.linalg.norm(mo):.2e}")
    # hierarchy-level comparisons of the dense coarsest solves
    for k in range(len(hier.levels)):
        fo = hier.levels[k].f_solver.hier
        print("F-relax AMG sizes", fo.level_sizes())
    print("coarse AMG sizes", hier.coarse_amg.level_sizes())


if __name__ == "__main__":
    main()
