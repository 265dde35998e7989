"""GMRES convergence trace, GPU vs oracle, for one synthetic system.

    python tools/gmres_trace.py CFG EDGE [rtol] [gpu|oracle]

GPU: MG_GMRES_TRACE=1 makes solver.cu print |g| per Arnoldi step and the true
residual at each cycle top (stderr).  Oracle: the same quantities from a traced
run of oracle/krylov.py's loop (the reference's krylov.py:44-144).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402


def oracle_trace(s, rtol):
    from oracle import amg as oamg, blockscale, krylov, mgr as omgr, pipeline as opipe
    from paper_1801_08464_b200 import pipeline as gpipe
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    (a, dinv, hier), _ = opipe.setup_synthetic(s, amg_opts=oamg.AmgOptions(**gpipe.DEFAULT_AMG), plan=plan)
    bn = np.linalg.norm(s.rhs)
    hn_log = []
    orig_norm = np.linalg.norm

    def apply_a(v):
        return a @ v

    def apply_m(v):
        return omgr.mgr_apply(hier, blockscale.prescale(dinv, v))
    # re-run with growing max_iter is costly; instead instrument via the |g|
    # recurrence: replay the oracle's loop verbatim with prints
    import inspect
    src = inspect.getsource(krylov.gmres)
    src = src.replace("        res = float(np.linalg.norm(r))\n",
                      "        res = float(np.linalg.norm(r))\n        print(f'[oracle] cycle top: total {total} res {res!r} relres {res / b_norm:.6e}')\n")
    src = src.replace("            happy = hn <= 1e-14 * max(res, 1.0)\n",
                      "            happy = hn <= 1e-14 * max(res, 1.0)\n            print(f'[oracle] it {total} |g| {abs(g[j + 1])!r} hn {hn!r}')\n")
    ns = dict(krylov.__dict__)
    exec(compile(src, "traced_gmres", "exec"), ns)
    r = ns["gmres"](apply_a, apply_m, s.rhs, krylov.GmresOptions(rel_tol=rtol, restart=30, max_iter=400))
    print("oracle iterations", r.iterations, "relres", r.residual_norm / bn)
    return r


def main():
    cfg, edge = int(sys.argv[1]), int(sys.argv[2])
    rtol = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-10
    which = sys.argv[4] if len(sys.argv) > 4 else "both"
    from paper_1801_08464_b200 import synth
    s = synth.make_config(cfg, edge)
    if which in ("both", "oracle"):
        oracle_trace(s, rtol)
    if which in ("both", "gpu"):
        os.environ["MG_GMRES_TRACE"] = "1"
        from paper_1801_08464_b200 import pipeline as gpipe
        for ortho in ("dcgs2", "cgs2"):
            print("GPU", ortho, flush=True)
            rg, _ = gpipe.SyntheticSolver(rel_tol=rtol, orthogonalization=ortho).solve_system(s)
            sys.stderr.flush()
            print("gpu iterations", rg.iterations, "relres", rg.residual_norm / rg.rhs_norm, flush=True)


if __name__ == "__main__":
    main()
