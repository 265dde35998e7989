"""Quick GPU exploration: iterations / setup / solve for configs and AMG knobs.

usage: python tools/explore.py CFG EDGE [key=value ...]
keys: theta, pre, post, fpre, fpost, pmax, rp (inj|noninj), rtol
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1801_08464_b200 import _lib, pipeline, synth  # noqa: E402
from paper_1801_08464_b200.amg import AmgOptions  # noqa: E402
from paper_1801_08464_b200.mgr import FRelax, RpKind  # noqa: E402


def run(cfg, edge, kw):
    theta = float(kw.get("theta", 0.25))
    pre, post = int(kw.get("pre", 2)), int(kw.get("post", 2))
    fpre, fpost = int(kw.get("fpre", 2)), int(kw.get("fpost", 2))
    pmax = int(kw.get("pmax", 4))
    rtol = float(kw.get("rtol", 1e-8))
    rp = {"inj": RpKind.INJECTIVE, "noninj": RpKind.NONINJECTIVE}.get(kw.get("rp"), None)
    t = time.perf_counter()
    s = synth.make_config(cfg, edge)
    tg = time.perf_counter() - t
    ctx = _lib.ctx()
    solver = pipeline.SyntheticSolver(rel_tol=rtol, amg_opts=AmgOptions(strength_theta=theta, pre_sweeps=pre,
                                                                          post_sweeps=post, max_elmts=pmax),
                                      rp=rp, frelax=FRelax("amg", pre=fpre, post=fpost))
    solver.upload(s)
    ctx.sync()
    out = []
    for rep in range(2):
        t0 = time.perf_counter()
        solver.setup()
        ctx.sync()
        t1 = time.perf_counter()
        res = solver.solve(s.rhs)
        t2 = time.perf_counter()
        out.append((t1 - t0, t2 - t1, res.iterations, res.converged, res.residual_norm / res.rhs_norm))
    su, so, it, cv, rr = out[-1]
    h = solver.hier
    camg = h.amg(-1)
    famg = h.amg(0)
    print(f"cfg{cfg} {edge}^3 n={s.n} gen={tg:.1f}s its={it} conv={cv} relres={rr:.2e} setup={su*1e3:.1f}ms "
          f"solve={so*1e3:.1f}ms dofs/s={s.n/(su+so):.3e} kw={kw} coarse_levels={camg.level_sizes()[:6]} "
          f"coarse_opc={camg.operator_complexity():.2f} f_levels={len(famg.level_sizes())} "
          f"f_opc={famg.operator_complexity():.2f} dev_mem={ctx.device_bytes/2**30:.2f}GiB", flush=True)


if __name__ == "__main__":
    cfg, edge = int(sys.argv[1]), int(sys.argv[2])
    kw = dict(a.split("=") for a in sys.argv[3:])
    run(cfg, edge, kw)
