"""Oracle end-to-end wiring for the synthetic configs (test infrastructure only).

The recommended reading of SURVEY.md §8(d) / §7 D2 in the reference API:

    h = setup_from_matrix(Ahat = D^-1 A, plan, AmgOptions(pre=2, post=2))
    gmres(lambda v: A @ v, lambda v: mgr_apply(h, Dinv @ v), b, opts)

plan: b=2 [(S, NONINJECTIVE, FRelax('amg', 1, 1))];
      b=3 [(S, INJECTIVE, AMG-F), (rho, INJECTIVE, AMG-F)].
"""
from __future__ import annotations

import time

import numpy as np

from . import amg as oamg
from . import blockscale, krylov, mgr
from .sparse import CsrMatrix


def default_plan(b, N, rp=None, frelax=None):
    import importlib
    synth = importlib.import_module("paper_1801_08464_b200.synth")
    fsets = synth.mgr_f_indices(b, N, order="cell")
    if rp is None:
        rp = mgr.RpKind.NONINJECTIVE if b == 2 else mgr.RpKind.INJECTIVE
    fr = frelax or mgr.FRelax("amg", pre=1, post=1)
    return [(f, mgr.MgrLevelSpec((), rp, fr)) for f in fsets]


def scalar_a(sysm):
    import importlib
    synth = importlib.import_module("paper_1801_08464_b200.synth")
    return synth.to_scalar_csr(sysm, order="cell", drop_zeros=False)


def solve_synthetic(sysm, *, rel_tol=1e-8, restart=30, max_iter=400, amg_opts=None,
                    rp=None, plan=None):
    t0 = time.perf_counter()
    a = scalar_a(sysm)
    dinv, ahat = blockscale.block_scale(sysm)
    if plan is None:
        plan = default_plan(sysm.b, sysm.n_cells, rp)
    opts = amg_opts or oamg.AmgOptions(pre_sweeps=2, post_sweeps=2)
    hier = mgr.setup_from_matrix(CsrMatrix(ahat), plan, opts)
    t1 = time.perf_counter()
    res = krylov.gmres(lambda v: a @ v,
                       lambda v: mgr.mgr_apply(hier, blockscale.prescale(dinv, v)),
                       sysm.rhs, krylov.GmresOptions(rel_tol=rel_tol, restart=restart,
                                                     max_iter=max_iter))
    t2 = time.perf_counter()
    return res, hier, dict(setup_s=t1 - t0, solve_s=t2 - t1)
