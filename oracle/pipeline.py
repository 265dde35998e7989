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


def setup_synthetic(sysm, *, amg_opts=None, rp=None, plan=None):
    """A (scalar CSR, cell-major), the per-cell prescale and the MGR hierarchy on Â."""
    t0 = time.perf_counter()
    a = scalar_a(sysm)
    dinv, ahat = blockscale.block_scale(sysm)
    if plan is None:
        plan = default_plan(sysm.b, sysm.n_cells, rp)
    opts = amg_opts or oamg.AmgOptions(pre_sweeps=2, post_sweeps=2)
    hier = mgr.setup_from_matrix(CsrMatrix(ahat), plan, opts)
    return (a, dinv, hier), time.perf_counter() - t0


def gmres_synthetic(state, rhs, *, rel_tol=1e-8, restart=30, max_iter=400, perturb_seed=None,
                    perturb=(1e-15, 1e-13)):
    """GMRES on A with M^-1 v = MGR_Â(D^-1 v).  ``perturb_seed`` (self-perturbation
    runs, the parity envelope of tests/test_gpu_parity_sweep.py): the operators
    become (I + perturb[0]·U_a)·A and (I + perturb[1]·U_m)·M^-1 with fixed diagonal
    U_a, U_m ~ U[-1, 1) drawn once from ``np.random.default_rng(perturb_seed)`` —
    rounding-sized changes of the kind a different (equally valid) summation
    order makes.  The perturbed operators stay linear and deterministic, as the
    GPU's are: a fresh random perturbation per call would make M^-1 non-linear,
    so the solution GMRES assembles (M^-1 applied to V y, krylov.py:92-94) would
    stop matching the Arnoldi relation and force extra restarts."""
    a, dinv, hier = state
    apply_a = lambda v: a @ v  # noqa: E731
    apply_m = lambda v: mgr.mgr_apply(hier, blockscale.prescale(dinv, v))  # noqa: E731
    if perturb_seed is not None:
        rng = np.random.default_rng(perturb_seed)
        n = rhs.size
        sa = 1.0 + perturb[0] * rng.uniform(-1.0, 1.0, n)
        sm = 1.0 + perturb[1] * rng.uniform(-1.0, 1.0, n)
        fa, fm = apply_a, apply_m
        apply_a = lambda v: fa(v) * sa  # noqa: E731
        apply_m = lambda v: fm(v) * sm  # noqa: E731
    return krylov.gmres(apply_a, apply_m, rhs,
                        krylov.GmresOptions(rel_tol=rel_tol, restart=restart, max_iter=max_iter))


def solve_synthetic(sysm, *, rel_tol=1e-8, restart=30, max_iter=400, amg_opts=None,
                    rp=None, plan=None, perturb_seed=None):
    state, setup_s = setup_synthetic(sysm, amg_opts=amg_opts, rp=rp, plan=plan)
    t1 = time.perf_counter()
    res = gmres_synthetic(state, sysm.rhs, rel_tol=rel_tol, restart=restart, max_iter=max_iter,
                          perturb_seed=perturb_seed)
    return res, state[2], dict(setup_s=setup_s, solve_s=time.perf_counter() - t1)


def envelope(sysm, seeds=(1, 2, 3, 4), *, rel_tol=1e-10, amg_opts=None, plan=None, restart=30,
             max_iter=400):
    """Iteration counts of the unperturbed oracle and of its self-perturbed runs
    (one setup, len(seeds) + 1 GMRES solves): [unperturbed, seed 1, ...]."""
    state, _ = setup_synthetic(sysm, amg_opts=amg_opts, plan=plan)
    out = [gmres_synthetic(state, sysm.rhs, rel_tol=rel_tol, restart=restart, max_iter=max_iter)]
    for sd in seeds:
        out.append(gmres_synthetic(state, sysm.rhs, rel_tol=rel_tol, restart=restart, max_iter=max_iter,
                                   perturb_seed=sd))
    return out

