"""Oracle end-to-end wiring for the synthetic configs (test infrastructure only).

The recommended reading of SURVEY.md §8(d) / §7 D2 in the reference API:

    h = setup_from_matrix(Ahat = D^-1 A, plan, AmgOptions(pre=1, post=1, cutoff=2000))
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


def default_post_smoothing(b):
    """MGR sweep order (mgr.py:362-368) of the synthetic pipeline: for the b = 2 configs the
    coarse correction first and the F-relaxation after it (``post_smoothing=True``), for
    b = 3 the reference default (F-relaxation first).  Mirrors
    paper_1801_08464_b200.pipeline.default_post_smoothing."""
    return b == 2


def setup_synthetic(sysm, *, amg_opts=None, rp=None, plan=None, post_smoothing=None):
    """A (scalar CSR, cell-major), the per-cell prescale and the MGR hierarchy on Â."""
    t0 = time.perf_counter()
    a = scalar_a(sysm)
    dinv, ahat = blockscale.block_scale(sysm)
    if plan is None:
        plan = default_plan(sysm.b, sysm.n_cells, rp)
    if post_smoothing is None:
        post_smoothing = default_post_smoothing(sysm.b)
    opts = amg_opts or oamg.AmgOptions(coarse_size_cutoff=2000)
    hier = mgr.setup_from_matrix(CsrMatrix(ahat), plan, opts, post_smoothing=post_smoothing)
    return (a, dinv, hier), time.perf_counter() - t0


# Self-perturbation models (the parity envelope, tests/test_gpu_parity_*.py):
#   "linear": (I + 1e-15 U_a) A and (I + 1e-13 U_m) M^-1 with fixed random diagonals
#             -- a different but fixed operator;
#   "noise":  fresh per-call relative noise of 2e-16 on every A·v element, 1e-15 on
#             every M^-1 element and 1e-14 on the CGS2 projection coefficients --
#             rounding of a different summation order.  Calibrated against the
#             GPU: its M^-1 / A·v differ from the oracle's by 3e-16 / 1.4e-16
#             normwise, and its Arnoldi quantities (h_{j+1,j}, |g|) drift from the
#             oracle's by 1e-11-1e-10 relative by iteration 20 at config 3 10^3, the
#             same drift this model produces (tools/parity_diag.py, gmres_trace.py).
PERTURB_LINEAR = (1e-15, 1e-13)
PERTURB_NOISE = (2e-16, 1e-15, 1e-14)


def gmres_synthetic(state, rhs, *, rel_tol=1e-8, restart=30, max_iter=400, perturb_seed=None,
                    mode="linear", stats=None):
    """GMRES on A with M^-1 v = MGR_Â(D^-1 v); ``perturb_seed`` selects a
    self-perturbation run of the given ``mode`` (see PERTURB_* above)."""
    a, dinv, hier = state
    apply_a = lambda v: a @ v  # noqa: E731
    apply_m = lambda v: mgr.mgr_apply(hier, blockscale.prescale(dinv, v))  # noqa: E731
    coeffs = None
    if perturb_seed is not None:
        rng = np.random.default_rng(perturb_seed)
        fa, fm = apply_a, apply_m
        if mode == "linear":
            n = rhs.size
            sa = 1.0 + PERTURB_LINEAR[0] * rng.uniform(-1.0, 1.0, n)
            sm = 1.0 + PERTURB_LINEAR[1] * rng.uniform(-1.0, 1.0, n)
            apply_a = lambda v: fa(v) * sa  # noqa: E731
            apply_m = lambda v: fm(v) * sm  # noqa: E731
        elif mode == "noise":
            ea, em, ec = PERTURB_NOISE
            apply_a = lambda v: _noisy(fa(v), ea, rng)  # noqa: E731
            apply_m = lambda v: _noisy(fm(v), em, rng)  # noqa: E731
            coeffs = lambda c: _noisy(c, ec, rng)  # noqa: E731
        else:
            raise ValueError(f"unknown perturbation mode {mode!r}")
    return krylov.gmres(apply_a, apply_m, rhs,
                        krylov.GmresOptions(rel_tol=rel_tol, restart=restart, max_iter=max_iter),
                        perturb_coeffs=coeffs, stats=stats)


def _noisy(y, eps, rng):
    return y * (1.0 + eps * rng.uniform(-1.0, 1.0, y.size))


def solve_synthetic(sysm, *, rel_tol=1e-8, restart=30, max_iter=400, amg_opts=None,
                    rp=None, plan=None, perturb_seed=None, post_smoothing=None):
    state, setup_s = setup_synthetic(sysm, amg_opts=amg_opts, rp=rp, plan=plan, post_smoothing=post_smoothing)
    t1 = time.perf_counter()
    res = gmres_synthetic(state, sysm.rhs, rel_tol=rel_tol, restart=restart, max_iter=max_iter,
                          perturb_seed=perturb_seed)
    return res, state[2], dict(setup_s=setup_s, solve_s=time.perf_counter() - t1)


def envelope(sysm, linear_seeds=(1, 2, 3, 4), noise_seeds=(), *, rel_tol=1e-10, amg_opts=None, plan=None,
             restart=30, max_iter=400):
    """The unperturbed oracle solve, then its self-perturbed runs (one setup):
    [unperturbed, linear seeds..., noise seeds...]."""
    state, _ = setup_synthetic(sysm, amg_opts=amg_opts, plan=plan)
    kw = dict(rel_tol=rel_tol, restart=restart, max_iter=max_iter)
    out = [gmres_synthetic(state, sysm.rhs, **kw)]
    out += [gmres_synthetic(state, sysm.rhs, perturb_seed=sd, mode="linear", **kw) for sd in linear_seeds]
    out += [gmres_synthetic(state, sysm.rhs, perturb_seed=sd, mode="noise", **kw) for sd in noise_seeds]
    return out
