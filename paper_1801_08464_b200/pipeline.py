"""End-to-end MGR-GMRES on the synthetic block systems (BASELINE.json configs).

The recommended reading of SURVEY.md §8(d) / §7 D2 expressed in the
reference API, all on the GPU:

    Dinv, Ahat = block_scale(A)                      # per-cell inverses (D3)
    h = setup_from_matrix(Ahat, plan, amg_opts)      # MGR on Ahat = D^-1 A
    h.set_prescale(Dinv)                             # M^-1 v = MGR_Ahat(D^-1 v)
    gmres(A, h, b, GmresOptions(rel_tol, restart=30))

plan: b=2 [(S, NONINJECTIVE, AMG-F)]; b=3 [(S, INJECTIVE, AMG-F), (rho, INJECTIVE,
AMG-F)], F indices in the cell-major unknown order.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .amg import AmgOptions
from .krylov import GmresOptions, GmresResult
from .mgr import FRelax, MgrHierarchy, MgrLevelSpec, RpKind, compile_plan, setup_from_matrix
from .sparse import DeviceMatrix, block_scale

# defaults used by bench.py, smoke() and the parity tests (oracle uses the same).
# coarse_size_cutoff 2000 (reference default 50): both AMG hierarchies stop at
# n <= 2000 with an exact dense coarsest solve (amg.py:304-313, 330-336), instead of
# 3-4 more latency-bound levels (F-relaxation AMG 11 -> 7 levels, coarse AMG 8 -> 6
# at 128^3; iterations unchanged there, 51 -> 42 at config 2 64^3).
# pre_sweeps = post_sweeps = 1: the reference's AmgOptions defaults (amg.py:36-37);
# measured at 128^3 config 3 (tools/explore_opts.py, profiles/r02/explore_sweeps.txt):
# V(1,1) 75 its / 134 ms solve against V(2,2) 66 its / 164 ms, and at config 4
# 64^3 209 against 360 iterations (the L1-Jacobi V(2,2) over-smooths the non-M-matrix
# p-Schur complement of the 3-level reduction).
DEFAULT_AMG = dict(strength_theta=0.25, pre_sweeps=1, post_sweeps=1, max_elmts=4, coarse_size_cutoff=2000)
# the reference's own AmgOptions default cutoff, kept for the deep-hierarchy parity tests
REFERENCE_CUTOFF = 50
DEFAULT_FRELAX = dict(pre=1, post=1)


def default_amg_options(**kw) -> AmgOptions:
    d = dict(DEFAULT_AMG)
    d.update(kw)
    return AmgOptions(**d)


def default_post_smoothing(b: int) -> bool:
    """MGR sweep order of the synthetic pipeline (mgr.py:362-368, ``post_smoothing``): for
    the b = 2 configs the coarse correction runs first and the F-relaxation after it (fewer
    GMRES iterations on every b = 2 config and size); b = 3 keeps the
    reference default (F-relaxation first).  The oracle pipeline mirrors this."""
    return b == 2


def default_plan(b: int, n_cells: int, rp=None, frelax: FRelax | None = None, global_relax=False):
    from .synth import mgr_f_indices
    if rp is None:
        rp = RpKind.NONINJECTIVE if b == 2 else RpKind.INJECTIVE
    fr = frelax or FRelax("amg", **DEFAULT_FRELAX)
    return [(f, MgrLevelSpec((), rp, fr, global_relax)) for f in mgr_f_indices(b, n_cells, order="cell")]


@dataclass
class SolveStats:
    setup_ms: float = 0.0
    solve_ms: float = 0.0
    iterations: int = 0
    converged: bool = False
    relres: float = float("nan")
    extra: dict = field(default_factory=dict)


class SyntheticSolver:
    """Upload once, then setup / solve on the device."""

    def __init__(self, rel_tol=1e-8, restart=30, max_iter=400, amg_opts=None, rp=None, frelax=None, ctx=None,
                 orthogonalization="dcgs2", global_relax=False, post_smoothing=None):
        self.ctx = ctx or _lib.ctx()
        self.gopts = GmresOptions(rel_tol=rel_tol, restart=restart, max_iter=max_iter,
                                  orthogonalization=orthogonalization)
        self.amg_opts = amg_opts or default_amg_options()
        self.rp = rp
        self.frelax = frelax
        self.global_relax = global_relax  # per-cell block relaxation on every MGR level (mgr.py:212-251)
        # MGR sweep order (mgr.py:362-368): True = coarse correction, then F-relaxation;
        # None = default_post_smoothing(b)
        self.post_smoothing = post_smoothing
        self.a: DeviceMatrix | None = None
        self.hier: MgrHierarchy | None = None
        self.dinv = None
        self.ahat = None
        self._plan = None

    def upload(self, sysm, asynchronous=False) -> DeviceMatrix:
        """Upload the system's block CSR matrix.  ``asynchronous=True`` copies on the
        context's copy stream (mg_mat_upload_bsr_async) and returns at once: the arrays
        should be pinned (see PinnedSystem) so that the copy overlaps the solve of the
        previous system of a sequence."""
        self.sysm_meta = (sysm.b, sysm.n_cells)
        self.a = DeviceMatrix.from_bsr(sysm.rowptr, sysm.col, sysm.vals, ctx=self.ctx, asynchronous=asynchronous)
        return self.a

    def setup(self, a: DeviceMatrix | None = None, b: int | None = None, n_cells: int | None = None):
        a = a or self.a
        b = b or self.sysm_meta[0]
        n_cells = n_cells or self.sysm_meta[1]
        if self.hier is not None:
            self.hier.free()
            self.hier = None
        for m in (self.dinv, self.ahat):
            if m is not None:
                m.free()
        self.dinv, self.ahat = block_scale(a)
        key = (b, n_cells, a.nrows)
        if self._plan is None or self._plan[0] != key:
            # the plan is an input of the setup (fixed per system shape): built once
            self._plan = (key, compile_plan(default_plan(b, n_cells, self.rp, self.frelax, self.global_relax),
                                            a.nrows))
        cells = np.repeat(np.arange(n_cells, dtype=np.int64), b) if self.global_relax else None
        post = default_post_smoothing(b) if self.post_smoothing is None else self.post_smoothing
        self.hier = setup_from_matrix(self.ahat, self._plan[1], self.amg_opts, cells=cells, post_smoothing=post)
        self.hier.set_prescale(self.dinv)
        # Ahat is copied into the hierarchy; release the standalone copy
        self.ahat.free()
        self.ahat = None
        return self.hier

    def solve(self, rhs) -> GmresResult:
        from .krylov import gmres
        return gmres(self.a, self.hier, rhs, self.gopts)

    def solve_system(self, sysm) -> tuple[GmresResult, SolveStats]:
        t0 = time.perf_counter()
        self.upload(sysm)
        self.setup()
        t1 = time.perf_counter()
        res = self.solve(sysm.rhs)
        t2 = time.perf_counter()
        st = SolveStats(setup_ms=(t1 - t0) * 1e3, solve_ms=(t2 - t1) * 1e3, iterations=res.iterations,
                        converged=res.converged,
                        relres=res.residual_norm / res.rhs_norm if res.rhs_norm else 0.0)
        return res, st


class PinnedSystem:
    """Page-locked host staging for one synthetic system of a sequence (BASELINE config 5:
    20 successive 128^3 systems): the producer writes the next system here while the GPU
    solves the current one, and upload(asynchronous=True) copies it on the copy stream.
    Same fields as synth.BlockSystem as far as SyntheticSolver reads them."""

    def __init__(self, like):
        import torch
        self._keep = []

        def pin(a):
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            self._keep.append(t)
            return t.numpy()

        self.rowptr, self.col, self.vals, self.rhs = pin(like.rowptr), pin(like.col), pin(like.vals), pin(like.rhs)
        self._meta(like)

    def _meta(self, s):
        self.b, self.n_cells, self.n, self.nnzb = s.b, s.n_cells, s.n, s.nnzb

    def load(self, s):
        """Copy another system of the same block pattern size into the pinned arrays."""
        if s.rowptr.shape != self.rowptr.shape or s.col.shape != self.col.shape or s.vals.shape != self.vals.shape:
            raise ValueError("PinnedSystem.load: the system's shape differs from the staging buffers'")
        np.copyto(self.rowptr, s.rowptr)
        np.copyto(self.col, s.col)
        np.copyto(self.vals, s.vals)
        np.copyto(self.rhs, s.rhs)
        self._meta(s)
        return self

