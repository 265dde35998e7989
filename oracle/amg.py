"""Oracle AMG: PMIS + extended(+i) interpolation + L1-Jacobi (test infrastructure).

Drop-in for the reference's ``ncpflow.mgr.amg_mod`` seam (mgr.py:35,
193-201, 274, 305, 339): exposes ``AmgOptions``, ``AmgHierarchy``,
``amg_setup``, ``amg_vcycle`` and ``amg_apply`` with the reference's
signatures, so ``ncpflow.mgr.amg_mod = oracle.amg`` runs the reference MGR
and GMRES on top of this AMG.

Follows ncpflow/amg.py for everything the north star keeps:
  * option validation (amg.py:31-49), zero-diagonal / square checks and
    row-sign normalisation (amg.py:289-301; b is multiplied by row_sign in
    the cycle, amg.py:375-376);
  * strength of connection (amg.py:88-103, restated vectorised);
  * level loop and stop rules (amg.py:304-313): n <= coarse_size_cutoff or
    max_levels; empty C set raises; "no progress" stops;
  * Galerkin operator P^T (A P) with scipy semantics (amg.py:318);
  * V(pre, post) recursion and ``cycles`` (amg.py:355-386);
  * dense LU at the coarsest level when n <= max(cutoff, 200) (amg.py:330-333).
Replaced per the north star (SURVEY.md §8(c) contract, C loops in
oracle/csrc/amg_oracle.c): RS -> PMIS, classical -> extended+i (optional
max_elmts truncation), Gauss-Seidel -> L1-Jacobi.  Deviations, all mirrored
by the GPU path: a strength graph with no strong edge at all counts as "no
progress" (the reference's RS makes every point C there, amg.py:312-313);
a stalled coarsest level of n <= 8192 is solved by dense LU instead of
SuperLU (same solve, different factorisation); larger stalls raise.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import scipy.linalg
import scipy.sparse as sp

from . import clib
from .sparse import CsrMatrix, as_scipy

UNDECIDED, FPOINT, CPOINT = 0, 1, 2
DENSE_STALL_LIMIT = 8192


class AmgSetupError(RuntimeError):
    pass


@dataclass(frozen=True)
class AmgOptions:
    strength_theta: float = 0.25
    max_levels: int = 25
    coarse_size_cutoff: int = 50
    pre_sweeps: int = 1
    post_sweeps: int = 1
    cycles: int = 1
    interpolation: str = "extended"
    coarsening: str = "pmis"
    smoother: str = "l1_jacobi"
    max_elmts: int = 4
    seed: int = 0
    restriction: str = "galerkin"

    def __post_init__(self):
        if not (0.0 < self.strength_theta < 1.0):
            raise ValueError("strength_theta must lie in (0, 1)")
        if self.pre_sweeps < 0 or self.post_sweeps < 0:
            raise ValueError("sweep counts must be nonnegative")
        if self.max_levels < 1 or self.coarse_size_cutoff < 1 or self.cycles < 1:
            raise ValueError("max_levels, coarse_size_cutoff and cycles must be >= 1")
        if self.interpolation != "extended":
            raise ValueError(f"unknown interpolation {self.interpolation!r}")
        if self.coarsening != "pmis":
            raise ValueError(f"unknown coarsening {self.coarsening!r}")
        if self.smoother != "l1_jacobi":
            raise ValueError(f"unknown smoother {self.smoother!r}")
        if self.max_elmts < 0:
            raise ValueError("max_elmts must be >= 0")
        if self.restriction not in ("galerkin", "transpose_interp"):
            raise ValueError(f"unknown restriction {self.restriction!r}")


@dataclass
class AmgLevel:
    a: CsrMatrix
    p: CsrMatrix | None = None
    splitting: np.ndarray | None = None
    l1_inv: np.ndarray | None = None
    _asp: object = None
    _psp: object = None
    _rsp: object = None

    @property
    def n(self):
        return self.a.nrows


@dataclass
class AmgHierarchy:
    levels: list
    options: AmgOptions
    coarse_dense: tuple | None = None
    row_sign: np.ndarray | None = None

    @property
    def n(self):
        return self.levels[0].n

    def level_sizes(self):
        return [lvl.n for lvl in self.levels]

    def operator_complexity(self):
        nnz0 = self.levels[0].a.nnz
        return sum(lvl.a.nnz for lvl in self.levels) / max(nnz0, 1)


def strength_graph(a, theta):
    """Strong-connection mask over the stored pattern (ncpflow/amg.py:88-103).

    cand_ij = -a_ij for negative off-diagonals; rows with no negative
    off-diagonal use |a_ij|; strong iff rowmax > 0 and cand >= theta*rowmax.
    Returns int8 [nnz] aligned with a's entries.
    """
    m = as_scipy(a)
    n = m.shape[0]
    ip, ind, dat = m.indptr, m.indices, m.data
    rows = np.repeat(np.arange(n), np.diff(ip))
    off = ind != rows
    neg = off & (dat < 0.0)
    row_has_neg = np.zeros(n, dtype=bool)
    row_has_neg[rows[neg]] = True
    cand = np.zeros(dat.size)
    cand[neg] = -dat[neg]
    fallback = off & ~row_has_neg[rows]
    cand[fallback] = np.abs(dat[fallback])
    rowmax = np.zeros(n)
    np.maximum.at(rowmax, rows, cand)
    rm = rowmax[rows]
    return ((rm > 0.0) & (cand >= theta * rm)).astype(np.int8)


def pmis(a, strong, seed=0, level=0):
    m = as_scipy(a)
    n = m.shape[0]
    ip, ind = clib.c32(m.indptr), clib.c32(m.indices)
    st = np.ascontiguousarray(strong, dtype=np.int8)
    state = np.zeros(n, dtype=np.int8)
    clib.lib().pmis(n, clib.ptr(ip), clib.ptr(ind), clib.ptr(st), seed, level,
                    clib.ptr(state))
    return state


def extended_interpolation(a, strong, state, max_elmts=0):
    """Extended+i interpolation P (n x nc) per the pinned C loop."""
    m = as_scipy(a)
    n = m.shape[0]
    L = clib.lib()
    ip, ind = clib.c32(m.indptr), clib.c32(m.indices)
    dat = np.ascontiguousarray(m.data, dtype=float)
    st = np.ascontiguousarray(strong, dtype=np.int8)
    sp_ = np.ascontiguousarray(state, dtype=np.int8)
    cnt = np.zeros(n, dtype=np.int32)
    L.ext_interp_count(n, clib.ptr(ip), clib.ptr(ind), clib.ptr(dat), clib.ptr(st),
                       clib.ptr(sp_), int(max_elmts), clib.ptr(cnt))
    pp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(cnt, out=pp[1:])
    pc = np.zeros(int(pp[-1]), dtype=np.int32)
    pv = np.zeros(int(pp[-1]))
    bad = L.ext_interp_fill(n, clib.ptr(ip), clib.ptr(ind), clib.ptr(dat), clib.ptr(st),
                            clib.ptr(sp_), int(max_elmts), clib.ptr(pp), clib.ptr(pc),
                            clib.ptr(pv))
    if bad >= 0:
        raise AmgSetupError(f"extended interpolation hit a zero pivot at row {bad}")
    cmap = np.cumsum(state == CPOINT) - 1
    nc = int(np.sum(state == CPOINT))
    cols = cmap[pc].astype(np.int32) if pc.size else pc
    return CsrMatrix(sp.csr_matrix((pv, cols, pp), shape=(n, nc)))


def l1_row_norms(a):
    m = as_scipy(a)
    return np.asarray(abs(m).sum(axis=1)).ravel()


def _opts_from(opts):
    if opts is None:
        return AmgOptions()
    if isinstance(opts, AmgOptions):
        return opts
    # any object with the reference's field names (e.g. ncpflow.amg.AmgOptions)
    kw = {f: getattr(opts, f) for f in AmgOptions.__dataclass_fields__ if hasattr(opts, f)}
    if kw.get("interpolation") in ("classical", "direct"):
        kw["interpolation"] = "extended"
    return AmgOptions(**kw)


def amg_setup(a, opts=None) -> AmgHierarchy:
    opts = _opts_from(opts)
    m = as_scipy(a)
    if m.shape[0] != m.shape[1]:
        raise AmgSetupError("AMG expects a square operator")
    diag = m.diagonal()
    if np.any(diag == 0.0):
        raise AmgSetupError("AMG expects a nonzero diagonal")
    row_sign = None
    if np.any(diag < 0.0):
        row_sign = np.where(diag < 0.0, -1.0, 1.0)
        m = (sp.diags(row_sign) @ m).tocsr()
    levels = [AmgLevel(a=CsrMatrix(m))]
    while levels[-1].n > opts.coarse_size_cutoff and len(levels) < opts.max_levels:
        cur = levels[-1]
        strong = strength_graph(cur.a, opts.strength_theta)
        if not strong.any():
            break  # no strong connection anywhere: no progress
        state = pmis(cur.a, strong, opts.seed, len(levels) - 1)
        nc = int(np.sum(state == CPOINT))
        if nc == 0:
            raise AmgSetupError("coarsening produced an empty C set")
        if nc == cur.n:
            break
        p = extended_interpolation(cur.a, strong, state, opts.max_elmts)
        if opts.restriction == "galerkin":
            pt = p.m.T.tocsr()
        else:
            # R = (extended+i interpolation of A^T on the same C/F split)^T
            at = CsrMatrix(cur.a.m.T.tocsr())
            pt = extended_interpolation(at, strength_graph(at, opts.strength_theta), state,
                                        opts.max_elmts).m.T.tocsr()
        coarse = CsrMatrix((pt @ (cur.a.m @ p.m)).tocsr())
        cur.p = p
        cur.splitting = state
        cur._psp = p.m
        cur._rsp = pt
        levels.append(AmgLevel(a=coarse))
    hier = AmgHierarchy(levels=levels, options=opts, row_sign=row_sign)
    for lvl in levels[:-1]:
        lvl._asp = lvl.a.m
        lvl.l1_inv = 1.0 / l1_row_norms(lvl.a)
    last = levels[-1]
    last._asp = last.a.m
    if last.n > max(opts.coarse_size_cutoff, 200) and last.n > DENSE_STALL_LIMIT:
        raise AmgSetupError(f"coarsening stalled at n={last.n} (> {DENSE_STALL_LIMIT})")
    hier.coarse_dense = scipy.linalg.lu_factor(last.a.to_dense())
    return hier


def _sweep(level, x, b):
    return x + level.l1_inv * (b - level._asp @ x)


def _vcycle(hier, k, b, x, x_zero):
    level = hier.levels[k]
    if k == len(hier.levels) - 1:
        return scipy.linalg.lu_solve(hier.coarse_dense, b)
    for _ in range(hier.options.pre_sweeps):
        if x_zero:
            x = level.l1_inv * b
            x_zero = False
        else:
            x = _sweep(level, x, b)
    r = b - level._asp @ x if not x_zero else b.copy()
    rc = level._rsp @ r
    ec = _vcycle(hier, k + 1, rc, np.zeros(rc.size), True)
    x = x + level._psp @ ec
    for _ in range(hier.options.post_sweeps):
        x = _sweep(level, x, b)
    return x


def amg_vcycle(hier, b, x0=None):
    b = np.asarray(b, dtype=float)
    if b.shape != (hier.n,):
        raise ValueError("amg_vcycle: dimension mismatch")
    if hier.row_sign is not None:
        b = b * hier.row_sign
    if x0 is None:
        return _vcycle(hier, 0, b, np.zeros(hier.n), True)
    return _vcycle(hier, 0, b, np.array(x0, dtype=float), False)


def amg_apply(hier, b):
    x = amg_vcycle(hier, b)
    for _ in range(hier.options.cycles - 1):
        x = amg_vcycle(hier, b, x)
    return x
