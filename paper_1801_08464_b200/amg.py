"""GPU AMG with the reference's API (ncpflow/amg.py:31-49, 289-386).

``amg_setup(a, opts) -> AmgHierarchy``, ``amg_vcycle(hier, b, x0=None)`` and
``amg_apply(hier, b)`` keep the reference signatures, validation and error
types (AmgSetupError on a zero diagonal / empty C set / stalled coarsening,
ValueError on bad options or dimensions).  The algorithms are the ones the
north star names — PMIS coarsening, extended+i interpolation (optional
``max_elmts`` truncation), L1-Jacobi smoothing, dense direct solve on the
coarsest level — as sm_100a kernels (csrc/amg_setup.cu, spgemm.cu,
spmv.cu).  ``AmgOptions`` accepts the reference's fields plus the new knobs;
the reference's ``interpolation='classical'|'direct'`` values are accepted
and mapped to extended+i (the GPU has no RS/classical path).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields

import numpy as np

from . import _lib
from .errors import AmgSetupError  # noqa: F401  (re-exported, reference name)
from .sparse import DeviceMatrix, as_device

UNDECIDED, FPOINT, CPOINT = 0, 1, 2


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

    def __post_init__(self):
        if not (0.0 < self.strength_theta < 1.0):
            raise ValueError("strength_theta must lie in (0, 1)")
        if self.pre_sweeps < 0 or self.post_sweeps < 0:
            raise ValueError("sweep counts must be nonnegative")
        if self.max_levels < 1 or self.coarse_size_cutoff < 1 or self.cycles < 1:
            raise ValueError("max_levels, coarse_size_cutoff and cycles must be >= 1")
        if self.interpolation not in ("extended", "classical", "direct"):
            raise ValueError(f"unknown interpolation {self.interpolation!r}")
        if self.coarsening != "pmis":
            raise ValueError(f"unknown coarsening {self.coarsening!r}")
        if self.smoother != "l1_jacobi":
            raise ValueError(f"unknown smoother {self.smoother!r}")
        if self.max_elmts < 0:
            raise ValueError("max_elmts must be >= 0")

    def to_c(self) -> _lib.AmgOpts:
        return _lib.AmgOpts(float(self.strength_theta), int(self.max_levels), int(self.coarse_size_cutoff),
                            int(self.pre_sweeps), int(self.post_sweeps), int(self.cycles), int(self.max_elmts),
                            int(self.seed) & 0xFFFFFFFFFFFFFFFF)


def as_options(opts) -> AmgOptions:
    """Accept our AmgOptions, the reference's, or None."""
    if opts is None:
        return AmgOptions()
    if isinstance(opts, AmgOptions):
        return opts
    kw = {f.name: getattr(opts, f.name) for f in fields(AmgOptions) if hasattr(opts, f.name)}
    if kw.get("interpolation") in ("classical", "direct"):
        kw["interpolation"] = "extended"
    return AmgOptions(**kw)


class AmgLevelView:
    """Lazy host views of one level (the reference's AmgLevel attributes)."""

    def __init__(self, hier, k):
        self._h, self._k = hier, k

    def _mat(self, what):
        h = _lib.P()
        self._h.ctx.call("mg_amg_level_mat", self._h.h, self._k, what, ctypes.byref(h))
        return DeviceMatrix(self._h.ctx, h)

    @property
    def a(self):
        return self._mat(0)

    @property
    def p(self):
        return self._mat(1) if self._k + 1 < self._h.nlevels else None

    @property
    def splitting(self):
        if self._k + 1 >= self._h.nlevels:
            return None
        s = np.zeros(self.n, dtype=np.int8)
        self._h.ctx.call("mg_amg_splitting", self._h.h, self._k, _lib.ptr(s))
        return s

    @property
    def n(self):
        return self._h.sizes[self._k]


class AmgHierarchy:
    """Handle to a device AMG hierarchy (ncpflow.amg.AmgHierarchy surface)."""

    def __init__(self, ctx, handle, options, owned=True):
        self.ctx, self.h, self.options, self._owned = ctx, handle, options, owned
        nl, hs = ctypes.c_int(), ctypes.c_int()
        ctx.call("mg_amg_nlevels", handle, ctypes.byref(nl), ctypes.byref(hs))
        self.nlevels = nl.value
        self.has_row_sign = bool(hs.value)
        self.levels = [AmgLevelView(self, k) for k in range(self.nlevels)]
        self._sizes = None
        self._nnz = None

    def _stats(self):
        if self._sizes is None:
            sizes, nnz = [], []
            for k in range(self.nlevels):
                m = self.levels[k].a
                sizes.append(m.nrows)
                nnz.append(m.nnz)
                m.free()
            self._sizes, self._nnz = sizes, nnz
        return self._sizes, self._nnz

    @property
    def sizes(self):
        return self._stats()[0]

    @property
    def n(self):
        return self.sizes[0]

    @property
    def row_sign(self):
        if not self.has_row_sign:
            return None
        s = np.empty(self.n)
        self.ctx.call("mg_amg_row_sign", self.h, _lib.ptr(s))
        return s

    def level_sizes(self):
        return list(self.sizes)

    def level_nnz(self):
        return list(self._stats()[1])

    def operator_complexity(self):
        nnz = self._stats()[1]
        return sum(nnz) / max(nnz[0], 1)

    def free(self):
        if self.h:
            self.ctx.lib.mg_amg_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass


def strength_graph(a, theta: float):
    """Strong-connection mask aligned with a's stored entries (amg.py:88-103), on
    the device (mg_strength): returned as the reference does, a scipy CSR of int8
    with a's own pattern."""
    import scipy.sparse as sp
    from .sparse import DeviceMatrix
    d = DeviceMatrix.from_host(a)
    ip, ix, _ = d.download()
    mask = np.zeros(ix.size, dtype=np.int8)
    d.ctx.call("mg_strength", d.h, float(theta), _lib.ptr(mask), None)
    n = ip.size - 1
    return sp.csr_matrix((mask, ix, ip), shape=(n, n))


def amg_setup(a, opts=None) -> AmgHierarchy:
    o = as_options(opts)
    d = as_device(a)
    h = _lib.P()
    c = o.to_c()
    d.ctx.call("mg_amg_setup", d.h, ctypes.byref(c), ctypes.byref(h))
    return AmgHierarchy(d.ctx, h, o)


def amg_vcycle(hier: AmgHierarchy, b, x0=None) -> np.ndarray:
    """One V(pre, post) cycle; a fixed linear operation in (b, x0) (amg.py:370-378)."""
    b = _lib.f64(b)
    if b.shape != (hier.n,):
        raise ValueError("amg_vcycle: dimension mismatch")
    x = np.empty(hier.n)
    if x0 is None:
        hier.ctx.call("mg_amg_vcycle", hier.h, _lib.ptr(b), None, _lib.ptr(x))
    else:
        x0 = _lib.f64(x0)
        hier.ctx.call("mg_amg_vcycle", hier.h, _lib.ptr(b), _lib.ptr(x0), _lib.ptr(x))
    return x


def amg_apply(hier: AmgHierarchy, b) -> np.ndarray:
    """``cycles`` V-cycles from zero (amg.py:381-386)."""
    b = _lib.f64(b)
    if b.shape != (hier.n,):
        raise ValueError("amg_apply: dimension mismatch")
    x = np.empty(hier.n)
    hier.ctx.call("mg_amg_apply", hier.h, _lib.ptr(b), _lib.ptr(x))
    return x
