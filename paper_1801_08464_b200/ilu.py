"""GPU ILU(k) with the reference's API (ncpflow/ilu.py:53-174).

``ilu_factor(a, level)`` returns an ``IluFactorization`` whose ``matrix`` is the
combined L\\U factor (unit lower diagonal implicit) with the reference's
structural level-of-fill pattern; ``ilu_apply(fact, r)`` runs the forward and
backward substitutions.  Symbolic fill for level >= 1 on the host (row-ordered
closure), numeric IKJ elimination and both substitutions on the device
(csrc/ilu.cu).  A vanishing pivot raises ``ZeroPivot(row)`` for the same row as
the reference (ilu.py:131-140).
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import ZeroPivot  # noqa: F401  (reference name)
from .sparse import DeviceMatrix, as_device


class IluFactorization:
    """Device ILU(k) factors (ilu.py:30-50 surface)."""

    def __init__(self, ctx, handle, n, level):
        self.ctx, self.h, self._n, self.level = ctx, handle, n, level

    @property
    def n(self):
        return self._n

    @property
    def matrix(self) -> DeviceMatrix:
        h = _lib.P()
        self.ctx.call("mg_ilu_matrix", self.h, ctypes.byref(h))
        return DeviceMatrix(self.ctx, h)

    def pattern(self):
        """Set of (row, col) structural positions, for fill-nesting checks."""
        ip, ix, _ = self.matrix.download()
        return {(i, int(j)) for i in range(self.n) for j in ix[ip[i]:ip[i + 1]]}

    def free(self):
        if self.h:
            self.ctx.lib.mg_ilu_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass


def ilu_factor(a, level: int = 0) -> IluFactorization:
    d = as_device(a)
    if d.nrows != d.ncols:
        raise ValueError("ILU expects a square matrix")
    if level < 0:
        raise ValueError("fill level must be nonnegative")
    h = _lib.P()
    d.ctx.call("mg_ilu_factor", d.h, int(level), ctypes.byref(h))
    return IluFactorization(d.ctx, h, d.nrows, int(level))


def ilu_apply(fact: IluFactorization, r) -> np.ndarray:
    """Forward/backward triangular solves on the incomplete factors (ilu.py:166-174)."""
    r = _lib.f64(r)
    if r.shape != (fact.n,):
        raise ValueError("ilu_apply: dimension mismatch")
    x = np.empty_like(r)
    fact.ctx.call("mg_ilu_apply", fact.h, _lib.ptr(r), _lib.ptr(x))
    return x
