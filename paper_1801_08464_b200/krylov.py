"""GPU restarted right-preconditioned GMRES with the reference's API (ncpflow/krylov.py).

``gmres(apply_a, apply_m, b, opts, a_norm=None)`` keeps the reference's
signature and control flow (CGS2, Givens, happy breakdown, true-residual
restarts, optional backward-error acceptance; krylov.py:44-144) but runs the
whole Arnoldi loop on the device (csrc/solver.cu).  ``apply_a`` must be a
matrix (a ``DeviceMatrix`` or any host CSR / ``ncpflow.sparse.CsrMatrix``,
uploaded once) and ``apply_m`` an ``MgrHierarchy`` or ``None``: an arbitrary
Python callable cannot run on the GPU and raises ``TypeError`` rather than
falling back to the CPU.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .mgr import MgrHierarchy
from .sparse import DeviceMatrix, as_device


@dataclass(frozen=True)
class GmresOptions:
    rel_tol: float = 1e-12
    max_iter: int = 400
    restart: int = 30
    reorthogonalize: bool = True
    check_every: int = 25
    # GPU-only knob (not in the reference schema): how the CGS2 of krylov.py:101-107
    # runs.  "dcgs2": one-reduction CGS2 with delayed reorthogonalisation (two basis
    # passes per step); "cgs2": the reference's two full projection passes.
    orthogonalization: str = "dcgs2"

    def __post_init__(self):
        if self.rel_tol <= 0.0:
            raise ValueError("rel_tol must be positive")
        if self.restart < 1 or self.max_iter < 1:
            raise ValueError("restart and max_iter must be at least 1")
        if self.orthogonalization not in ("dcgs2", "cgs2"):
            raise ValueError(f"unknown orthogonalization {self.orthogonalization!r}")

    def to_c(self):
        reorth = 0 if not self.reorthogonalize else (2 if self.orthogonalization == "cgs2" else 1)
        return _lib.GmresOpts(float(self.rel_tol), int(self.max_iter), int(self.restart), reorth,
                              int(self.check_every or 0))


@dataclass
class GmresResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_norm: float
    rhs_norm: float
    cycles: int = 0                   # GPU extra: restart cycles run
    first_cycle_iterations: int = -1  # GPU extra: iterations when the first cycle ended


def _as_operator(apply_a) -> DeviceMatrix:
    if isinstance(apply_a, DeviceMatrix):
        return apply_a
    if hasattr(apply_a, "m") or hasattr(apply_a, "tocsr"):
        return as_device(apply_a)
    raise TypeError("gmres on the GPU needs the operator as a matrix (DeviceMatrix, scipy sparse or "
                    "ncpflow CsrMatrix); a Python callable cannot run on the device")


def _as_precond(apply_m):
    from .ilu import IluFactorization
    if apply_m is None or isinstance(apply_m, (MgrHierarchy, IluFactorization)):
        return apply_m
    raise TypeError("gmres on the GPU needs apply_m to be an MgrHierarchy or IluFactorization (or None); a "
                    "Python callable cannot run on the device")


def gmres(apply_a, apply_m, b, opts: GmresOptions = GmresOptions(), a_norm: float | None = None) -> GmresResult:
    a = _as_operator(apply_a)
    m = _as_precond(apply_m)
    b = _lib.f64(b)
    if b.shape != (a.nrows,):
        raise ValueError("gmres: dimension mismatch")
    if not isinstance(opts, GmresOptions):
        opts = GmresOptions(**{k: getattr(opts, k) for k in GmresOptions.__dataclass_fields__ if hasattr(opts, k)})
    x = np.empty_like(b)
    res = _lib.GmresRes()
    c = opts.to_c()
    from .ilu import IluFactorization
    if isinstance(m, IluFactorization):
        a.ctx.call("mg_gmres_ilu", a.h, m.h, _lib.ptr(b), _lib.ptr(x), ctypes.byref(c),
                   -1.0 if a_norm is None else float(a_norm), ctypes.byref(res))
    else:
        a.ctx.call("mg_gmres", a.h, None if m is None else m.h, _lib.ptr(b), _lib.ptr(x), ctypes.byref(c),
                   -1.0 if a_norm is None else float(a_norm), ctypes.byref(res))
    return GmresResult(x, int(res.iterations), bool(res.converged), float(res.residual_norm),
                       float(res.rhs_norm), int(res.cycles), int(res.first_cycle_iterations))
