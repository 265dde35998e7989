"""GPU drop-in for the reference's linear-solver plugin (ncpflow/linsolve.py:46-122).

``GmresSolver`` keeps the reference constructor (preconditioner, gmres_opts,
mgr_specs, amg_opts, ilu_level, post_smoothing, equilibrate) and
``.solve(system) -> LinearSolveResult`` (linsolve.py:26-31), so Newton
(newton.py:101) can call it unchanged.  Per system, on the device:

  * symmetric infinity-norm equilibration (linsolve.py:107-122,
    ``sparse.equilibrate``; the rhs division and the final column unscaling
    are the reference's own numpy vector operations);
  * the MGR hierarchy from the system's unknown labels
    (``mgr.mgr_setup``, mgr.py:313-333) for 'mgr' (``mgr_specs``) or 'cpr'
    (``mgr.cpr_specs()``); setup failures become ``LinearSolveFailure``
    exactly where the reference converts them (linsolve.py:88-91);
  * ``a_norm`` = max row abs sum of the (scaled) matrix (linsolve.py:97-98)
    and right-preconditioned GMRES with the backward-error acceptance.

preconditioner='ilu' builds the ILU(ilu_level) comparator on the device
(``ilu.ilu_factor``; a zero pivot becomes ``LinearSolveFailure`` as in
linsolve.py:79-83).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .amg import AmgOptions
from .errors import LinearSolveFailure, ZeroFDiagonal, ZeroPivot
from .ilu import IluFactorization, ilu_factor
from .krylov import GmresOptions, gmres
from .mgr import cpr_specs, mgr_setup
from .sparse import DeviceMatrix, abs_row_sum_max, as_device, equilibrate


@dataclass
class LinearSolveResult:
    x: np.ndarray
    iterations: int
    converged: bool
    residual_norm: float


class _ScaledSystem:
    """The BlockSystem surface mgr_setup needs, over a device matrix."""

    def __init__(self, a: DeviceMatrix, system):
        self.a = a
        self._system = system

    def labels(self):
        return self._system.labels()

    def cells(self):
        return self._system.cells()


class GmresSolver:
    """GMRES with a per-system GPU preconditioner (linsolve.py:46-73).

    preconditioner: 'mgr' (uses mgr_specs), 'cpr' (MGR in the CPR-emulation
    configuration), 'ilu' (level ilu_level) or 'none'."""

    def __init__(self, preconditioner="none", gmres_opts: GmresOptions | None = None, mgr_specs=None,
                 amg_opts: AmgOptions | None = None, ilu_level: int = 0, post_smoothing: bool = False,
                 equilibrate: bool = True, ctx=None):
        if preconditioner not in ("mgr", "cpr", "ilu", "none"):
            raise ValueError(f"unknown preconditioner {preconditioner!r}")
        self.preconditioner = preconditioner
        self.gmres_opts = gmres_opts or GmresOptions()
        self.mgr_specs = mgr_specs
        self.amg_opts = amg_opts or AmgOptions(pre_sweeps=2, post_sweeps=2)
        self.ilu_level = ilu_level
        self.post_smoothing = post_smoothing
        self.equilibrate = equilibrate
        self.ctx = ctx or _lib.ctx()
        self.last_hierarchy = None

    def _build_preconditioner(self, system, a: DeviceMatrix):
        if self.preconditioner == "none":
            return None
        if self.preconditioner == "ilu":
            try:
                return ilu_factor(a, self.ilu_level)
            except ZeroPivot as err:
                raise LinearSolveFailure(f"ILU({self.ilu_level}) setup failed: {err}") from err
        specs = self.mgr_specs if self.preconditioner == "mgr" else cpr_specs()
        if specs is None:
            raise ValueError("GmresSolver(preconditioner='mgr') needs mgr_specs")
        if self.last_hierarchy is not None:
            self.last_hierarchy.free()
            self.last_hierarchy = None
        try:
            hier = mgr_setup(_ScaledSystem(a, system), specs, self.amg_opts, post_smoothing=self.post_smoothing)
        except (ZeroFDiagonal, RuntimeError) as err:
            raise LinearSolveFailure(f"MGR setup failed: {err}") from err
        self.last_hierarchy = hier
        return hier

    def solve(self, system) -> LinearSolveResult:
        a = as_device(system.a, ctx=self.ctx) if not isinstance(system.a, DeviceMatrix) else system.a
        rhs = np.asarray(system.rhs, dtype=np.float64)
        col_scale = None
        if self.equilibrate:
            a, row, col_scale = equilibrate(a)
            rhs = rhs / row
        pc = self._build_preconditioner(system, a)
        a_norm = abs_row_sum_max(a)
        result = gmres(a, pc, rhs, self.gmres_opts, a_norm=a_norm)
        x = result.x if col_scale is None else col_scale * result.x
        return LinearSolveResult(x=x, iterations=result.iterations, converged=result.converged,
                                 residual_norm=result.residual_norm)
