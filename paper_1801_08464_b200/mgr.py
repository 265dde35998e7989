"""GPU MGR preconditioner with the reference's API (ncpflow/mgr.py).

Same schema as the reference: ``RpKind`` (:47-51), ``FRelax`` (:54-68),
``MgrLevelSpec`` (:71-78) and level plans of ``(f_idx, spec)`` pairs in
current-level local indices (:265-310).  ``setup_from_matrix`` /
``mgr_apply`` / ``build_rp`` keep the reference signatures, skip rules
(|F| in {0, n}) and errors (``ZeroFDiagonal(row)`` from the D_ff check,
including RpKind.INJECTION as the reference does at :132-135).  The
reference's own spec objects (ncpflow.mgr.MgrLevelSpec / FRelax / RpKind)
are accepted too (duck-typed by field names / enum value).

Deviation (SURVEY.md §7 hard part viii, mirrored by oracle/mgr.py): the
F-relaxation AMG keeps every AmgOptions field except those FRelax overrides
(the reference's _AmgF drops ``interpolation``, mgr.py:193-197).
FRelax('gauss_seidel') runs a sync-free forward substitution with tril(A_ff)
on the device (csrc/trisolve.cu; the reference uses SuperLU, mgr.py:175-188).
'exact' / IDEAL / coarse='exact' and a coarsest AMG level use dense inverses
and are limited to 8192 unknowns.

The label-based ``mgr_setup(system, specs)`` (mgr.py:313-333) and the scenario
presets ``default_2p2c_specs`` / ``cpr_specs`` (mgr.py:380-427) are mirrored
for the physics drop-in (``linsolve.GmresSolver``).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from enum import Enum

import numpy as np

from . import _lib
from .amg import AmgHierarchy, as_options
from .errors import ZeroFDiagonal  # noqa: F401  (reference name)
from .sparse import DeviceMatrix, as_device


class RpKind(Enum):
    INJECTIVE = "injective"
    NONINJECTIVE = "noninjective"
    INJECTION = "injection"
    IDEAL = "ideal"


_RP_CODE = {"injective": 0, "noninjective": 1, "injection": 2, "ideal": 3}
_FR_CODE = {"jacobi": 0, "gauss_seidel": 1, "amg": 2, "exact": 3}


@dataclass(frozen=True)
class FRelax:
    kind: str = "jacobi"
    sweeps: int = 1
    pre: int = 1
    post: int = 1
    max_levels: int = 0

    def __post_init__(self):
        if self.kind not in _FR_CODE:
            raise ValueError(f"unknown F-relaxation {self.kind!r}")
        if self.sweeps < 1:
            raise ValueError("sweeps must be >= 1")


@dataclass(frozen=True)
class MgrLevelSpec:
    f_labels: tuple = ()
    rp: RpKind = RpKind.INJECTIVE
    f_relax: FRelax = field(default_factory=FRelax)
    global_relax: bool = False


def _rp_code(kind) -> int:
    v = kind.value if hasattr(kind, "value") else kind
    if v not in _RP_CODE:
        raise ValueError(f"unknown RpKind {kind!r}")
    return _RP_CODE[v]


class MgrHierarchy:
    """Handle to a device MGR hierarchy (ncpflow.mgr.MgrHierarchy surface)."""

    def __init__(self, ctx, handle, n, dims, coarse_kind, post_smoothing, a_ref=None):
        self.ctx, self.h, self.n = ctx, handle, n
        self._dims = dims
        self.coarse_kind = coarse_kind
        self.post_smoothing = post_smoothing
        self._a_ref = a_ref
        self._prescale = None

    @property
    def nlevels(self):
        return len(self._dims) - 1

    def level_dims(self):
        return list(self._dims)

    def level_matrix(self, level, what="a") -> DeviceMatrix:
        code = {"a": 0, "r": 1, "p": 2, "coarse_a": 3, "a_ff": 4}[what]
        h = _lib.P()
        self.ctx.call("mg_mgr_level_mat", self.h, int(level), code, ctypes.byref(h))
        return DeviceMatrix(self.ctx, h)

    def coarse_operator(self) -> DeviceMatrix:
        if not self.nlevels:
            raise ValueError("empty hierarchy")
        return self.level_matrix(self.nlevels - 1, "coarse_a")

    def amg(self, level=-1) -> AmgHierarchy:
        """F-relaxation AMG of ``level`` (or the bottom coarse AMG for -1)."""
        h = _lib.P()
        self.ctx.call("mg_mgr_level_amg", self.h, int(level), ctypes.byref(h))
        return AmgHierarchy(self.ctx, h, None, owned=False)

    def set_prescale(self, dinv: DeviceMatrix):
        """apply becomes MGR(Dinv v)."""
        self.ctx.call("mg_mgr_set_prescale", self.h, dinv.h)
        self._prescale = dinv

    def free(self):
        if self.h:
            self.ctx.lib.mg_mgr_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass


def build_rp(a, part, kind):
    """(R, P) device matrices (mgr.py:117-156); ``part`` has ``f_points`` / ``c_points``."""
    d = as_device(a)
    f = np.asarray(part.f_points, dtype=np.int64)
    c = np.asarray(part.c_points, dtype=np.int64)
    if f.size == 0 or c.size == 0:
        raise ValueError("both F and C sets must be nonempty")
    mask = np.zeros(d.nrows, dtype=np.uint8)
    mask[f] = 1
    r, p = _lib.P(), _lib.P()
    d.ctx.call("mg_build_rp", d.h, _lib.ptr(mask), _rp_code(kind), ctypes.byref(r), ctypes.byref(p))
    return DeviceMatrix(d.ctx, r), DeviceMatrix(d.ctx, p)


def compile_plan(level_plan, n0: int):
    """Host side of setup_from_matrix: (f_idx, spec) pairs -> per-level F masks,
    C level specs and level dims.  Reusable across setups of the same plan."""
    specs, masks = [], []
    cur_n = n0
    dims = []
    for f_idx, spec in level_plan:
        f_idx = np.asarray(f_idx, dtype=np.int64)
        mask = np.zeros(cur_n, dtype=np.uint8)
        if f_idx.size:
            mask[f_idx] = 1
        fr = spec.f_relax
        if fr.kind not in _FR_CODE:
            raise ValueError(f"unknown F-relaxation {fr.kind!r}")
        masks.append(mask)
        specs.append(_lib.LevelSpec(_lib.ptr(mask), _rp_code(spec.rp), _FR_CODE[fr.kind], int(fr.sweeps),
                                    int(fr.pre), int(fr.post), int(fr.max_levels), int(bool(spec.global_relax))))
        nf = int(mask.sum())
        if 0 < nf < cur_n:
            dims.append(cur_n)
            cur_n -= nf
    dims.append(cur_n)
    arr = (_lib.LevelSpec * max(len(specs), 1))(*specs)
    return CompiledPlan(n0, masks, arr, len(specs), dims)


@dataclass
class CompiledPlan:
    n0: int
    masks: list
    specs: object
    nspecs: int
    dims: list


def setup_from_matrix(a, level_plan, amg_opts=None, *, coarse="amg", post_smoothing=False,
                      cells=None) -> MgrHierarchy:
    """Generic MGR setup from (f_indices, spec) pairs (mgr.py:265-310), on the GPU.

    ``level_plan`` may also be a ``CompiledPlan`` (``compile_plan``) to skip the
    host-side mask construction when the same plan is set up repeatedly."""
    if coarse not in ("amg", "exact"):
        raise ValueError(f"unknown coarse solver {coarse!r}")
    d = as_device(a)
    n0 = d.nrows
    opts = as_options(amg_opts)
    cp = level_plan if isinstance(level_plan, CompiledPlan) else compile_plan(level_plan, n0)
    if cp.n0 != n0:
        raise ValueError("setup_from_matrix: plan compiled for a different dimension")
    dims = cp.dims
    c_opts = opts.to_c()
    cells_arr = None if cells is None else _lib.i64(cells)
    h = _lib.P()
    d.ctx.call("mg_mgr_setup", d.h, cp.specs, cp.nspecs, ctypes.byref(c_opts), 0 if coarse == "amg" else 1,
               int(bool(post_smoothing)), None if cells_arr is None else _lib.ptr(cells_arr), ctypes.byref(h))
    return MgrHierarchy(d.ctx, h, n0, dims, coarse, post_smoothing, a_ref=d)


def mgr_apply(hier: MgrHierarchy, r) -> np.ndarray:
    """One multiplicative MGR sweep; linear and deterministic in r (mgr.py:372-377)."""
    r = _lib.f64(r)
    if r.shape != (hier.n,):
        raise ValueError("mgr_apply: dimension mismatch")
    e = np.empty(hier.n)
    hier.ctx.call("mg_mgr_apply", hier.h, _lib.ptr(r), _lib.ptr(e))
    return e


# -- label-based setup and scenario presets (mgr.py:313-333, 380-427) ---------
# unknown labels of a BlockSystem (assembly.py:32-35)
LABEL_P, LABEL_S, LABEL_RHO_ACTIVE, LABEL_RHO_INACTIVE = 0, 1, 2, 3
ACTIVE_CONSTRAINTS = (LABEL_RHO_ACTIVE,)
SATURATIONS = (LABEL_S,)
INACTIVE_CONSTRAINTS = (LABEL_RHO_INACTIVE,)
NON_PRESSURE = (LABEL_S, LABEL_RHO_ACTIVE, LABEL_RHO_INACTIVE)


def label_plan(labels, specs):
    """(f_idx, spec) pairs from unknown labels (mgr.py:322-331): each spec takes the
    current level's unknowns whose label is in ``spec.f_labels``; the labels of
    surviving C points carry down, and a spec matching nothing (or everything)
    is kept in the plan and skipped by the setup."""
    plan = []
    remaining = np.asarray(labels)
    for spec in specs:
        f_idx = np.where(np.isin(remaining, spec.f_labels))[0]
        plan.append((f_idx, spec))
        if 0 < f_idx.size < remaining.size:
            keep = np.ones(remaining.size, dtype=bool)
            keep[f_idx] = False
            remaining = remaining[keep]
    return plan


def mgr_setup(system, specs, amg_opts=None, *, coarse="amg", post_smoothing=False) -> MgrHierarchy:
    """Reduction hierarchy for a two-phase NCP block system (mgr.py:313-333).

    ``system`` is duck-typed like ncpflow's BlockSystem: ``.a`` (CsrMatrix,
    scipy sparse or DeviceMatrix), ``.labels()`` and ``.cells()``."""
    plan = label_plan(system.labels(), specs)
    return setup_from_matrix(system.a, plan, amg_opts, coarse=coarse, post_smoothing=post_smoothing,
                             cells=system.cells())


def default_2p2c_specs(scenario_kind: str):
    """Per-scenario reduction configuration (mgr.py:388-416), same data."""
    if scenario_kind == "unsaturated":
        return [
            MgrLevelSpec(ACTIVE_CONSTRAINTS, RpKind.INJECTIVE, FRelax("gauss_seidel", sweeps=3)),
            MgrLevelSpec(SATURATIONS, RpKind.INJECTIVE, FRelax("amg", pre=0, post=1)),
        ]
    if scenario_kind in ("gas_appearance", "box3d"):
        return [
            MgrLevelSpec(ACTIVE_CONSTRAINTS, RpKind.NONINJECTIVE, FRelax("jacobi", sweeps=1)),
            MgrLevelSpec(SATURATIONS, RpKind.NONINJECTIVE, FRelax("amg", pre=1, post=1, max_levels=2)),
            MgrLevelSpec(INACTIVE_CONSTRAINTS, RpKind.NONINJECTIVE, FRelax("amg", pre=1, post=1, max_levels=2)),
        ]
    raise ValueError(f"no default MGR configuration for scenario {scenario_kind!r}")


def cpr_specs(gs_sweeps: int = 1):
    """CPR-AMG emulation (mgr.py:419-427): every non-pressure unknown an F point,
    pure injection transfers, Gauss-Seidel F-relaxation."""
    return [MgrLevelSpec(NON_PRESSURE, RpKind.INJECTION, FRelax("gauss_seidel", sweeps=gs_sweeps))]
