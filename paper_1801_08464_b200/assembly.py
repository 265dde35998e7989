"""GPU Newton residual / Jacobian assembly.

Replaces ``ncpflow.assembly.Problem._assemble`` (assembly.py:247-346) and the
COO -> CSR merge of ``CsrMatrix.from_coo`` (sparse.py:88-93): the step right
before the linear solve.  The problem's static geometry (interior faces with
T, T_geo and g.dx, the resolved Neumann / Dirichlet boundary groups, the
constitutive models) is taken from a reference ``Problem`` once
(``AssemblyProblem.from_reference``) or from saved arrays; per Newton step the
device evaluates the constitutive laws, the two-point fluxes, the residual (in
the reference's accumulation order) and the Jacobian triplets, and merges
them into a 3N x 3N CSR that ``linsolve.GmresSolver`` consumes directly.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, fields

import numpy as np

from . import _lib
from .sparse import DeviceMatrix

_B_SIDE = 1 << 30


@dataclass
class AssemblyProblem:
    """Host description of a discrete problem (the ``mg_asm_desc`` fields)."""

    n_cells: int
    cell_volume: float
    phi: float
    diff_lh: float
    mu_l: float
    mu_g: float
    rho_w_std: float
    c_h: float
    c_v: float
    rp_van_genuchten: int
    s_lr: float
    s_gr: float
    rp_m: float
    rp_eps: float
    cp_van_genuchten: int
    p_entry: float
    cp_n: float
    cp_m: float
    cp_eps: float
    face_a: np.ndarray
    face_b: np.ndarray
    trans: np.ndarray
    tgeo: np.ndarray
    gdx: np.ndarray
    dir_cell: np.ndarray
    dir_rule: np.ndarray
    dir_trans: np.ndarray
    dir_tgeo: np.ndarray
    dir_gdx: np.ndarray
    rule_p: np.ndarray
    rule_s: np.ndarray
    rule_rho: np.ndarray
    rule_pc: np.ndarray
    rule_dpc: np.ndarray
    rule_lam_l: np.ndarray
    rule_lam_g: np.ndarray
    neu_cell: np.ndarray
    neu_w: np.ndarray
    neu_h: np.ndarray

    # -- constructors ---------------------------------------------------------
    @classmethod
    def from_reference(cls, problem) -> "AssemblyProblem":
        """Static data of an ``ncpflow.assembly.Problem`` (its constructor already
        resolved the boundary rules and transmissibilities)."""
        from ncpflow import physics as rphys
        grid, prm, rp, cp = problem.grid, problem.params, problem.relperm, problem.capillary
        neu_cell, neu_w, neu_h = [], [], []
        for cells_b, areas, rule in problem.neumann_groups:
            neu_cell.append(np.asarray(cells_b))
            neu_w.append(-rule.w_inflow * np.asarray(areas))
            neu_h.append(-rule.h_inflow * np.asarray(areas))
        d_cell, d_rule, d_t, d_tg, d_g = [], [], [], [], []
        rp_, rs_, rr_, rpc_, rdpc_, rll_, rlg_ = [], [], [], [], [], [], []
        for k, (cells_b, t_b, tgeo_b, gdx_b, rule) in enumerate(problem.dirichlet_groups):
            d_cell.append(np.asarray(cells_b))
            d_rule.append(np.full(len(cells_b), k))
            d_t.append(np.asarray(t_b))
            d_tg.append(np.asarray(tgeo_b))
            d_g.append(np.asarray(gdx_b))
            pc_b, dpc_b = rphys.capillary(rule.s_l, cp, rp)
            krl_b, krg_b, _, _ = rphys.relperm(rule.s_l, rp)
            rp_.append(rule.p_l)
            rs_.append(rule.s_l)
            rr_.append(rule.rho_lh)
            rpc_.append(pc_b)
            rdpc_.append(dpc_b)
            rll_.append(krl_b / prm.mu_l)
            rlg_.append(krg_b / prm.mu_g)
        cat = (lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt))
        return cls(
            n_cells=grid.n_cells, cell_volume=float(problem.cell_vol),
            phi=prm.phi, diff_lh=prm.diff_lh, mu_l=prm.mu_l, mu_g=prm.mu_g, rho_w_std=prm.rho_w_std,
            c_h=prm.c_h, c_v=prm.c_v,
            rp_van_genuchten=int(rp.variant == rphys.VAN_GENUCHTEN), s_lr=rp.s_lr, s_gr=rp.s_gr,
            rp_m=rp.m if rp.variant == rphys.VAN_GENUCHTEN else 0.0, rp_eps=rp.eps,
            cp_van_genuchten=int(cp.variant == rphys.VAN_GENUCHTEN), p_entry=cp.p_entry, cp_n=cp.n,
            cp_m=cp.m if cp.variant == rphys.VAN_GENUCHTEN else 0.0, cp_eps=cp.eps,
            face_a=np.asarray(grid.face_a, np.int32), face_b=np.asarray(grid.face_b, np.int32),
            trans=np.asarray(problem.trans, float), tgeo=np.asarray(problem.tgeo, float),
            gdx=np.asarray(problem.gdx, float),
            dir_cell=cat(d_cell, np.int32), dir_rule=cat(d_rule, np.int32), dir_trans=cat(d_t, float),
            dir_tgeo=cat(d_tg, float), dir_gdx=cat(d_g, float),
            rule_p=np.asarray(rp_, float), rule_s=np.asarray(rs_, float), rule_rho=np.asarray(rr_, float),
            rule_pc=np.asarray(rpc_, float), rule_dpc=np.asarray(rdpc_, float),
            rule_lam_l=np.asarray(rll_, float), rule_lam_g=np.asarray(rlg_, float),
            neu_cell=cat(neu_cell, np.int32), neu_w=cat(neu_w, float), neu_h=cat(neu_h, float))

    def to_arrays(self, prefix=""):
        return {prefix + f.name: np.asarray(getattr(self, f.name)) for f in fields(self)}

    @classmethod
    def from_arrays(cls, d, prefix=""):
        kw = {}
        for f in fields(cls):
            v = d[prefix + f.name]
            kw[f.name] = v if v.ndim else v.item()
        return cls(**kw)

    # -- per-cell incidence in the reference's np.add.at order -----------------
    def incidence(self):
        """Offsets and entries: a-side faces (face order), b-side faces, Neumann
        contributions (group order), Dirichlet faces (group order)."""
        n, nf = self.n_cells, self.face_a.size
        cells = np.concatenate([self.face_a, self.face_b, self.neu_cell, self.dir_cell]).astype(np.int64)
        kind = np.concatenate([np.zeros(nf), np.ones(nf), np.full(self.neu_cell.size, 2),
                               np.full(self.dir_cell.size, 3)]).astype(np.int64)
        ent = np.concatenate([np.arange(nf), np.arange(nf) + _B_SIDE, -1 - np.arange(self.neu_cell.size),
                              nf + np.arange(self.dir_cell.size)]).astype(np.int64)
        order = np.argsort(cells * 4 + kind, kind="stable")
        rp = np.zeros(n + 1, np.int32)
        np.add.at(rp, cells + 1, 1)
        return np.cumsum(rp).astype(np.int32), ent[order].astype(np.int32)


class _Desc(ctypes.Structure):
    _fields_ = ([(nm, ctypes.c_int) for nm in ("n_cells", "n_faces", "n_dirichlet", "n_neumann", "n_rules")]
                + [("cell_volume", ctypes.c_double)]
                + [(nm, ctypes.c_double) for nm in ("phi", "diff_lh", "mu_l", "mu_g", "rho_w_std", "c_h", "c_v")]
                + [("rp_van_genuchten", ctypes.c_int)]
                + [(nm, ctypes.c_double) for nm in ("s_lr", "s_gr", "rp_m", "rp_eps")]
                + [("cp_van_genuchten", ctypes.c_int)]
                + [(nm, ctypes.c_double) for nm in ("p_entry", "cp_n", "cp_m", "cp_eps")]
                + [(nm, ctypes.c_void_p) for nm in (
                    "face_a", "face_b", "trans", "tgeo", "gdx", "dir_cell", "dir_rule", "dir_trans", "dir_tgeo",
                    "dir_gdx", "rule_p", "rule_s", "rule_rho", "rule_pc", "rule_dpc", "rule_lam_l", "rule_lam_g",
                    "inc_rp", "inc_ent", "neu_w", "neu_h")])


@dataclass
class _ActiveSet:
    active: np.ndarray
    inactive: np.ndarray

    @property
    def n(self):
        return self.active.size + self.inactive.size

    @property
    def n_active(self):
        return self.active.size


class AssembledSystem:
    """BlockSystem surface (assembly.py:95-121) with the Jacobian on the device."""

    def __init__(self, a: DeviceMatrix, n_cells, active_set, rhs):
        self.a, self.n_cells, self.active_set, self.rhs = a, n_cells, active_set, rhs

    @property
    def n(self):
        return 3 * self.n_cells

    def labels(self):
        n = self.n_cells
        lab = np.empty(3 * n, dtype=np.int64)
        lab[:n] = 0
        lab[n:2 * n] = 1
        lab[2 * n:] = 3
        lab[2 * n + self.active_set.active] = 2
        return lab

    def cells(self):
        return np.tile(np.arange(self.n_cells), 3)


class GpuAssembler:
    """Device assembly of ``Problem.residual`` / ``Problem.jacobian`` (assembly.py:240-246)."""

    def __init__(self, problem, ctx=None):
        if not isinstance(problem, AssemblyProblem):
            problem = AssemblyProblem.from_reference(problem)
        self.problem = problem
        self.ctx = ctx or _lib.ctx()
        pb = problem
        inc_rp, inc_ent = pb.incidence()
        self._keep = {
            "face_a": np.ascontiguousarray(pb.face_a, np.int32), "face_b": np.ascontiguousarray(pb.face_b, np.int32),
            "trans": _lib.f64(pb.trans), "tgeo": _lib.f64(pb.tgeo), "gdx": _lib.f64(pb.gdx),
            "dir_cell": np.ascontiguousarray(pb.dir_cell, np.int32),
            "dir_rule": np.ascontiguousarray(pb.dir_rule, np.int32),
            "dir_trans": _lib.f64(pb.dir_trans), "dir_tgeo": _lib.f64(pb.dir_tgeo), "dir_gdx": _lib.f64(pb.dir_gdx),
            "rule_p": _lib.f64(pb.rule_p), "rule_s": _lib.f64(pb.rule_s), "rule_rho": _lib.f64(pb.rule_rho),
            "rule_pc": _lib.f64(pb.rule_pc), "rule_dpc": _lib.f64(pb.rule_dpc),
            "rule_lam_l": _lib.f64(pb.rule_lam_l), "rule_lam_g": _lib.f64(pb.rule_lam_g),
            "inc_rp": inc_rp, "inc_ent": inc_ent, "neu_w": _lib.f64(pb.neu_w), "neu_h": _lib.f64(pb.neu_h)}
        d = _Desc()
        d.n_cells, d.n_faces, d.n_dirichlet = pb.n_cells, pb.face_a.size, pb.dir_cell.size
        d.n_neumann, d.n_rules = pb.neu_cell.size, pb.rule_p.size
        for nm in ("cell_volume", "phi", "diff_lh", "mu_l", "mu_g", "rho_w_std", "c_h", "c_v", "s_lr", "s_gr",
                   "rp_m", "rp_eps", "p_entry", "cp_n", "cp_m", "cp_eps"):
            setattr(d, nm, float(getattr(pb, nm)))
        d.rp_van_genuchten, d.cp_van_genuchten = int(pb.rp_van_genuchten), int(pb.cp_van_genuchten)
        for nm, arr in self._keep.items():
            setattr(d, nm, arr.ctypes.data if arr.size else None)
        h = _lib.P()
        self._desc = d
        self.ctx.call("mg_asm_create", ctypes.addressof(d), ctypes.byref(h))
        self.h = h

    def _run(self, state, state_old, dt, want_jac):
        n = self.problem.n_cells
        args = [_lib.f64(x) for x in (state.p_l, state.s_l, state.rho_lh, state_old.p_l, state_old.s_l,
                                      state_old.rho_lh)]
        if any(a.shape != (n,) for a in args):
            raise ValueError("state dimension mismatch")
        if dt <= 0.0:
            raise ValueError("dt must be positive")
        res = np.empty(3 * n)
        act = np.empty(n, dtype=np.int32)
        jac = _lib.P() if want_jac else None
        self.ctx.call("mg_asm_assemble", self.h, *[_lib.ptr(a) for a in args], ctypes.c_double(dt), _lib.ptr(res),
                      _lib.ptr(act), ctypes.byref(jac) if want_jac else None)
        return res, act.astype(bool), jac

    def residual(self, state, state_old, dt) -> np.ndarray:
        return self._run(state, state_old, dt, False)[0]

    def jacobian(self, state, state_old, dt) -> AssembledSystem:
        res, act, jac = self._run(state, state_old, dt, True)
        idx = np.arange(self.problem.n_cells)
        return AssembledSystem(DeviceMatrix(self.ctx, jac), self.problem.n_cells,
                               _ActiveSet(active=idx[act], inactive=idx[~act]), -res)

    def free(self):
        if getattr(self, "h", None):
            self.ctx.lib.mg_asm_free(self.ctx.h, self.h)
            self.h = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass
