"""Golden fixtures for the physics drop-in, from the reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_physics.py

Builds two-phase NCP Newton systems with the reference's own assembly
(ncpflow.assembly.Problem.jacobian on a grid with a mixed gas-present /
gas-absent state, as the reference's tests do) and records the UNMODIFIED
reference's outputs on them:

  * GmresSolver._equilibrated (linsolve.py:107-122): scaled matrix, rhs,
    column scale (bit-exact targets for mg_equilibrate);
  * mgr_setup(default_2p2c_specs('gas_appearance'), coarse='exact'): level
    dimensions and the dense coarse operators (mgr.py:313-333);
  * mgr_apply on the equilibrated system with FRelax('gauss_seidel') levels
    (cpr_specs, the 'unsaturated' preset) and with global relaxation + exact F
    solves;
  * GmresSolver(...).solve(system) for 'mgr' (gas_appearance specs), 'cpr'
    and 'none', with the oracle AMG (PMIS / extended+i / L1-Jacobi) plugged
    into the ncpflow.mgr.amg_mod seam so the algorithms match the GPU path.

tests/test_physics_dropin.py compares the GPU drop-in against these.
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from ncpflow import linsolve as rls  # noqa: E402
from ncpflow import mgr as rmgr  # noqa: E402
from ncpflow import physics  # noqa: E402
from ncpflow.assembly import Problem, State  # noqa: E402
from ncpflow.grid import BoundarySpec, build_grid  # noqa: E402
from ncpflow.krylov import GmresOptions  # noqa: E402

from oracle import amg as oamg  # noqa: E402

RP = physics.RelPermModel(variant=physics.VAN_GENUCHTEN, s_lr=0.01, s_gr=0.0, n=1.54)
CP = physics.CapPressModel(variant=physics.VAN_GENUCHTEN, p_entry=2e6, n=1.54, eps=1e-5)

# (name, nx, ny, nz, seed, fraction of gas-absent cells, dt)
SYSTEMS = [("s3x3", 3, 3, 1, 0, 0.4, 10.0),
           ("s3x3b", 3, 3, 1, 5, 0.4, 10.0),
           ("m12x10", 12, 10, 1, 1, 0.4, 1.0),
           ("f12x10", 12, 10, 1, 1, 0.0, 10.0),     # all gas present: cpr_specs applies
           ("b8x8x4", 8, 8, 4, 2, 0.3, 0.1),
           ("f8x8x4", 8, 8, 4, 2, 0.0, 5.0)]


def block_system(nx, ny, nz, seed, frac_inactive, dt):
    grid = build_grid(nx, ny, nz, 1.0, 1.0, 1.0)
    problem = Problem(grid, physics.FluidParams(), RP, CP, BoundarySpec())
    n = grid.n_cells
    rng = np.random.default_rng(seed)
    p = 1e6 + rng.uniform(-5e4, 5e4, n)
    s = rng.uniform(0.7, 0.9, n)
    inactive = rng.random(n) < frac_inactive
    s[inactive] = 1.0 + rng.uniform(0.0005, 0.002, inactive.sum())
    pc, _ = physics.capillary(s, CP, RP)
    ch = problem.params.c_h
    rho = np.where(inactive, 0.3 * ch * (p + pc), ch * (p + pc) - 3e-4)
    state = State(p, s, rho)
    return problem.jacobian(state, state.copy(), dt)


def put_csr(d, name, m):
    m = sp.csr_matrix(m.m if hasattr(m, "m") else m)
    d[name + "_indptr"] = m.indptr.astype(np.int64)
    d[name + "_indices"] = m.indices.astype(np.int64)
    d[name + "_data"] = m.data
    d[name + "_shape"] = np.array(m.shape)


def main():
    out = {}
    for name, nx, ny, nz, seed, frac, dt in SYSTEMS:
        system = block_system(nx, ny, nz, seed, frac, dt)
        n = system.n_cells
        put_csr(out, f"{name}_a", system.a)
        out[f"{name}_rhs"] = system.rhs
        out[f"{name}_ncells"] = np.array(n)
        out[f"{name}_active"] = np.asarray(system.active_set.active, dtype=np.int64)
        out[f"{name}_inactive"] = np.asarray(system.active_set.inactive, dtype=np.int64)
        rng = np.random.default_rng(100 + seed)
        r = rng.standard_normal(system.n)
        out[f"{name}_r"] = r

        # equilibration (linsolve.py:107-122)
        gs = rls.GmresSolver("none")
        scaled, col_scale = gs._equilibrated(system)
        put_csr(out, f"{name}_eq", scaled.a)
        out[f"{name}_eq_rhs"] = scaled.rhs
        out[f"{name}_eq_colscale"] = col_scale

        # label-based setup, exact coarse: dims + coarse operators
        hier = rmgr.mgr_setup(system, rmgr.default_2p2c_specs("gas_appearance"),
                              oamg.AmgOptions(pre_sweeps=2, post_sweeps=2), coarse="exact")
        out[f"{name}_gas_dims"] = np.array(hier.level_dims(), dtype=np.int64)
        if system.n <= 400:
            for k, lvl in enumerate(hier.levels):
                out[f"{name}_gas_coarse{k}"] = lvl.coarse_a.to_dense()

        # Gauss-Seidel F-relaxation (cpr_specs) and global relaxation + exact F, on the
        # equilibrated system (the raw Newton rows span ~10 orders of magnitude and make
        # the exact coarse solves too ill-conditioned to compare two factorisations)
        try:
            h_cpr = rmgr.mgr_setup(scaled, rmgr.cpr_specs(gs_sweeps=2), oamg.AmgOptions(), coarse="exact")
            out[f"{name}_cpr_e"] = rmgr.mgr_apply(h_cpr, r)
        except rmgr.ZeroFDiagonal as err:  # injection F = all non-pressure rows: zero diagonals occur
            out[f"{name}_cpr_zero_row"] = np.array(err.row)
        specs_g = [rmgr.MgrLevelSpec(rmgr.ACTIVE_CONSTRAINTS, rmgr.RpKind.NONINJECTIVE, rmgr.FRelax("exact"),
                                     global_relax=True),
                   rmgr.MgrLevelSpec(rmgr.SATURATIONS, rmgr.RpKind.NONINJECTIVE, rmgr.FRelax("exact"),
                                     global_relax=True)]
        if system.n <= 400:
            h_g = rmgr.mgr_setup(scaled, specs_g, oamg.AmgOptions(), coarse="exact")
            out[f"{name}_glob_e"] = rmgr.mgr_apply(h_g, r)

        # oracle AMG in the reference seam for everything that builds an AMG
        saved = rmgr.amg_mod
        rmgr.amg_mod = oamg
        try:
            h_u = rmgr.mgr_setup(scaled, rmgr.default_2p2c_specs("unsaturated"),
                                 oamg.AmgOptions(pre_sweeps=2, post_sweeps=2), coarse="exact")
            out[f"{name}_unsat_e"] = rmgr.mgr_apply(h_u, r)
            for pc in ("mgr", "cpr", "none") if system.n <= 100 else ("mgr", "cpr"):
                solver = rls.GmresSolver(pc, GmresOptions(rel_tol=1e-10, max_iter=400, restart=30),
                                         mgr_specs=rmgr.default_2p2c_specs("gas_appearance"),
                                         amg_opts=oamg.AmgOptions(pre_sweeps=2, post_sweeps=2))
                try:
                    res = solver.solve(system)
                except Exception as err:  # noqa: BLE001  (LinearSolveFailure from the setup)
                    out[f"{name}_gs_{pc}_fail"] = np.array(str(err))
                    print(name, pc, "failed:", err)
                    continue
                out[f"{name}_gs_{pc}_x"] = res.x
                out[f"{name}_gs_{pc}_its"] = np.array(res.iterations)
                out[f"{name}_gs_{pc}_conv"] = np.array(bool(res.converged))
                print(name, pc, res.iterations, res.converged, res.residual_norm)
        finally:
            rmgr.amg_mod = saved
    np.savez_compressed(os.path.join(HERE, "physics.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
