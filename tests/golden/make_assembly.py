"""Golden fixtures for the GPU Newton assembly, from the reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_assembly.py

Problems built with the reference's own classes (grids, fluid parameters,
Van Genuchten / power-law / linear models, Neumann and Dirichlet boundary
rules, gravity on and off) and mixed gas-present / gas-absent states; for each
the UNMODIFIED reference's Problem.residual / Problem.jacobian (residual,
Jacobian CSR, rhs, active set) and the static problem description the GPU
assembler consumes (AssemblyProblem.from_reference).
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from ncpflow import physics  # noqa: E402
from ncpflow.assembly import Problem, State  # noqa: E402
from ncpflow.grid import DIRICHLET, NEUMANN, BoundaryCondition, BoundarySpec, build_grid  # noqa: E402

from paper_1801_08464_b200.assembly import AssemblyProblem  # noqa: E402

VG_RP = physics.RelPermModel(variant=physics.VAN_GENUCHTEN, s_lr=0.01, s_gr=0.0, n=1.54)
VG_CP = physics.CapPressModel(variant=physics.VAN_GENUCHTEN, p_entry=2e6, n=1.54, eps=1e-5)
PL_RP = physics.RelPermModel(variant=physics.POWER_LAW, s_lr=0.05, s_gr=0.02)
LIN_CP = physics.CapPressModel(variant=physics.LINEAR, p_entry=1e5)


def problem(case):
    if case == "vg2d":
        grid = build_grid(6, 5, 1, 60.0, 50.0, 1.0)
        bc = BoundarySpec().add(BoundaryCondition("xmin", kind=NEUMANN, w_inflow=1e-6, h_inflow=2e-7)) \
                           .add(BoundaryCondition("xmax", kind=DIRICHLET, p_l=1e6, s_l=1.0, rho_lh=0.0))
        return Problem(grid, physics.FluidParams(), VG_RP, VG_CP, bc)
    if case == "vg3d_gravity":
        grid = build_grid(5, 4, 4, 10.0, 8.0, 8.0)
        bc = BoundarySpec().add(BoundaryCondition("zmax", kind=DIRICHLET, p_l=1.02e6, s_l=0.95, rho_lh=0.01)) \
                           .add(BoundaryCondition("zmin", kind=NEUMANN, h_inflow=5e-8))
        return Problem(grid, physics.FluidParams(gravity=(0.0, 0.0, -9.81)), VG_RP, VG_CP, bc)
    if case == "pl_linear":
        grid = build_grid(8, 3, 2, 8.0, 3.0, 2.0)
        bc = BoundarySpec().add(BoundaryCondition("ymin", kind=DIRICHLET, p_l=9.9e5, s_l=0.8, rho_lh=0.002))
        return Problem(grid, physics.FluidParams(mu_l=1e-3), PL_RP, LIN_CP, bc)
    raise ValueError(case)


def state_pair(pb, seed):
    n = pb.grid.n_cells
    rng = np.random.default_rng(seed)
    p = 1e6 + rng.uniform(-5e4, 5e4, n)
    s = rng.uniform(0.7, 0.9, n)
    inactive = rng.random(n) < 0.4
    s[inactive] = 1.0 + rng.uniform(0.0005, 0.002, inactive.sum())
    s[rng.random(n) < 0.1] = rng.uniform(0.001, 0.02, None)  # exercise the clamp bands
    pc, _ = physics.capillary(s, pb.capillary, pb.relperm)
    ch = pb.params.c_h
    rho = np.where(inactive, 0.3 * ch * (p + pc), ch * (p + pc) - 3e-4)
    st = State(p, s, rho)
    old = State(p - rng.uniform(0, 1e3, n), np.clip(s - rng.uniform(0, 0.01, n), 0.0, 1.2), rho * 0.99)
    return st, old


def main():
    out = {}
    for case in ("vg2d", "vg3d_gravity", "pl_linear"):
        pb = problem(case)
        ap = AssemblyProblem.from_reference(pb)
        out.update(ap.to_arrays(prefix=f"{case}_pb_"))
        for k, (seed, dt) in enumerate([(1, 10.0), (2, 3600.0)]):
            st, old = state_pair(pb, seed)
            key = f"{case}_{k}"
            for nm, arr in (("p", st.p_l), ("s", st.s_l), ("r", st.rho_lh), ("po", old.p_l), ("so", old.s_l),
                            ("ro", old.rho_lh)):
                out[f"{key}_{nm}"] = np.asarray(arr, float)
            out[f"{key}_dt"] = np.array(dt)
            out[f"{key}_res"] = pb.residual(st, old, dt)
            system = pb.jacobian(st, old, dt)
            m = sp.csr_matrix(system.a.m)
            m.sort_indices()
            out[f"{key}_jac_indptr"] = m.indptr.astype(np.int64)
            out[f"{key}_jac_indices"] = m.indices.astype(np.int64)
            out[f"{key}_jac_data"] = m.data
            out[f"{key}_rhs"] = system.rhs
            out[f"{key}_active"] = np.asarray(system.active_set.active, np.int64)
            print(case, k, "n", pb.grid.n_cells, "nnz", m.nnz, "active", system.active_set.n_active)
    np.savez_compressed(os.path.join(HERE, "assembly.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
