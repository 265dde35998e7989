"""GPU Newton assembly against the reference's
Problem.residual / Problem.jacobian (tests/golden/make_assembly.py)."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "assembly.npz")
CASES = [("vg2d", 0), ("vg2d", 1), ("vg3d_gravity", 0), ("vg3d_gravity", 1), ("pl_linear", 0), ("pl_linear", 1)]


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


class _State:
    def __init__(self, p, s, r):
        self.p_l, self.s_l, self.rho_lh = p, s, r


def states(g, key):
    return (_State(g[key + "_p"], g[key + "_s"], g[key + "_r"]), _State(g[key + "_po"], g[key + "_so"], g[key + "_ro"]),
            float(g[key + "_dt"]))


def test_incidence_order(gold):
    """Per-cell incidence: a-side faces, b-side faces, Neumann, Dirichlet (np.add.at order)."""
    from paper_1801_08464_b200.assembly import AssemblyProblem
    pb = AssemblyProblem.from_arrays(gold, prefix="vg3d_gravity_pb_")
    rp, ent = pb.incidence()
    n, nf = pb.n_cells, pb.face_a.size
    assert rp[-1] == 2 * nf + pb.neu_cell.size + pb.dir_cell.size
    for i in range(n):
        e = ent[rp[i]:rp[i + 1]]
        kinds = [0 if 0 <= x < nf else 1 if x >= (1 << 30) else 2 if x < 0 else 3 for x in e]
        assert kinds == sorted(kinds)
        a_faces = [x for x in e if 0 <= x < nf]
        assert a_faces == sorted(a_faces) and all(pb.face_a[f] == i for f in a_faces)


@pytest.mark.gpu
@pytest.mark.parametrize("case,k", CASES)
def test_residual_and_jacobian(gpu, gold, case, k):
    from paper_1801_08464_b200.assembly import AssemblyProblem, GpuAssembler
    asm = GpuAssembler(AssemblyProblem.from_arrays(gold, prefix=f"{case}_pb_"))
    key = f"{case}_{k}"
    st, old, dt = states(gold, key)
    res = asm.residual(st, old, dt)
    ref = gold[key + "_res"]
    n = len(ref) // 3
    for blk in range(3):  # balance rows and constraint rows have their own scales
        r, q = res[blk * n:(blk + 1) * n], ref[blk * n:(blk + 1) * n]
        assert np.max(np.abs(r - q)) <= 1e-12 * max(np.max(np.abs(q)), 1e-300)
    system = asm.jacobian(st, old, dt)
    ip, ix, v = system.a.download()
    assert np.array_equal(ip, gold[key + "_jac_indptr"]) and np.array_equal(ix, gold[key + "_jac_indices"])
    vr = gold[key + "_jac_data"]
    rows = np.repeat(np.arange(3 * n), np.diff(ip))
    rowmax = np.maximum.reduceat(np.abs(vr), ip[:-1]) if vr.size else vr
    assert np.all(np.abs(v - vr) <= 1e-12 * rowmax[rows] + 1e-300)
    assert np.array_equal(system.active_set.active, gold[key + "_active"])
    assert np.max(np.abs(system.rhs - gold[key + "_rhs"])) <= 1e-12 * np.max(np.abs(gold[key + "_rhs"]))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["vg2d", "pl_linear"])
def test_assemble_then_solve_on_device(gpu, gold, case):
    """The device-assembled Jacobian feeds GmresSolver directly (no host round
    trip); same solution as solving the reference's Jacobian."""
    from paper_1801_08464_b200 import mgr
    from paper_1801_08464_b200.assembly import AssemblyProblem, GpuAssembler
    from paper_1801_08464_b200.krylov import GmresOptions
    from paper_1801_08464_b200.linsolve import GmresSolver
    asm = GpuAssembler(AssemblyProblem.from_arrays(gold, prefix=f"{case}_pb_"))
    key = f"{case}_0"
    st, old, dt = states(gold, key)
    system = asm.jacobian(st, old, dt)
    opts = GmresOptions(rel_tol=1e-10, max_iter=400, restart=30)
    specs = mgr.default_2p2c_specs("gas_appearance")
    r1 = GmresSolver("mgr", opts, mgr_specs=specs).solve(system)
    n = system.n_cells
    ref = sp.csr_matrix((gold[key + "_jac_data"], gold[key + "_jac_indices"], gold[key + "_jac_indptr"]),
                        shape=(3 * n, 3 * n))

    class _Sys:
        a, rhs, n_cells, active_set = ref, gold[key + "_rhs"], n, system.active_set
        labels, cells = system.labels, system.cells

    r2 = GmresSolver("mgr", opts, mgr_specs=specs).solve(_Sys)
    assert r1.converged and r2.converged and abs(r1.iterations - r2.iterations) <= 1
    assert np.linalg.norm(r1.x - r2.x) <= 1e-8 * np.linalg.norm(r2.x)
