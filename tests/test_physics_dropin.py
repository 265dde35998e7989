"""Physics drop-in: GmresSolver / label-based mgr_setup /
presets / Gauss-Seidel F-relaxation / equilibration on two-phase NCP Newton
systems assembled by the reference (tests/golden/make_physics.py).

Mirrors the reference's own physics tests (tests/test_mgr.py:173-310 of
ncpflow) against the recorded outputs of the unmodified reference.
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "physics.npz")
NAMES = ["s3x3", "s3x3b", "m12x10", "f12x10", "b8x8x4", "f8x8x4"]


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def csr(g, name):
    return sp.csr_matrix((g[name + "_data"], g[name + "_indices"], g[name + "_indptr"]),
                         shape=tuple(g[name + "_shape"]))


class ActiveSet:
    def __init__(self, active, inactive):
        self.active, self.inactive = active, inactive

    @property
    def n_active(self):
        return self.active.size


class BlockSystem:
    """The reference BlockSystem surface (assembly.py:95-121) over fixture arrays."""

    def __init__(self, g, name, equilibrated=False):
        self.a = csr(g, name + ("_eq" if equilibrated else "_a"))
        self.rhs = g[name + ("_eq_rhs" if equilibrated else "_rhs")]
        self.n_cells = int(g[name + "_ncells"])
        self.active_set = ActiveSet(g[name + "_active"], g[name + "_inactive"])

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


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# ---- host-side pieces (no GPU) -------------------------------------------------------
def test_presets_catalog():
    from paper_1801_08464_b200 import mgr
    uns = mgr.default_2p2c_specs("unsaturated")
    assert len(uns) == 2 and uns[0].rp is mgr.RpKind.INJECTIVE
    assert uns[0].f_relax == mgr.FRelax("gauss_seidel", sweeps=3)
    gas = mgr.default_2p2c_specs("gas_appearance")
    assert len(gas) == 3 and gas[0].rp is mgr.RpKind.NONINJECTIVE and gas[0].f_relax.kind == "jacobi"
    assert gas[1].f_relax.max_levels == 2
    assert mgr.default_2p2c_specs("box3d") == gas
    with pytest.raises(ValueError):
        mgr.default_2p2c_specs("mystery")
    cpr = mgr.cpr_specs(2)
    assert cpr[0].rp is mgr.RpKind.INJECTION and cpr[0].f_relax == mgr.FRelax("gauss_seidel", sweeps=2)


@pytest.mark.parametrize("name", NAMES)
def test_label_plan_dims(gold, name):
    """The label-based plan (mgr.py:322-331) gives the reference's level dims."""
    from paper_1801_08464_b200 import mgr
    s = BlockSystem(gold, name)
    plan = mgr.label_plan(s.labels(), mgr.default_2p2c_specs("gas_appearance"))
    cp = mgr.compile_plan(plan, s.n)
    assert cp.dims == list(gold[name + "_gas_dims"])


def test_gmres_solver_validation():
    from paper_1801_08464_b200.linsolve import GmresSolver
    with pytest.raises(ValueError):
        GmresSolver("mystery", ctx=object())


# ---- GPU -------------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_equilibrate_bit_exact(gpu, gold, name):
    from paper_1801_08464_b200 import sparse
    s = BlockSystem(gold, name)
    scaled, row, col = sparse.equilibrate(sparse.as_device(s.a))
    ip, ix, vals = scaled.download()
    ref = csr(gold, name + "_eq")
    ref.sort_indices()
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
    assert np.array_equal(vals, ref.data)
    assert np.array_equal(col, gold[name + "_eq_colscale"])
    assert np.array_equal(s.rhs / row, gold[name + "_eq_rhs"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["s3x3", "s3x3b", "m12x10", "f12x10"])
def test_gas_appearance_levels_and_coarse_operators(gpu, gold, name):
    """dims [3n, 3n - m, 2n - m] and pressure-sized coarse (test_mgr.py:190-220)."""
    from paper_1801_08464_b200 import amg, mgr
    s = BlockSystem(gold, name)
    h = mgr.mgr_setup(s, mgr.default_2p2c_specs("gas_appearance"), amg.AmgOptions(pre_sweeps=2, post_sweeps=2),
                      coarse="exact")
    assert h.level_dims() == list(gold[name + "_gas_dims"])
    assert h.level_dims()[-1] == s.n_cells
    for k in range(h.nlevels):
        key = f"{name}_gas_coarse{k}"
        if key not in gold:
            continue
        got = h.level_matrix(k, "coarse_a").to_scipy().toarray()
        assert rel(got, gold[key]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["s3x3", "s3x3b", "m12x10", "f12x10"])
def test_global_relaxation_exact_f_apply(gpu, gold, name):
    """global block relaxation with mixed 2/3-unknown cells + exact F solves."""
    from paper_1801_08464_b200 import amg, mgr
    s = BlockSystem(gold, name, equilibrated=True)
    specs = [mgr.MgrLevelSpec(mgr.ACTIVE_CONSTRAINTS, mgr.RpKind.NONINJECTIVE, mgr.FRelax("exact"),
                              global_relax=True),
             mgr.MgrLevelSpec(mgr.SATURATIONS, mgr.RpKind.NONINJECTIVE, mgr.FRelax("exact"), global_relax=True)]
    h = mgr.mgr_setup(s, specs, amg.AmgOptions(), coarse="exact")
    e = mgr.mgr_apply(h, gold[name + "_r"])
    assert rel(e, gold[name + "_glob_e"]) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_cpr_gauss_seidel_apply(gpu, gold, name):
    """cpr_specs: injection + Gauss-Seidel (2 sweeps) F-relaxation on the device, or
    the reference's ZeroFDiagonal row when an F diagonal vanishes."""
    from paper_1801_08464_b200 import amg, mgr
    from paper_1801_08464_b200.errors import ZeroFDiagonal
    s = BlockSystem(gold, name, equilibrated=True)
    if name + "_cpr_zero_row" in gold:
        with pytest.raises(ZeroFDiagonal) as ei:
            mgr.mgr_setup(s, mgr.cpr_specs(gs_sweeps=2), amg.AmgOptions(), coarse="exact")
        assert ei.value.row == int(gold[name + "_cpr_zero_row"])
        return
    h = mgr.mgr_setup(s, mgr.cpr_specs(gs_sweeps=2), amg.AmgOptions(), coarse="exact")
    e = mgr.mgr_apply(h, gold[name + "_r"])
    # F part = the Gauss-Seidel relaxation itself.  The C (pressure) part is an exact
    # solve with the closed-boundary pressure block (condition ~1e16-1e17 on these
    # all-gas states): two factorisations (and scipy vs SuperLU) disagree there.
    f = np.where(s.labels() != 0)[0]
    assert rel(e[f], gold[name + "_cpr_e"][f]) <= 1e-11


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_unsaturated_preset_apply(gpu, gold, name):
    """'unsaturated': GS(3) on the active constraints, AMG V(0,1) on S (oracle AMG seam)."""
    from paper_1801_08464_b200 import amg, mgr
    s = BlockSystem(gold, name, equilibrated=True)
    h = mgr.mgr_setup(s, mgr.default_2p2c_specs("unsaturated"), amg.AmgOptions(pre_sweeps=2, post_sweeps=2),
                      coarse="exact")
    e = mgr.mgr_apply(h, gold[name + "_r"])
    assert rel(e, gold[name + "_unsat_e"]) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
@pytest.mark.parametrize("pc", ["mgr", "cpr", "none"])
def test_gmres_solver_parity(gpu, gold, name, pc):
    """GmresSolver.solve(system) vs the reference GmresSolver (oracle AMG in the seam):
    iterations +-1, solution within 1e-8 at rtol 1e-10."""
    from paper_1801_08464_b200 import amg, mgr
    from paper_1801_08464_b200.errors import LinearSolveFailure
    from paper_1801_08464_b200.krylov import GmresOptions
    from paper_1801_08464_b200.linsolve import GmresSolver
    s = BlockSystem(gold, name)
    key = f"{name}_gs_{pc}"
    if key + "_its" not in gold and key + "_fail" not in gold:
        pytest.skip("not recorded for this system")
    solver = GmresSolver(pc, GmresOptions(rel_tol=1e-10, max_iter=400, restart=30),
                         mgr_specs=mgr.default_2p2c_specs("gas_appearance"),
                         amg_opts=amg.AmgOptions(pre_sweeps=2, post_sweeps=2))
    if key + "_fail" in gold:
        with pytest.raises(LinearSolveFailure):
            solver.solve(s)
        return
    res = solver.solve(s)
    assert bool(res.converged) == bool(gold[key + "_conv"])
    assert abs(res.iterations - int(gold[key + "_its"])) <= 1
    x_ref = gold[key + "_x"]
    assert np.linalg.norm(res.x - x_ref) <= 1e-8 * np.linalg.norm(x_ref)
