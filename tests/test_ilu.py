"""ILU(k) comparator on the GPU against the reference's
ilu_factor / ilu_apply / GmresSolver('ilu') outputs (tests/golden/make_ilu.py),
mirroring the reference's tests/test_ilu.py."""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from test_physics_dropin import BlockSystem

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ilu.npz")
PHYS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "physics.npz")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


@pytest.fixture(scope="module")
def phys():
    return np.load(PHYS)


def csr(g, name):
    m = sp.csr_matrix((g[name + "_data"], g[name + "_indices"], g[name + "_indptr"]),
                      shape=tuple(g[name + "_shape"]))
    m.sort_indices()
    return m


@pytest.mark.gpu
@pytest.mark.parametrize("case", [0, 1, 2])
@pytest.mark.parametrize("level", [0, 1, 2])
def test_ilu_factor_pattern_and_values(gpu, gold, case, level):
    """Combined L\\U: the level-of-fill pattern bit-exact, values to rounding."""
    from paper_1801_08464_b200 import ilu
    f = ilu.ilu_factor(csr(gold, f"r{case}_a"), level)
    ip, ix, v = f.matrix.download()
    ref = csr(gold, f"r{case}_lu{level}")
    assert np.array_equal(ip, ref.indptr) and np.array_equal(ix, ref.indices)
    assert np.max(np.abs(v - ref.data)) <= 1e-12 * np.max(np.abs(ref.data))
    x = ilu.ilu_apply(f, gold[f"r{case}_r"])
    xr = gold[f"r{case}_x{level}"]
    assert np.max(np.abs(x - xr)) <= 1e-12 * np.max(np.abs(xr))


@pytest.mark.gpu
def test_ilu_identity_and_diagonal(gpu):
    from paper_1801_08464_b200 import ilu
    f = ilu.ilu_factor(sp.identity(5, format="csr"), 0)
    assert np.allclose(ilu.ilu_apply(f, np.arange(5.0)), np.arange(5.0))
    f = ilu.ilu_factor(sp.diags([2.0, 4.0, 8.0]).tocsr(), 0)
    assert np.allclose(ilu.ilu_apply(f, np.array([2.0, 4.0, 8.0])), [1.0, 1.0, 1.0])


@pytest.mark.gpu
def test_ilu_full_fill_equals_dense_lu(gpu):
    """Level >= n - 1 closes the pattern: the factor is the exact LU (ilu tests :60-69)."""
    from paper_1801_08464_b200 import ilu
    rng = np.random.default_rng(3)
    n = 12
    a = rng.standard_normal((n, n)) * (rng.random((n, n)) < 0.3)
    np.fill_diagonal(a, np.abs(a).sum(axis=1) + 1.0)
    f = ilu.ilu_factor(sp.csr_matrix(a), n)
    b = rng.standard_normal(n)
    assert np.allclose(ilu.ilu_apply(f, b), np.linalg.solve(a, b), rtol=1e-12, atol=1e-12)


@pytest.mark.gpu
def test_ilu_zero_pivot_rows(gpu):
    from paper_1801_08464_b200 import ilu
    from paper_1801_08464_b200.errors import ZeroPivot
    a = sp.csr_matrix(np.array([[0.0, 1.0], [1.0, 2.0]]))
    with pytest.raises(ZeroPivot) as ei:
        ilu.ilu_factor(a, 0)
    assert ei.value.row == 0
    b = sp.csr_matrix(np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 1.0], [0.0, 1.0, 0.0]]))
    b.eliminate_zeros()  # (2,2) structurally missing
    with pytest.raises(ZeroPivot) as ei:
        ilu.ilu_factor(b, 0)
    assert ei.value.row == 2


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["s3x3", "m12x10", "f12x10", "f8x8x4"])
@pytest.mark.parametrize("level", [0, 1])
def test_gmres_solver_ilu_parity(gpu, gold, phys, name, level):
    """GmresSolver('ilu', ilu_level=k) on reference-assembled Newton systems: iterations +-1 and
    solution 1e-8 at rtol 1e-10, or the reference's LinearSolveFailure (zero pivot)."""
    from paper_1801_08464_b200 import ilu
    from paper_1801_08464_b200.errors import LinearSolveFailure, ZeroPivot
    from paper_1801_08464_b200.krylov import GmresOptions
    from paper_1801_08464_b200.linsolve import GmresSolver
    s = BlockSystem(phys, name)
    if f"{name}_ilu{level}_zero_row" in gold:
        with pytest.raises(ZeroPivot) as ei:
            ilu.ilu_factor(s.a, level)
        assert ei.value.row == int(gold[f"{name}_ilu{level}_zero_row"])
    solver = GmresSolver("ilu", GmresOptions(rel_tol=1e-10, max_iter=400, restart=30), ilu_level=level)
    key = f"{name}_gsilu{level}"
    if key + "_fail" in gold:
        with pytest.raises(LinearSolveFailure):
            solver.solve(s)
        return
    res = solver.solve(s)
    assert bool(res.converged) == bool(gold[key + "_conv"])
    assert abs(res.iterations - int(gold[key + "_its"])) <= 1
    xr = gold[key + "_x"]
    assert np.linalg.norm(res.x - xr) <= 1e-8 * np.linalg.norm(xr)


def test_mm_write_host(tmp_path):
    """write_matrix_market (sparse.py:262-264) from a host matrix (no GPU needed)."""
    import scipy.io
    from paper_1801_08464_b200.sparse import write_matrix_market
    m = sp.random(20, 20, density=0.2, random_state=1, format="csr") + sp.identity(20, format="csr")
    p = tmp_path / "a.mtx"
    write_matrix_market(str(p), m, comment="graft")
    back = sp.csr_matrix(scipy.io.mmread(str(p), spmatrix=False))
    assert abs(back - m).max() == 0.0


@pytest.mark.gpu
def test_mm_roundtrip_device(gpu, tmp_path):
    from paper_1801_08464_b200.sparse import read_matrix_market, write_matrix_market
    m = sp.random(30, 30, density=0.1, random_state=2, format="csr") + sp.identity(30, format="csr")
    m.sort_indices()
    p = tmp_path / "b.mtx"
    write_matrix_market(str(p), m)
    d = read_matrix_market(str(p))
    ip, ix, v = d.download()
    assert np.array_equal(ip, m.indptr) and np.array_equal(ix, m.indices) and np.array_equal(v, m.data)
    import scipy.io
    q = tmp_path / "c.mtx"
    write_matrix_market(str(q), d)
    assert abs(sp.csr_matrix(scipy.io.mmread(str(q), spmatrix=False)) - m).max() == 0.0
