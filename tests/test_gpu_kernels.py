"""GPU parity: sparse kernels, block scaling, build_rp (through the C-ABI).

Mirrors the reference's sparse/MGR unit tests (tests/test_sparse.py:27-116,
tests/test_mgr.py:50-98) with the oracle as the checker; integer outputs and
the scipy-order products are compared bit for bit.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from helpers import assert_bitwise, assert_close_csr, poisson2d, poisson3d, rand_csr, relerr
from oracle import blockscale as obs
from oracle import mgr as omgr
from paper_1801_08464_b200 import mgr as gmgr
from paper_1801_08464_b200 import sparse as gsp
from paper_1801_08464_b200 import synth
from paper_1801_08464_b200.errors import DimensionMismatch, ZeroFDiagonal

pytestmark = pytest.mark.gpu


def test_spmv_identity_and_zero(gpu):
    n = 17
    x = np.arange(n, dtype=float)
    np.testing.assert_array_equal(gsp.spmv(sp.identity(n, format="csr"), x), x)
    np.testing.assert_array_equal(gsp.spmv(sp.csr_matrix((n, n)), x), np.zeros(n))


@pytest.mark.parametrize("seed", range(4))
def test_spmv_matches_scipy(gpu, seed):
    rng = np.random.default_rng(seed)
    for n, m, dens in ((50, 50, 0.2), (300, 200, 0.05), (2000, 2000, 0.03), (5000, 5000, 0.0005)):
        a = rand_csr(rng, n, m, dens)
        x = rng.standard_normal(m)
        assert relerr(gsp.spmv(a, x), a @ x) <= 1e-14


def _stencil_rows(rng, nr, nc, offsets, anchor, lmin=1, lmax=None):
    """Rows of random length (lmin..len(offsets)) over a sorted random subset of
    anchor(row) + offsets, clipped to [0, nc): exercises every SELL tail length."""
    indptr, cols = [0], []
    for r in range(nr):
        k = rng.integers(lmin, (lmax or len(offsets)) + 1)
        c = np.unique(anchor(r) + rng.choice(offsets, size=k, replace=False))
        c = c[(c >= 0) & (c < nc)]
        cols.append(c)
        indptr.append(indptr[-1] + len(c))
    cols = np.concatenate(cols)
    return sp.csr_matrix((rng.standard_normal(len(cols)), cols, np.array(indptr)), shape=(nr, nc))


@pytest.mark.parametrize("case,want_ib", [("stencil", 1), ("r_shape", 1), ("p_shape", 1),
                                          ("band", 2), ("scattered", 4)])
def test_spmv_sell_column_codes_bitwise(gpu, case, want_ib):
    """SELL-32 copies (>= 32768 rows) with u8-dictionary / int16 / int32 columns:
    same entries in the same order, so y is bit-identical to scipy's row sums."""
    rng = np.random.default_rng(7)
    n = 40000
    if case == "stencil":
        a = poisson3d(34)  # 39304 rows, 7 codes
        a.data[:] = rng.standard_normal(a.nnz)
    elif case == "r_shape":  # nc = 2 nr: anchor(row) = 2 row
        a = _stencil_rows(rng, n, 2 * n, np.array([-70, -2, 0, 1, 2, 3, 70, 71]), lambda r: 2 * r)
    elif case == "p_shape":  # nr = 2 nc: anchor(row) = row // 2
        a = _stencil_rows(rng, n, n // 2, np.array([-35, -1, 0, 1, 35]), lambda r: r // 2, lmin=3)
    elif case == "band":  # > 256 distinct codes, all within int16
        a = _stencil_rows(rng, n, n, rng.choice(np.arange(-30000, 30000), 400, replace=False), lambda r: r, 4, 12)
    else:  # columns anywhere: int32
        a = rand_csr(rng, n, n, 12.0 / n)
    a.sort_indices()
    d = gsp.DeviceMatrix.from_host(a)
    assert d.spmv_layout() == (True, want_ib, False)
    x = rng.standard_normal(a.shape[1])
    np.testing.assert_array_equal(gsp.spmv(d, x), a @ x)


def _irregular_rows(rng, n, offsets, lmin, lmax):
    """n x n, row lengths ~U[lmin, lmax] (before merging repeats) drawn from
    row + offsets, vectorised (sizes past the SELL-C-sigma row threshold)."""
    lens = rng.integers(lmin, lmax + 1, n)
    rows = np.repeat(np.arange(n), lens)
    cols = rows + rng.choice(offsets, size=len(rows))
    ok = (cols >= 0) & (cols < n)
    a = sp.coo_matrix((rng.standard_normal(ok.sum()), (rows[ok], cols[ok])), shape=(n, n)).tocsr()
    a.sum_duplicates()
    a.sort_indices()
    return a


@pytest.mark.parametrize("case,want_ib", [("long_band", 2), ("long_dict", 1), ("long_scattered", 4)])
def test_spmv_sorted_sell_bitwise(gpu, case, want_ib):
    """Irregular long rows (SELL padding over its cap in row order) on operators
    with >= 262144 rows get a SELL-C-sigma copy, rows length-sorted inside
    1024-row windows; each row is still summed sequentially by one thread, so y is
    bit-identical to scipy."""
    rng = np.random.default_rng(11)
    n = 300000
    off = {"long_band": rng.choice(np.arange(-30000, 30000), 600, replace=False),
           "long_dict": np.arange(-100, 100) * 37,
           "long_scattered": rng.choice(np.arange(-250000, 250000), 2000, replace=False)}[case]
    a = _irregular_rows(rng, n, off, 10, 60)
    d = gsp.DeviceMatrix.from_host(a)
    assert d.spmv_layout() == (True, want_ib, True)
    x = rng.standard_normal(n)
    np.testing.assert_array_equal(gsp.spmv(d, x), a @ x)
    # below the row threshold no sorted copy is made
    b = a[: 200000, : 200000].tocsr()
    db = gsp.DeviceMatrix.from_host(b)
    assert db.spmv_layout()[2] is False
    assert relerr(gsp.spmv(db, x[:200000]), b @ x[:200000]) <= 1e-14


@pytest.mark.parametrize("case,want_ib", [("short_dict", 1), ("short_band", 2), ("short_scattered", 4)])
def test_spmv_csr_column_codes(gpu, case, want_ib):
    """Large operators left in CSR (< 3 entries per row) carry u8 / int16 column
    codes in CSR order when they fit.  The CSR kernel splits a row over a lane
    group (tree-summed partials), so the bar is the CSR SpMV's 1e-14; a
    mis-decoded column would be an O(1) error."""
    rng = np.random.default_rng(12)
    n = 600000
    off = {"short_dict": rng.integers(-100, 100, n) * 3, "short_band": rng.integers(-30000, 30000, n),
           "short_scattered": rng.integers(-n // 2, n // 2, n)}[case]
    c2 = np.arange(n) + off
    c2 = np.where((c2 >= 0) & (c2 < n), c2, np.arange(n))
    cols = np.stack([np.minimum(np.arange(n), c2), np.maximum(np.arange(n), c2)], 1).ravel()
    a = sp.csr_matrix((rng.standard_normal(2 * n), cols, np.arange(0, 2 * n + 1, 2)), shape=(n, n))
    a.sum_duplicates()
    a.sort_indices()
    d = gsp.DeviceMatrix.from_host(a)
    assert d.spmv_layout() == (False, want_ib, False)
    x = rng.standard_normal(n)
    assert relerr(gsp.spmv(d, x), a @ x) <= 1e-14


def test_spmv_dimension_mismatch(gpu):
    with pytest.raises(DimensionMismatch):
        gsp.spmv(sp.identity(4, format="csr"), np.ones(5))


@pytest.mark.parametrize("cfg,edge", [(1, 16), (2, 8), (3, 10), (4, 8)])
def test_bsr_spmv_matches_scipy(gpu, cfg, edge):
    s = synth.make_config(cfg, edge)
    a = synth.to_scalar_csr(s, "cell", drop_zeros=False)
    d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
    x = np.random.default_rng(cfg).standard_normal(s.n)
    assert relerr(gsp.spmv(d, x), a @ x) <= 1e-14


@pytest.mark.parametrize("cfg,edge", [(2, 32), (4, 32), (3, 40)])
def test_bsell_spmv_matches_scipy(gpu, cfg, edge):
    """The GMRES operator as the benchmarks run it: >= 32768 block rows take the
    block-SELL copy (spmv.cu k_bsell<2|3>, linsolve.py:100's a @ v)."""
    s = synth.make_config(cfg, edge)
    a = synth.to_scalar_csr(s, "cell", drop_zeros=False)
    d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
    assert d.spmv_layout()[0] == 1
    rng = np.random.default_rng(cfg)
    for _ in range(2):
        x = rng.standard_normal(s.n)
        assert relerr(gsp.spmv(d, x), a @ x) <= 1e-14


@pytest.mark.parametrize("cfg,edge", [(1, 16), (2, 10), (4, 8), (3, 40)])
def test_csr_varmajor_to_bsr(gpu, cfg, edge):
    """mg_mat_upload_csr_varmajor: the reference's variable-major
    scalar CSR converted on the device into cell-major block CSR -- the block
    pattern and every block value equal the host-built BCSR of the same system
    (explicit zeros where a block position has no entry), and its SpMV on
    cell-major vectors equals scipy's on variable-major ones."""
    s = synth.make_config(cfg, edge)
    avm = synth.to_scalar_csr(s, "var", drop_zeros=True)
    d = gsp.DeviceMatrix.from_csr_varmajor(avm.indptr, avm.indices, avm.data, s.b)
    rp, ci, v = d.download()
    # host reference: the synthetic generator's own cell-major BCSR restricted to the
    # blocks that hold a nonzero
    ref = synth.to_scalar_csr(s, "cell", drop_zeros=True)
    from paper_1801_08464_b200.sparse import to_cell_major, to_var_major
    x = np.random.default_rng(cfg).standard_normal(s.n)
    y_gpu = gsp.spmv(d, to_cell_major(x, s.b))
    assert relerr(to_var_major(y_gpu, s.b), avm @ x) <= 1e-14
    # the block matrix equals the cell-major scalar matrix entry by entry
    import scipy.sparse as sp
    blocks = np.asarray(v).reshape(-1, s.b, s.b)
    bsr = sp.bsr_matrix((blocks, np.asarray(ci), np.asarray(rp)), shape=(s.n, s.n)).tocsr()
    assert abs(bsr - ref).max() == 0.0
    assert np.all(np.diff(np.asarray(rp)) >= 0) and rp[-1] == len(ci)


def test_async_upload_pipeline(gpu):
    """mg_mat_upload_bsr_async: matrices uploaded on the copy stream while the
    context is busy equal synchronous uploads; an async upload freed before
    any use (the destructor waits for its copies) leaves the pool consistent."""
    import torch
    s = synth.make_config(3, 20)
    rp = torch.from_numpy(np.ascontiguousarray(s.rowptr, dtype=np.int32)).pin_memory().numpy()
    ci = torch.from_numpy(np.ascontiguousarray(s.col, dtype=np.int32)).pin_memory().numpy()
    vals = torch.from_numpy(np.ascontiguousarray(s.vals)).pin_memory().numpy()
    x = np.random.default_rng(5).standard_normal(s.n)
    ref = gsp.spmv(gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals), x)
    unused = gsp.DeviceMatrix.from_bsr(rp, ci, vals, asynchronous=True)
    unused.free()
    nxt = gsp.DeviceMatrix.from_bsr(rp, ci, vals, asynchronous=True)
    for _ in range(3):
        cur, nxt = nxt, gsp.DeviceMatrix.from_bsr(rp, ci, vals, asynchronous=True)
        np.testing.assert_array_equal(gsp.spmv(cur, x), ref)
        ip, ix, v = cur.download()
        np.testing.assert_array_equal(ix, s.col)
        cur.free()
    nxt.free()


@pytest.mark.parametrize("seed", range(6))
def test_spgemm_bitwise_scipy(gpu, seed):
    """csr_matmat order, separate mul/add, exact zeros dropped."""
    rng = np.random.default_rng(100 + seed)
    shapes = [(40, 30, 50, 0.2), (400, 300, 500, 0.02), (300, 300, 300, 0.3), (50, 2000, 50, 0.2)]
    for n, k, m, dens in shapes:
        a = rand_csr(rng, n, k, dens)
        b = rand_csr(rng, k, m, dens)
        got = gsp.matmul(a, b).to_scipy()
        assert_bitwise(got, (a @ b).tocsr())


def test_spgemm_drops_cancellation_zeros(gpu):
    # the behaviour scipy actually has (reference test_sparse.py:111-116 asserts the opposite)
    a = sp.csr_matrix(np.array([[1.0, 1.0], [1.0, -1.0]]))
    b = sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 1.0]]))
    got = gsp.matmul(a, b).to_scipy()
    assert got.nnz == 2
    assert_bitwise(got, (a @ b).tocsr())


def test_triple_product_and_transpose(gpu):
    a = poisson2d(12)
    rng = np.random.default_rng(5)
    p = rand_csr(rng, a.shape[0], 40, 0.05)
    got = gsp.triple_product(p.T.tocsr(), a, p).to_scipy()
    assert_bitwise(got, (p.T.tocsr() @ (a @ p)).tocsr())
    t = gsp.as_device(p).transpose().to_scipy()
    assert_bitwise(t, p.T.tocsr())


def test_extract_keeps_stored_zeros(gpu):
    a = sp.csr_matrix((np.array([1.0, 0.0, 2.0, 3.0]), np.array([0, 1, 1, 2]), np.array([0, 2, 3, 4])),
                      shape=(3, 3))
    got = gsp.extract(a, [0, 2], [1, 2]).to_scipy()
    want = a[[0, 2]][:, [1, 2]].tocsr()
    assert_bitwise(got, want)
    assert got.nnz == 2


@pytest.mark.parametrize("cfg,edge", [(1, 32), (2, 10), (3, 12), (4, 8)])
def test_block_scale_bitwise_oracle(gpu, cfg, edge):
    s = synth.make_config(cfg, edge)
    d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
    dinv_g, ahat_g = gsp.block_scale(d)
    dinv_o, ahat_o = obs.block_scale(s)
    _, _, dv = dinv_g.download()
    np.testing.assert_array_equal(dv.reshape(dinv_o.shape).view(np.int64), dinv_o.view(np.int64))
    assert_bitwise(ahat_g.to_scipy(), ahat_o)
    v = np.random.default_rng(1).standard_normal(s.n)
    np.testing.assert_array_equal(gsp.block_apply(dinv_g, v), obs.prescale(dinv_o, v))


@pytest.mark.parametrize("kind", ["injective", "noninjective", "injection"])
def test_build_rp_bitwise_oracle(gpu, kind):
    rng = np.random.default_rng(0)
    n = 40
    a = rng.standard_normal((n, n)) * 0.3 * (rng.random((n, n)) < 0.3) + np.diag(rng.uniform(2, 4, n))
    A = sp.csr_matrix(a)
    f = np.sort(rng.choice(n, 15, replace=False))
    c = np.setdiff1d(np.arange(n), f)
    r_o, p_o = omgr.build_rp(A, f, c, omgr.RpKind(kind))
    part = type("Part", (), {"f_points": f, "c_points": c})
    r_g, p_g = gmgr.build_rp(A, part, gmgr.RpKind(kind))
    assert_bitwise(r_g.to_scipy(), r_o)
    assert_bitwise(p_g.to_scipy(), p_o)


def test_build_rp_ideal_close(gpu):
    rng = np.random.default_rng(1)
    n = 30
    a = rng.standard_normal((n, n)) * 0.3 + np.diag(rng.uniform(2, 4, n)) * 5
    A = sp.csr_matrix(a)
    f = np.arange(0, n, 3)
    c = np.setdiff1d(np.arange(n), f)
    r_o, p_o = omgr.build_rp(A, f, c, omgr.RpKind.IDEAL)
    part = type("Part", (), {"f_points": f, "c_points": c})
    r_g, p_g = gmgr.build_rp(A, part, gmgr.RpKind.IDEAL)
    assert np.max(np.abs(r_g.to_dense() - r_o.toarray())) < 1e-13
    assert np.max(np.abs(p_g.to_dense() - p_o.toarray())) < 1e-13


def test_build_rp_zero_f_diagonal_raises(gpu):
    a = np.eye(4)
    a[1, 1] = 0.0
    a[1, 2] = 1.0
    a[2, 1] = 1.0
    part = type("Part", (), {"f_points": np.array([0, 1]), "c_points": np.array([2, 3])})
    with pytest.raises(ZeroFDiagonal) as ei:
        gmgr.build_rp(sp.csr_matrix(a), part, gmgr.RpKind.INJECTIVE)
    assert ei.value.row == 1
