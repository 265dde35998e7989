"""Run-to-run bitwise determinism of the kernels with inter-thread protocols.

A shared-memory race in the hash SpGEMM (hash inserts, the ordered accumulation
of a 32-product window), in the PMIS rounds, in extended+i, in the column-code
bitmap, or a missing acquire / release in the sync-free triangular solve shows up
as results that change between runs of the same input.  Each operation is
repeated and compared bit for bit with its first result, on inputs large enough
to fill every SM (so warps of different blocks interleave differently between
runs).  With MG_LIB=checked (tools/checked_tests.sh) the same tests also run the
device-side bounds / probe / dependency checks of libmgrgpu_checked.so.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from helpers import assert_bitwise, poisson3d, rand_csr
from paper_1801_08464_b200 import amg as gamg
from paper_1801_08464_b200 import mgr as gmgr
from paper_1801_08464_b200 import pipeline as gpipe
from paper_1801_08464_b200 import sparse as gsp
from paper_1801_08464_b200 import synth

pytestmark = pytest.mark.gpu
REPS = 8


def test_spgemm_repeatable(gpu):
    rng = np.random.default_rng(3)
    a = rand_csr(rng, 30000, 30000, 4e-4, diag=1.0)
    b = rand_csr(rng, 30000, 20000, 6e-4)
    da, db = gsp.DeviceMatrix.from_host(a), gsp.DeviceMatrix.from_host(b)
    first = gsp.matmul(da, db).to_scipy()
    assert_bitwise(first, (a @ b).tocsr())
    for _ in range(REPS):
        assert_bitwise(gsp.matmul(da, db).to_scipy(), first)


def test_amg_setup_repeatable(gpu):
    """Strength, PMIS rounds, extended+i (smem and global tables), Galerkin."""
    a = poisson3d(40, 0.05)
    first = gamg.amg_setup(a, gamg.AmgOptions(max_elmts=4))
    for _ in range(REPS // 2):
        h = gamg.amg_setup(a, gamg.AmgOptions(max_elmts=4))
        assert h.level_sizes() == first.level_sizes()
        for k in range(len(first.levels) - 1):
            np.testing.assert_array_equal(h.levels[k].splitting, first.levels[k].splitting)
            assert_bitwise(h.levels[k].p.to_scipy(), first.levels[k].p.to_scipy())
            assert_bitwise(h.levels[k + 1].a.to_scipy(), first.levels[k + 1].a.to_scipy())


def test_gauss_seidel_trisolve_repeatable(gpu):
    """The sync-free forward substitution (atomic row tickets, acquire / release
    ready flags) on a 3D operator with long dependency chains."""
    s = synth.make_config(2, 24)
    d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
    _, ahat = gsp.block_scale(d)
    f = np.arange(s.n_cells) * 2 + 1
    spec = gmgr.MgrLevelSpec((), gmgr.RpKind.INJECTION, gmgr.FRelax("gauss_seidel", sweeps=2))
    h = gmgr.setup_from_matrix(ahat, [(f, spec)], gamg.AmgOptions())
    r = np.random.default_rng(1).standard_normal(s.n)
    e0 = gmgr.mgr_apply(h, r)
    for _ in range(REPS):
        np.testing.assert_array_equal(gmgr.mgr_apply(h, r), e0)


def test_column_codes_repeatable(gpu):
    """Code range / bitmap / dictionary passes (spmv.cu) on a u8-coded SELL copy."""
    a = poisson3d(36)
    x = np.random.default_rng(2).standard_normal(a.shape[0])
    ys = []
    for _ in range(REPS // 2):
        d = gsp.DeviceMatrix.from_host(a)
        assert d.spmv_layout()[1] == 1
        ys.append(gsp.spmv(d, x))
    for y in ys[1:]:
        np.testing.assert_array_equal(y, ys[0])


def test_unsorted_columns_safe(gpu):
    """Unsorted CSR rows (legal in scipy) take the column-code path without an
    out-of-range code: the code range is the min / max over every entry."""
    a = poisson3d(34).tocsr()
    rng = np.random.default_rng(5)
    indices = a.indices.copy()
    data = a.data.copy()
    for r in range(0, a.shape[0], 7):  # reverse every 7th row
        s0, e0 = a.indptr[r], a.indptr[r + 1]
        indices[s0:e0] = indices[s0:e0][::-1]
        data[s0:e0] = data[s0:e0][::-1]
    u = sp.csr_matrix((data, indices, a.indptr), shape=a.shape)
    x = rng.standard_normal(a.shape[0])
    y = gsp.spmv(gsp.DeviceMatrix.from_csr(u.indptr, u.indices, u.data, u.shape), x)
    assert np.max(np.abs(y - a @ x)) <= 1e-13 * np.max(np.abs(a @ x))


def test_full_solve_repeatable(gpu):
    s = synth.make_config(3, 48)
    sol = gpipe.SyntheticSolver(rel_tol=1e-10)
    r0, _ = sol.solve_system(s)
    for _ in range(2):
        r, _ = sol.solve_system(s)
        assert r.iterations == r0.iterations
        np.testing.assert_array_equal(r.x, r0.x)
