"""GPU parity: AMG setup (strength / PMIS / extended+i / Galerkin) and V-cycle.

Integer outputs (C/F splittings, P and coarse-operator patterns) and — because
the GPU reproduces the oracle's pinned operation order — P and A_l values are
compared bit for bit; V-cycles within 1e-12 relative.  Property tests mirror
the reference's tests/test_amg.py.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from helpers import assert_bitwise, poisson1d, poisson2d, poisson3d, relerr
from oracle import amg as oamg
from oracle import blockscale as obs
from oracle import mgr as omgr
from oracle.sparse import extract as oextract
from paper_1801_08464_b200 import amg as gamg
from paper_1801_08464_b200 import synth
from paper_1801_08464_b200.errors import AmgSetupError

pytestmark = pytest.mark.gpu


def synth_blocks(cfg, edge):
    s = synth.make_config(cfg, edge)
    _, ahat = obs.block_scale(s)
    N = s.n_cells
    f = np.arange(N) * 2 + 1
    c = np.arange(N) * 2
    aff = oextract(ahat, f, f).m
    r, p = omgr.build_rp(ahat, f, c, omgr.RpKind.NONINJECTIVE)
    ac = (r @ (ahat @ p)).tocsr()
    ac.sort_indices()
    return aff, ac


def compare_hierarchies(a, opts_kw):
    oo = oamg.AmgOptions(**opts_kw)
    ho = oamg.amg_setup(a, oo)
    hg = gamg.amg_setup(a, gamg.AmgOptions(**opts_kw))
    assert hg.level_sizes() == ho.level_sizes()
    for k in range(len(ho.levels)):
        assert_bitwise(hg.levels[k].a.to_scipy(), ho.levels[k].a.m)
        if k + 1 < len(ho.levels):
            np.testing.assert_array_equal(hg.levels[k].splitting, ho.levels[k].splitting)
            assert_bitwise(hg.levels[k].p.to_scipy(), ho.levels[k].p.m)
    return ho, hg


MATRICES = {
    "poisson1d": lambda: poisson1d(200),
    "poisson2d": lambda: poisson2d(24),
    "poisson3d_aniso": lambda: poisson3d(10, 0.01),
    "cfg1_aff": lambda: synth_blocks(1, 32)[0],
    "cfg1_ac": lambda: synth_blocks(1, 32)[1],
    "cfg3_aff": lambda: synth_blocks(3, 12)[0],
    "cfg3_ac": lambda: synth_blocks(3, 12)[1],
}


@pytest.mark.parametrize("name", sorted(MATRICES))
@pytest.mark.parametrize("pmax", [0, 4])
def test_hierarchy_bitwise_oracle(gpu, name, pmax):
    a = MATRICES[name]()
    compare_hierarchies(a, dict(max_elmts=pmax, coarse_size_cutoff=20))


@pytest.mark.parametrize("name", ["poisson2d", "cfg1_ac", "cfg3_aff"])
def test_vcycle_matches_oracle(gpu, name):
    a = MATRICES[name]()
    kw = dict(pre_sweeps=2, post_sweeps=2)
    ho, hg = compare_hierarchies(a, kw)
    rng = np.random.default_rng(3)
    b = rng.standard_normal(a.shape[0])
    x0 = rng.standard_normal(a.shape[0])
    assert relerr(gamg.amg_vcycle(hg, b), oamg.amg_vcycle(ho, b)) <= 1e-12
    assert relerr(gamg.amg_vcycle(hg, b, x0), oamg.amg_vcycle(ho, b, x0)) <= 1e-12


def test_negative_rows_normalised(gpu):
    a = poisson2d(16)
    signs = np.where(np.random.default_rng(3).random(a.shape[0]) < 0.5, -1.0, 1.0)
    flipped = (sp.diags(signs) @ a).tocsr()
    ho, hg = compare_hierarchies(flipped, dict(pre_sweeps=1, post_sweeps=1))
    assert hg.row_sign is not None
    np.testing.assert_array_equal(hg.row_sign, signs)
    b = np.random.default_rng(1).standard_normal(a.shape[0])
    assert relerr(gamg.amg_vcycle(hg, b), oamg.amg_vcycle(ho, b)) <= 1e-12


def test_single_level_direct(gpu):
    a = poisson1d(20)
    h = gamg.amg_setup(a, gamg.AmgOptions(coarse_size_cutoff=50))
    assert h.nlevels == 1
    b = np.arange(20.0)
    assert np.max(np.abs(a @ gamg.amg_vcycle(h, b) - b)) < 1e-10


def test_diagonal_matrix_fallback(gpu):
    d = sp.diags(np.linspace(1.0, 3.0, 300)).tocsr()
    h = gamg.amg_setup(d, gamg.AmgOptions())
    x = gamg.amg_vcycle(h, np.ones(300))
    assert np.max(np.abs(d @ x - 1.0)) < 1e-12


def test_zero_diagonal_rejected(gpu):
    with pytest.raises(AmgSetupError):
        gamg.amg_setup(sp.csr_matrix(np.array([[1.0, 2.0], [3.0, 0.0]])))


def test_linear_and_zero(gpu):
    a = poisson2d(12)
    h = gamg.amg_setup(a, gamg.AmgOptions())
    rng = np.random.default_rng(1)
    b1, b2 = rng.standard_normal(a.shape[0]), rng.standard_normal(a.shape[0])
    lhs = gamg.amg_vcycle(h, b1 + b2)
    rhs = gamg.amg_vcycle(h, b1) + gamg.amg_vcycle(h, b2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(np.max(np.abs(rhs)), 1.0)
    np.testing.assert_array_equal(gamg.amg_vcycle(h, np.zeros(a.shape[0])), np.zeros(a.shape[0]))


def test_poisson_reduction_and_cycles(gpu):
    a = poisson2d(32)
    h = gamg.amg_setup(a, gamg.AmgOptions(pre_sweeps=2, post_sweeps=2))
    rng = np.random.default_rng(0)
    b = rng.standard_normal(a.shape[0])
    x = np.zeros(a.shape[0])
    norms = [np.linalg.norm(b)]
    for _ in range(10):
        x = gamg.amg_vcycle(h, b, x)
        norms.append(np.linalg.norm(b - a @ x))
    factors = [norms[i + 1] / norms[i] for i in range(10)]
    assert np.mean(factors) < 0.45
    h3 = gamg.amg_setup(a, gamg.AmgOptions(cycles=3))
    h1 = gamg.amg_setup(a, gamg.AmgOptions(cycles=1))
    r1 = np.linalg.norm(b - a @ gamg.amg_apply(h1, b))
    r3 = np.linalg.norm(b - a @ gamg.amg_apply(h3, b))
    assert r3 < r1 ** 1.5
    assert 1.0 < h.operator_complexity() < 3.5


@pytest.mark.parametrize("n_edge,cut", [(14, 3000), (16, 2000)])
def test_large_dense_coarsest(gpu, n_edge, cut):
    """coarse_size_cutoff in the thousands: the coarsest level is inverted by the
    blocked Gauss-Jordan (dense.cu, n > 256) -- the V-cycle matches the oracle's
    (scipy lu_factor at the coarsest level) within 1e-12."""
    a = poisson3d(n_edge, 0.3)
    kw = dict(coarse_size_cutoff=cut, pre_sweeps=2, post_sweeps=2)
    ho = oamg.amg_setup(a, oamg.AmgOptions(**kw))
    hg = gamg.amg_setup(a, gamg.AmgOptions(**kw))
    assert hg.level_sizes() == ho.level_sizes() and ho.level_sizes()[-1] > 256
    b = np.random.default_rng(3).standard_normal(a.shape[0])
    assert relerr(gamg.amg_vcycle(hg, b), oamg.amg_vcycle(ho, b)) <= 1e-12
    if len(ho.levels) == 1:
        x = gamg.amg_vcycle(hg, b)
        assert np.linalg.norm(a @ x - b) <= 1e-12 * np.linalg.norm(b) * 1e3
