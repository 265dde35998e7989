"""Oracle checks on the CPU: against the live reference (build container) and
against the algorithm contracts the reference has no implementation of
(PMIS / extended+i / L1-Jacobi)."""
import numpy as np
import pytest
import scipy.sparse as sp

from helpers import assert_bitwise, poisson1d, poisson2d, poisson3d, relerr
from oracle import amg as oamg
from oracle import blockscale as obs
from oracle import krylov as okr
from oracle import mgr as omgr
from oracle import pipeline as opipe
from oracle import sparse as osp
from paper_1801_08464_b200 import pipeline as gpipe
from paper_1801_08464_b200 import synth


# ------------------------------------------------------------------ vs the live reference
def test_strength_matches_reference(ncpflow):
    from ncpflow.amg import strength_graph
    from ncpflow.sparse import CsrMatrix
    rng = np.random.default_rng(0)
    for m in (poisson2d(10), sp.random(80, 80, 0.1, random_state=1, data_rvs=rng.standard_normal).tocsr()
              + sp.identity(80)):
        m = sp.csr_matrix(m)
        m.sort_indices()
        for th in (0.25, 0.6):
            np.testing.assert_array_equal(oamg.strength_graph(m, th), strength_graph(CsrMatrix(m), th).data)


def test_spgemm_c_matches_scipy_order():
    rng = np.random.default_rng(2)
    for _ in range(10):
        a = sp.random(70, 60, 0.1, random_state=int(rng.integers(1 << 30)), data_rvs=rng.standard_normal).tocsr()
        b = sp.random(60, 80, 0.1, random_state=int(rng.integers(1 << 30)), data_rvs=rng.standard_normal).tocsr()
        assert_bitwise(osp.spgemm_c(a, b).m, (a @ b).tocsr())


@pytest.mark.parametrize("post", [False, True])
@pytest.mark.parametrize("cfg,edge", [(1, 16), (2, 6), (4, 5)])
def test_reference_mgr_with_oracle_amg_seam(ncpflow, cfg, edge, post, monkeypatch):
    """The reference's own MGR + GMRES with the oracle AMG plugged into the
    ``ncpflow.mgr.amg_mod`` seam reproduces the oracle pipeline exactly, in both MGR
    sweep orders (``post_smoothing``, mgr.py:362-368)."""
    import ncpflow.krylov as rkr
    import ncpflow.mgr as rmgr
    from ncpflow.sparse import CsrMatrix
    monkeypatch.setattr(rmgr, "amg_mod", oamg)
    s = synth.make_config(cfg, edge)
    a = opipe.scalar_a(s)
    g, ahat = obs.block_scale(s)
    rp = rmgr.RpKind.NONINJECTIVE if s.b == 2 else rmgr.RpKind.INJECTIVE
    # FRelax V(1,1) == the reference _AmgF rebuild (which keeps pre/post/cycles/theta/levels/cutoff)
    plan = [(f, rmgr.MgrLevelSpec((), rp, rmgr.FRelax("amg", pre=1, post=1)))
            for f in synth.mgr_f_indices(s.b, s.n_cells)]
    opts = oamg.AmgOptions(pre_sweeps=2, post_sweeps=2)
    h = rmgr.setup_from_matrix(CsrMatrix(ahat), plan, opts, post_smoothing=post)
    rref = rkr.gmres(lambda v: a @ v, lambda v: rmgr.mgr_apply(h, obs.prescale(g, v)), s.rhs,
                     rkr.GmresOptions(rel_tol=1e-10))
    plan_o = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", pre=1, post=1))
    ro, ho, _ = opipe.solve_synthetic(s, rel_tol=1e-10, plan=plan_o, amg_opts=opts, post_smoothing=post)
    assert ro.iterations == rref.iterations
    assert relerr(ro.x, rref.x) <= 1e-12
    for lr, lo in zip(h.levels, ho.levels):
        assert_bitwise(lo.coarse_a, lr.coarse_a.m)


def test_gmres_matches_reference(ncpflow):
    import ncpflow.krylov as rkr
    rng = np.random.default_rng(7)
    n = 120
    a = rng.standard_normal((n, n)) * 0.3 + np.diag(rng.uniform(2, 4, n)) * 3
    b = rng.standard_normal(n)
    for kw in (dict(rel_tol=1e-10), dict(rel_tol=1e-9, restart=7), dict(rel_tol=1e-6, check_every=3)):
        an = float(np.max(np.abs(a).sum(axis=1))) if "check_every" in kw else None
        r1 = rkr.gmres(lambda v: a @ v, None, b, rkr.GmresOptions(**kw), a_norm=an)
        r2 = okr.gmres(lambda v: a @ v, None, b, okr.GmresOptions(**kw), a_norm=an)
        assert r1.iterations == r2.iterations
        np.testing.assert_array_equal(r1.x, r2.x)


# ------------------------------------------------------------------ algorithm contracts
def test_pmis_is_independent_and_maximal():
    for m in (poisson2d(30), poisson3d(10), poisson3d(10, 0.01)):
        s = oamg.strength_graph(m, 0.25)
        st = oamg.pmis(m, s, seed=3)
        assert set(np.unique(st)) <= {1, 2}
        rows = np.repeat(np.arange(m.shape[0]), np.diff(m.indptr))
        strong = (s == 1) & (m.indices != rows)
        # independence: no strong edge between two C points
        assert not np.any((st[rows] == 2) & (st[m.indices] == 2) & strong)
        # every F point with a strong influencer count > 0 has a C in S_i or was forced F
        has_c = np.zeros(m.shape[0], bool)
        np.logical_or.at(has_c, rows[strong & (st[m.indices] == 2)], True)
        tcount = np.bincount(m.indices[strong], minlength=m.shape[0])
        assert np.all(has_c | (st == 2) | (tcount == 0))


def test_pmis_deterministic_in_seed():
    m = poisson2d(25)
    s = oamg.strength_graph(m, 0.25)
    np.testing.assert_array_equal(oamg.pmis(m, s, 1), oamg.pmis(m, s, 1))
    assert not np.array_equal(oamg.pmis(m, s, 1), oamg.pmis(m, s, 2))


def test_extended_interp_preserves_constants_on_zero_row_sum():
    n = 64
    e = np.ones(n)
    a = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1]).tolil()
    a[0, 0] = 1.0
    a[n - 1, n - 1] = 1.0
    a = a.tocsr()
    a2 = (sp.kron(a, sp.identity(8)) + sp.kron(sp.identity(n), sp.diags([-np.ones(7), 2 * np.ones(8),
                                                                          -np.ones(7)], [-1, 0, 1]).tolil()))
    for m in (a, poisson2d(20) - sp.diags(np.asarray(poisson2d(20).sum(axis=1)).ravel())):
        m = sp.csr_matrix(m)
        s = oamg.strength_graph(m, 0.25)
        st = oamg.pmis(m, s)
        p = oamg.extended_interpolation(m, s, st, 0).m
        sums = np.asarray(p.sum(axis=1)).ravel()
        nonempty = np.diff(p.indptr) > 0
        assert np.allclose(sums[nonempty], 1.0)


def test_truncation_keeps_row_sums():
    m = poisson3d(8)
    s = oamg.strength_graph(m, 0.25)
    st = oamg.pmis(m, s)
    p0 = oamg.extended_interpolation(m, s, st, 0).m
    p4 = oamg.extended_interpolation(m, s, st, 4).m
    assert np.diff(p4.indptr).max() <= 4
    np.testing.assert_allclose(np.asarray(p4.sum(axis=1)).ravel(), np.asarray(p0.sum(axis=1)).ravel(),
                               rtol=1e-12, atol=1e-14)


def test_oracle_amg_properties():
    """Reference tests/test_amg.py properties, on the PMIS/ext+i/L1 AMG."""
    a = poisson1d(20)
    h = oamg.amg_setup(a, oamg.AmgOptions(coarse_size_cutoff=50))
    assert len(h.levels) == 1
    b = np.arange(20.0)
    assert np.max(np.abs(a @ oamg.amg_vcycle(h, b) - b)) < 1e-10
    p2 = poisson2d(32)
    h = oamg.amg_setup(p2, oamg.AmgOptions(pre_sweeps=2, post_sweeps=2))
    rng = np.random.default_rng(0)
    b = rng.standard_normal(p2.shape[0])
    x = np.zeros_like(b)
    norms = [np.linalg.norm(b)]
    for _ in range(10):
        x = oamg.amg_vcycle(h, b, x)
        norms.append(np.linalg.norm(b - p2 @ x))
    assert np.mean([norms[i + 1] / norms[i] for i in range(10)]) < 0.45
    assert 1.0 < h.operator_complexity() < 3.5
    lvl = h.levels[0]
    assert_bitwise(h.levels[1].a.m, (lvl.p.m.T.tocsr() @ (lvl.a.m @ lvl.p.m)).tocsr())
    d = sp.diags(np.linspace(1.0, 3.0, 300)).tocsr()
    hd = oamg.amg_setup(d)
    assert np.max(np.abs(d @ oamg.amg_vcycle(hd, np.ones(300)) - 1.0)) < 1e-12
    with pytest.raises(oamg.AmgSetupError):
        oamg.amg_setup(sp.csr_matrix(np.array([[1.0, 2.0], [3.0, 0.0]])))


def test_block_scale_pins():
    """D3: scaled diagonal blocks are exactly diag(lambda); no exact cancellations in the RAP pattern
    (symbolic pattern == numeric pattern)."""
    s = synth.make_config(2, 8)
    g, ahat = obs.block_scale(s)
    lam = obs.row_scale(obs.diag_blocks(s)).reshape(-1)
    np.testing.assert_array_equal(ahat.diagonal(), lam)
    f = synth.mgr_f_indices(2, s.n_cells)[0]
    c = np.setdiff1d(np.arange(s.n), f)
    r, p = omgr.build_rp(ahat, f, c, omgr.RpKind.NONINJECTIVE)
    num = (r @ (ahat @ p)).tocsr()
    ones = lambda m: sp.csr_matrix((np.ones(m.nnz), m.indices, m.indptr), shape=m.shape)  # noqa: E731
    sym = (ones(r) @ (ones(ahat) @ ones(p))).tocsr()
    assert num.nnz == sym.nnz


@pytest.mark.parametrize("cfg,edge", [(1, 32), (2, 12), (3, 12), (4, 8)])
def test_oracle_pipeline_converges(cfg, edge):
    s = synth.make_config(cfg, edge)
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    res, _, _ = opipe.solve_synthetic(s, rel_tol=1e-8, plan=plan, amg_opts=oamg.AmgOptions(**gpipe.DEFAULT_AMG))
    assert res.converged
    a = opipe.scalar_a(s)
    assert np.linalg.norm(s.rhs - a @ res.x) <= 1e-8 * np.linalg.norm(s.rhs) * (1 + 1e-6)


def test_oracle_self_perturbation_moves_iterations():
    """The explanation the GPU parity sweep leans on, shown on the oracle alone
    (reference AMG cutoff, deep hierarchies): at config 3 11^3 (rtol 1e-10) rounding-size noise (oracle.pipeline PERTURB_NOISE)
    moves the oracle's own GMRES iteration count by several iterations while the
    solutions agree to ~1e-10; and at 10^3 the oracle's first restart is forced by
    a rounding gap (|g| <= tol, true residual > tol)."""
    from oracle import amg as oamg, mgr as omgr, pipeline as opipe
    from paper_1801_08464_b200 import pipeline as gpipe, synth
    s = synth.make_config(3, 11)
    plan = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    opts = oamg.AmgOptions(**dict(gpipe.DEFAULT_AMG, coarse_size_cutoff=gpipe.REFERENCE_CUTOFF))
    state, _ = opipe.setup_synthetic(s, amg_opts=opts, plan=plan, post_smoothing=False)
    base = opipe.gmres_synthetic(state, s.rhs, rel_tol=1e-10)
    runs = [opipe.gmres_synthetic(state, s.rhs, rel_tol=1e-10, perturb_seed=100 + k, mode="noise") for k in range(1, 9)]
    its = [base.iterations] + [r.iterations for r in runs]
    assert max(its) - min(its) >= 2, its
    for r in runs:
        assert r.converged and np.linalg.norm(r.x - base.x) <= 1e-8 * np.linalg.norm(base.x)
    s10 = synth.make_config(3, 10)
    state10, _ = opipe.setup_synthetic(s10, amg_opts=opts, plan=opipe.default_plan(
        s10.b, s10.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX)), post_smoothing=False)
    st = {}
    r10 = opipe.gmres_synthetic(state10, s10.rhs, rel_tol=1e-10, stats=st)
    tol = 1e-10 * r10.rhs_norm
    assert st["ends"][0][1] <= tol < st["tops"][1][1]
