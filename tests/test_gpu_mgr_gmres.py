"""GPU parity: MGR setup/apply, GMRES, and the end-to-end synthetic solve.

Mirrors tests/test_mgr.py (:101-170, 190-250) and tests/test_krylov.py of the
reference with the oracle as the checker.  End-to-end bar (BASELINE.json):
GMRES iterations within +-1 and solution within 1e-8 relative at rtol 1e-10.
"""
import numpy as np
import pytest
import scipy.sparse as sp

from helpers import assert_bitwise, relerr
from oracle import amg as oamg
from oracle import blockscale as obs
from oracle import krylov as okr
from oracle import mgr as omgr
from oracle import pipeline as opipe
from paper_1801_08464_b200 import amg as gamg
from paper_1801_08464_b200 import krylov as gkr
from paper_1801_08464_b200 import mgr as gmgr
from paper_1801_08464_b200 import pipeline as gpipe
from paper_1801_08464_b200 import sparse as gsp
from paper_1801_08464_b200 import synth

pytestmark = pytest.mark.gpu


def random_system(rng, n):
    a = rng.standard_normal((n, n)) * 0.3
    a += np.diag(rng.uniform(2.0, 4.0, n)) * np.sqrt(n)
    return a


def spec_pair(kind, frelax, **fr):
    return (omgr.MgrLevelSpec((), omgr.RpKind(kind), omgr.FRelax(frelax, **fr)),
            gmgr.MgrLevelSpec((), gmgr.RpKind(kind), gmgr.FRelax(frelax, **fr)))


@pytest.mark.parametrize("kind", ["injective", "noninjective", "injection"])
@pytest.mark.parametrize("post", [False, True])
def test_mgr_apply_exact_coarse(gpu, kind, post):
    rng = np.random.default_rng(4)
    n = 60
    A = sp.csr_matrix(random_system(rng, n))
    f = np.sort(rng.choice(n, 24, replace=False))
    so, sg = spec_pair(kind, "jacobi", sweeps=2)
    ho = omgr.setup_from_matrix(A, [(f, so)], coarse="exact", post_smoothing=post)
    hg = gmgr.setup_from_matrix(A, [(f, sg)], coarse="exact", post_smoothing=post)
    assert hg.level_dims() == ho.level_dims()
    r = rng.standard_normal(n)
    assert relerr(gmgr.mgr_apply(hg, r), omgr.mgr_apply(ho, r)) <= 1e-12
    assert_bitwise(hg.coarse_operator().to_scipy(), ho.levels[-1].coarse_a)


def test_ideal_exact_one_iteration(gpu):
    rng = np.random.default_rng(2)
    for _ in range(5):
        n = int(rng.integers(8, 100))
        A = sp.csr_matrix(random_system(rng, n))
        nf = int(rng.integers(1, n))
        f = np.sort(rng.choice(n, nf, replace=False))
        spec = gmgr.MgrLevelSpec((), gmgr.RpKind.IDEAL, gmgr.FRelax("exact"))
        h = gmgr.setup_from_matrix(A, [(f, spec)], coarse="exact")
        b = rng.standard_normal(n)
        res = gkr.gmres(A, h, b, gkr.GmresOptions(rel_tol=1e-10, max_iter=10, restart=10))
        assert res.converged and res.iterations == 1


def test_mgr_zero_and_linearity(gpu):
    rng = np.random.default_rng(3)
    n = 30
    A = sp.csr_matrix(random_system(rng, n))
    spec = gmgr.MgrLevelSpec((), gmgr.RpKind.NONINJECTIVE, gmgr.FRelax("jacobi", sweeps=2))
    h = gmgr.setup_from_matrix(A, [(np.arange(10), spec)], coarse="exact")
    np.testing.assert_array_equal(gmgr.mgr_apply(h, np.zeros(n)), np.zeros(n))
    r1, r2 = rng.standard_normal(n), rng.standard_normal(n)
    lhs = gmgr.mgr_apply(h, r1 + r2)
    rhs = gmgr.mgr_apply(h, r1) + gmgr.mgr_apply(h, r2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * max(np.max(np.abs(rhs)), 1.0)


def test_empty_levels_skipped(gpu):
    rng = np.random.default_rng(9)
    n = 20
    A = sp.csr_matrix(random_system(rng, n))
    _, sg = spec_pair("injective", "jacobi")
    h = gmgr.setup_from_matrix(A, [(np.array([], dtype=int), sg), (np.arange(n), sg), (np.arange(5), sg)],
                               coarse="exact")
    assert h.level_dims() == [20, 15]


# 32^3 / 40^3: operators with >= 32768 rows run on the SELL-32 copies with
# compressed column codes (spmv.cu), so mgr_apply covers that path too
@pytest.mark.parametrize("cfg,edge", [(1, 24), (2, 10), (3, 10), (4, 6), (2, 32), (3, 32), (4, 40)])
def test_synthetic_hierarchy_bitwise(gpu, cfg, edge):
    """MGR level operators, R/P and both AMG hierarchies equal the oracle bit for bit."""
    s = synth.make_config(cfg, edge)
    _, ahat_o = obs.block_scale(s)
    # the reference's cutoff: hierarchies as deep as the sizes allow
    opts_kw = dict(gpipe.DEFAULT_AMG, coarse_size_cutoff=gpipe.REFERENCE_CUTOFF)
    plan_o = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    ho = omgr.setup_from_matrix(ahat_o, plan_o, oamg.AmgOptions(**opts_kw))
    d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
    _, ahat_g = gsp.block_scale(d)
    hg = gmgr.setup_from_matrix(ahat_g, gpipe.default_plan(s.b, s.n_cells), gamg.AmgOptions(**opts_kw))
    assert hg.level_dims() == ho.level_dims()
    for k, lvl in enumerate(ho.levels):
        assert_bitwise(hg.level_matrix(k, "r").to_scipy(), lvl.r)
        assert_bitwise(hg.level_matrix(k, "p").to_scipy(), lvl.p)
        assert_bitwise(hg.level_matrix(k, "coarse_a").to_scipy(), lvl.coarse_a)
        fo = lvl.f_solver.hier
        fg = hg.amg(k)
        assert fg.level_sizes() == fo.level_sizes()
        for q in range(len(fo.levels)):
            assert_bitwise(fg.levels[q].a.to_scipy(), fo.levels[q].a.m)
    co, cg = ho.coarse_amg, hg.amg(-1)
    assert cg.level_sizes() == co.level_sizes()
    for q in range(len(co.levels) - 1):
        np.testing.assert_array_equal(cg.levels[q].splitting, co.levels[q].splitting)
        assert_bitwise(cg.levels[q].p.to_scipy(), co.levels[q].p.m)
    r = np.random.default_rng(0).standard_normal(s.n)
    assert relerr(gmgr.mgr_apply(hg, r), omgr.mgr_apply(ho, r)) <= 1e-12


def test_gmres_unpreconditioned_matches_oracle(gpu):
    rng = np.random.default_rng(11)
    n = 200
    A = sp.csr_matrix(random_system(rng, n) / np.sqrt(n))
    b = rng.standard_normal(n)
    for opts in (dict(rel_tol=1e-10, restart=30, max_iter=400), dict(rel_tol=1e-10, restart=5, max_iter=40),
                 dict(rel_tol=1e-8, restart=30, max_iter=400, reorthogonalize=False)):
        ro = okr.gmres(lambda v: A @ v, None, b, okr.GmresOptions(**opts))
        rg = gkr.gmres(A, None, b, gkr.GmresOptions(**opts))
        assert abs(rg.iterations - ro.iterations) <= 1
        assert rg.converged == ro.converged
        assert relerr(rg.x, ro.x) <= 1e-8


def test_gmres_zero_rhs_and_true_residual(gpu):
    A = sp.identity(10, format="csr") * 2.0
    r = gkr.gmres(A, None, np.zeros(10), gkr.GmresOptions())
    assert r.iterations == 0 and r.converged
    rng = np.random.default_rng(1)
    M = sp.csr_matrix(random_system(rng, 40))
    b = rng.standard_normal(40)
    res = gkr.gmres(M, None, b, gkr.GmresOptions(rel_tol=1e-9))
    assert res.converged
    assert np.linalg.norm(b - M @ res.x) <= 1e-9 * np.linalg.norm(b) * (1 + 1e-6)


def test_gmres_backward_error_acceptance(gpu):
    rng = np.random.default_rng(2)
    n = 60
    A = sp.csr_matrix(random_system(rng, n))
    b = rng.standard_normal(n)
    a_norm = float(np.max(np.abs(A).sum(axis=1)))
    ro = okr.gmres(lambda v: A @ v, None, b, okr.GmresOptions(rel_tol=1e-6, check_every=2), a_norm=a_norm)
    rg = gkr.gmres(A, None, b, gkr.GmresOptions(rel_tol=1e-6, check_every=2), a_norm=a_norm)
    assert abs(rg.iterations - ro.iterations) <= 1 and rg.converged


@pytest.mark.parametrize("ortho", ["dcgs2", "cgs2"])
@pytest.mark.parametrize("where", ["matrix", "rhs"])
def test_gmres_nonfinite_terminates(gpu, ortho, where):
    """A NaN in the system must end the solve with converged=False (the
    reference returns at max_iter, krylov.py:80-81); it must not loop forever."""
    rng = np.random.default_rng(5)
    n = 50
    A = random_system(rng, n)
    b = rng.standard_normal(n)
    if where == "matrix":
        A[3, 3] = np.nan
    else:
        b[7] = np.nan
    spec = gmgr.MgrLevelSpec((), gmgr.RpKind.NONINJECTIVE, gmgr.FRelax("jacobi"))
    h = gmgr.setup_from_matrix(sp.csr_matrix(random_system(rng, n)), [(np.arange(20), spec)], coarse="exact")
    for m in (None, h):
        res = gkr.gmres(sp.csr_matrix(A), m, b, gkr.GmresOptions(rel_tol=1e-10, max_iter=60,
                                                                 orthogonalization=ortho))
        assert not res.converged and res.iterations <= 60


@pytest.mark.parametrize("restart", [30, 7])
def test_gmres_cgs2_mode_matches_oracle(gpu, restart):
    """The reference's classic CGS2 pass order (krylov.py:101-107) on the device."""
    rng = np.random.default_rng(13)
    n = 300
    A = sp.csr_matrix(random_system(rng, n) / np.sqrt(n))
    b = rng.standard_normal(n)
    opts = dict(rel_tol=1e-10, restart=restart, max_iter=400)
    ro = okr.gmres(lambda v: A @ v, None, b, okr.GmresOptions(**opts))
    for ortho in ("cgs2", "dcgs2"):
        rg = gkr.gmres(A, None, b, gkr.GmresOptions(**opts, orthogonalization=ortho))
        assert abs(rg.iterations - ro.iterations) <= 1 and rg.converged == ro.converged
        assert relerr(rg.x, ro.x) <= 1e-8


def test_gmres_rejects_callables(gpu):
    with pytest.raises(TypeError):
        gkr.gmres(lambda v: v, None, np.ones(3))


# End-to-end parity (iterations vs the oracle's envelope, solution <= 1e-8 at rtol
# 1e-10): tests/test_gpu_parity_sweep.py (every edge of configs 3 / 4, configs 1 / 2
# small and at 32^3) and tests/test_gpu_parity_full.py (the BASELINE sizes).


def test_repeated_setup_and_solve_bitwise_deterministic(gpu):
    """Every kernel on the path has a fixed operation order (no atomics in any
    sum, fixed reduction trees), and the concurrent setup (worker streams,
    per-worker pools) must not change that: two setups + solves of the same
    system give bit-identical solutions, and a second solver object too."""
    s = synth.make_config(3, 40)
    sol = gpipe.SyntheticSolver(rel_tol=1e-10)
    r1, _ = sol.solve_system(s)
    r2, _ = sol.solve_system(s)
    r3, _ = gpipe.SyntheticSolver(rel_tol=1e-10).solve_system(s)
    assert r1.converged and r1.iterations == r2.iterations == r3.iterations
    np.testing.assert_array_equal(r1.x, r2.x)
    np.testing.assert_array_equal(r1.x, r3.x)


def test_graph_reuse_across_systems(gpu):
    """A solver reused on a new system of the same shape installs the new MGR apply
    graph into the previous hierarchy's parked executable (cudaGraphExecUpdate,
    solver.cu capture_apply): the solution must equal a fresh solver's bit for bit,
    for a system solved after another one with different values."""
    s1 = synth.make_config(3, 40, seed=11)
    s2 = synth.make_config(3, 40, seed=12)
    sol = gpipe.SyntheticSolver(rel_tol=1e-10)
    sol.solve_system(s1)
    r_reused, _ = sol.solve_system(s2)
    r_fresh, _ = gpipe.SyntheticSolver(rel_tol=1e-10).solve_system(s2)
    assert r_reused.converged and r_reused.iterations == r_fresh.iterations
    np.testing.assert_array_equal(r_reused.x, r_fresh.x)


def test_dense_inverse_needs_pivoting(gpu):
    """IDEAL R/P and exact F / coarse solves on blocks with zero diagonals (n > 256):
    the unpivoted blocked Gauss-Jordan rejects the pivot and the partially pivoted
    path takes over; the apply matches the oracle (splu) within 1e-12."""
    rng = np.random.default_rng(21)
    nf, nc = 300, 280
    perm = (np.arange(nf) + nf // 2) % nf
    aff = np.zeros((nf, nf))
    aff[np.arange(nf), perm] = 3.0 + rng.uniform(0, 1, nf)
    aff += rng.standard_normal((nf, nf)) * 0.01 * (rng.uniform(size=(nf, nf)) < 0.02)
    np.fill_diagonal(aff, 0.0)
    acc = np.diag(rng.uniform(4.0, 5.0, nc)) + rng.standard_normal((nc, nc)) * 0.01
    afc = rng.standard_normal((nf, nc)) * 0.05
    acf = rng.standard_normal((nc, nf)) * 0.05
    A = sp.csr_matrix(np.block([[aff, afc], [acf, acc]]))
    f = np.arange(nf)
    so, sg = spec_pair("ideal", "exact")
    ho = omgr.setup_from_matrix(A, [(f, so)], coarse="exact")
    hg = gmgr.setup_from_matrix(A, [(f, sg)], coarse="exact")
    r = rng.standard_normal(nf + nc)
    assert relerr(gmgr.mgr_apply(hg, r), omgr.mgr_apply(ho, r)) <= 1e-12


@pytest.mark.parametrize("step", [0, 7, 19])
def test_sequence_step_parity(gpu, step):
    """BASELINE config 5's time-step sequence (gas sphere radius + step cells,
    mobilities from seed + step): one solver object reused across the steps, as
    the sequence runs -- iterations +-1 and solution <= 1e-8 against the oracle at
    rtol 1e-10 for the step's own system."""
    sol = gpipe.SyntheticSolver(rel_tol=1e-10)
    for k in sorted({0, step}):
        s = synth.make_config(5, 24, step=k)
        rg, _ = sol.solve_system(s)
    opts = oamg.AmgOptions(**gpipe.DEFAULT_AMG)
    plan_o = opipe.default_plan(s.b, s.n_cells, frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    ro, _, _ = opipe.solve_synthetic(s, rel_tol=1e-10, plan=plan_o, amg_opts=opts)
    assert ro.converged and rg.converged
    assert abs(rg.iterations - ro.iterations) <= 1, (rg.iterations, ro.iterations)
    assert relerr(rg.x, ro.x) <= 1e-8


@pytest.mark.parametrize("kind", ["injective", "injection"])
@pytest.mark.parametrize("cfg,edge", [(1, 32), (2, 20), (3, 24)])
def test_synthetic_other_rp_kinds_parity(gpu, cfg, edge, kind):
    """the b = 2 configs run NONINJECTIVE (the north star's literal R / P)
    by default; the reference schema's other kinds (RpKind, mgr.py:47-51) on the same
    systems, end to end against the oracle at rtol 1e-10: iterations +-1, solution
    <= 1e-8."""
    s = synth.make_config(cfg, edge)
    rg, _ = gpipe.SyntheticSolver(rel_tol=1e-10, rp=gmgr.RpKind(kind)).solve_system(s)
    plan_o = opipe.default_plan(s.b, s.n_cells, rp=omgr.RpKind(kind),
                                frelax=omgr.FRelax("amg", **gpipe.DEFAULT_FRELAX))
    ro, _, _ = opipe.solve_synthetic(s, rel_tol=1e-10, plan=plan_o, amg_opts=oamg.AmgOptions(**gpipe.DEFAULT_AMG))
    assert ro.converged and rg.converged
    assert abs(rg.iterations - ro.iterations) <= 1, (rg.iterations, ro.iterations)
    assert relerr(rg.x, ro.x) <= 1e-8


@pytest.mark.parametrize("nf", [257, 320, 1001, 1708])
def test_blocked_dense_inverse_sizes(gpu, nf):
    """The blocked Gauss-Jordan inverse behind FRelax('exact') / coarse='exact' / the AMG
    coarsest level (amg.py:330-343), at sizes with a partial last panel, an odd and an even
    panel count: the MGR apply through it matches the oracle's LU solves within 1e-12."""
    rng = np.random.default_rng(nf)
    nc = 40
    n = nf + nc
    a = sp.random(n, n, density=min(1.0, 12.0 / n), random_state=rng, format="csr") * 0.2
    a = a + sp.diags(rng.uniform(3.0, 5.0, n))
    A = sp.csr_matrix(a)
    f = np.arange(nf)
    so, sg = spec_pair("injective", "exact")
    ho = omgr.setup_from_matrix(A, [(f, so)], coarse="exact")
    hg = gmgr.setup_from_matrix(A, [(f, sg)], coarse="exact")
    for _ in range(2):
        r = rng.standard_normal(n)
        assert relerr(gmgr.mgr_apply(hg, r), omgr.mgr_apply(ho, r)) <= 1e-12


def test_sequence_pipelined_upload_matches_synchronous(gpu):
    """BASELINE config 5's sequence as a pipeline: the next system staged in pinned memory
    and copied on the copy stream (mg_mat_upload_bsr_async) while the current one is set up
    and solved, one solver reused -- every step's solution and iteration count equal the
    synchronous solve_system of the same step bit for bit."""
    nsteps = 4
    systems = [synth.make_config(5, 20, step=k) for k in range(nsteps)]
    ref = []
    for s in systems:
        r, _ = gpipe.SyntheticSolver(rel_tol=1e-10).solve_system(s)
        ref.append(r)
    stage = [gpipe.PinnedSystem(systems[0]), gpipe.PinnedSystem(systems[1])]
    sol = gpipe.SyntheticSolver(rel_tol=1e-10)
    nxt = sol.upload(stage[0], asynchronous=True)
    for k in range(nsteps):
        cur = stage[k & 1]
        a = nxt
        nxt = sol.upload(stage[(k + 1) & 1], asynchronous=True) if k + 1 < nsteps else None
        sol.a = a
        sol.sysm_meta = (cur.b, cur.n_cells)
        sol.setup(a)
        r = sol.solve(cur.rhs)
        a.free()
        if k + 2 < nsteps:
            stage[k & 1].load(systems[k + 2])
        assert r.iterations == ref[k].iterations
        np.testing.assert_array_equal(r.x.view(np.int64), ref[k].x.view(np.int64))
