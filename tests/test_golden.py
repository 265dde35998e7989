"""Golden fixtures from the unmodified reference (tests/golden/make_golden.py).

CPU tests pin the oracle to the reference's own outputs; GPU tests check the
CUDA path against the same fixtures (integer patterns and scipy-order
products bit for bit, floating point within the north-star 1e-12).
"""
import os

import numpy as np
import pytest
import scipy.sparse as sp

from helpers import assert_bitwise, assert_close_csr, relerr
from oracle import amg as oamg
from oracle import blockscale as obs
from oracle import krylov as okr
from oracle import mgr as omgr
from oracle import sparse as osp
from paper_1801_08464_b200 import synth

G = np.load(os.path.join(os.path.dirname(__file__), "golden", "golden.npz"))


def mat(name):
    return sp.csr_matrix((G[name + "_data"], G[name + "_indices"], G[name + "_indptr"]),
                         shape=tuple(G[name + "_shape"]))


KINDS = ["injective", "noninjective", "injection", "ideal"]


# ---------------------------------------------------------------- oracle (CPU)
def test_oracle_products_bitwise():
    a, b = mat("g1_a"), mat("g1_b")
    assert_bitwise(osp.matmul(a, b).m, mat("g1_ab"))
    assert_bitwise(osp.spgemm_c(a, b).m, mat("g1_ab"))
    assert_bitwise(osp.triple_product(mat("g1_r"), mat("g1_sq"), mat("g1_p")).m, mat("g1_rap"))


@pytest.mark.parametrize("kind", KINDS)
def test_oracle_build_rp(kind):
    a = mat("g2_a")
    f = G["g2_f"]
    c = np.setdiff1d(np.arange(a.shape[0]), f)
    r, p = omgr.build_rp(a, f, c, omgr.RpKind(kind))
    if kind == "ideal":
        assert_close_csr(r, mat(f"g2_r_{kind}"), 1e-14)
        assert_close_csr(p, mat(f"g2_p_{kind}"), 1e-14)
    else:
        assert_bitwise(r, mat(f"g2_r_{kind}"))
        assert_bitwise(p, mat(f"g2_p_{kind}"))


@pytest.mark.parametrize("kind", ["injective", "noninjective"])
@pytest.mark.parametrize("post", [0, 1])
def test_oracle_mgr_apply(kind, post):
    a = mat("g3_a")
    spec = omgr.MgrLevelSpec((), omgr.RpKind(kind), omgr.FRelax("jacobi", sweeps=2))
    h = omgr.setup_from_matrix(a, [(G["g3_f"], spec)], coarse="exact", post_smoothing=bool(post))
    assert relerr(omgr.mgr_apply(h, G["g3_r"]), G[f"g3_e_{kind}_{post}"]) <= 1e-14
    assert_bitwise(h.levels[0].coarse_a, mat(f"g3_ac_{kind}_{post}"))


@pytest.mark.parametrize("tag,restart", [("r30", 30), ("r5", 5)])
def test_oracle_gmres(tag, restart):
    a = mat("g4_a")
    res = okr.gmres(lambda v: a @ v, None, G["g4_b"], okr.GmresOptions(rel_tol=1e-10, restart=restart))
    assert res.iterations == int(G[f"g4_its_{tag}"])
    assert relerr(res.x, G[f"g4_x_{tag}"]) <= 1e-13


@pytest.mark.parametrize("nm", ["poi", "ns"])
@pytest.mark.parametrize("th", [0.25, 0.5])
def test_oracle_strength(nm, th):
    np.testing.assert_array_equal(oamg.strength_graph(mat(f"g5_{nm}"), th), G[f"g5_s_{nm}_{th}"])


@pytest.mark.gpu
@pytest.mark.parametrize("nm", ["poi", "ns"])
@pytest.mark.parametrize("th", [0.25, 0.5])
def test_gpu_strength_golden(gpu, nm, th):
    """The device strength graph (mg_strength, amg_setup.cu k_strength) against the
    reference's own strength_graph outputs (golden g5), entry for entry."""
    from paper_1801_08464_b200 import amg as gamg
    s = gamg.strength_graph(mat(f"g5_{nm}"), th)
    np.testing.assert_array_equal(s.data, G[f"g5_s_{nm}_{th}"])


def test_oracle_synthetic_mgr_level():
    s = synth.make_config(1, 16)
    _, ahat = obs.block_scale(s)
    assert_bitwise(ahat, mat("g6_ahat"))
    f = synth.mgr_f_indices(2, s.n_cells)[0]
    c = np.setdiff1d(np.arange(s.n), f)
    r, p = omgr.build_rp(ahat, f, c, omgr.RpKind.NONINJECTIVE)
    assert_bitwise(r, mat("g6_r"))
    assert_bitwise(p, mat("g6_p"))
    assert_bitwise((r @ (ahat @ p)).tocsr(), mat("g6_ac"))


@pytest.mark.parametrize("tag,cfg,edge", [("c1", 1, 12), ("c4", 4, 6)])
def test_oracle_block_inverse_vs_reference(tag, cfg, edge):
    s = synth.make_config(cfg, edge)
    dinv = obs.block_inverse(obs.diag_blocks(s))
    ref = G[f"g7_inv_{tag}"]
    assert np.max(np.abs(dinv - ref)) <= 1e-12 * np.max(np.abs(ref))


# ---------------------------------------------------------------- GPU path
@pytest.mark.gpu
def test_gpu_products_bitwise(gpu):
    from paper_1801_08464_b200 import sparse as gsp
    assert_bitwise(gsp.matmul(mat("g1_a"), mat("g1_b")).to_scipy(), mat("g1_ab"))
    assert_bitwise(gsp.triple_product(mat("g1_r"), mat("g1_sq"), mat("g1_p")).to_scipy(), mat("g1_rap"))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", KINDS)
def test_gpu_build_rp(gpu, kind):
    from paper_1801_08464_b200 import mgr as gmgr
    a = mat("g2_a")
    f = G["g2_f"]
    part = type("Part", (), {"f_points": f, "c_points": np.setdiff1d(np.arange(a.shape[0]), f)})
    r, p = gmgr.build_rp(a, part, gmgr.RpKind(kind))
    if kind == "ideal":
        assert np.max(np.abs(r.to_dense() - mat(f"g2_r_{kind}").toarray())) < 1e-13
        assert np.max(np.abs(p.to_dense() - mat(f"g2_p_{kind}").toarray())) < 1e-13
    else:
        assert_bitwise(r.to_scipy(), mat(f"g2_r_{kind}"))
        assert_bitwise(p.to_scipy(), mat(f"g2_p_{kind}"))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["injective", "noninjective"])
@pytest.mark.parametrize("post", [0, 1])
def test_gpu_mgr_apply(gpu, kind, post):
    from paper_1801_08464_b200 import mgr as gmgr
    spec = gmgr.MgrLevelSpec((), gmgr.RpKind(kind), gmgr.FRelax("jacobi", sweeps=2))
    h = gmgr.setup_from_matrix(mat("g3_a"), [(G["g3_f"], spec)], coarse="exact", post_smoothing=bool(post))
    assert relerr(gmgr.mgr_apply(h, G["g3_r"]), G[f"g3_e_{kind}_{post}"]) <= 1e-12
    assert_bitwise(h.coarse_operator().to_scipy(), mat(f"g3_ac_{kind}_{post}"))


@pytest.mark.gpu
@pytest.mark.parametrize("tag,restart", [("r30", 30), ("r5", 5)])
def test_gpu_gmres(gpu, tag, restart):
    from paper_1801_08464_b200 import krylov as gkr
    res = gkr.gmres(mat("g4_a"), None, G["g4_b"], gkr.GmresOptions(rel_tol=1e-10, restart=restart))
    assert abs(res.iterations - int(G[f"g4_its_{tag}"])) <= 1
    assert relerr(res.x, G[f"g4_x_{tag}"]) <= 1e-8


@pytest.mark.gpu
def test_gpu_synthetic_mgr_level(gpu):
    from paper_1801_08464_b200 import mgr as gmgr, sparse as gsp
    s = synth.make_config(1, 16)
    d = gsp.DeviceMatrix.from_bsr(s.rowptr, s.col, s.vals)
    _, ahat = gsp.block_scale(d)
    assert_bitwise(ahat.to_scipy(), mat("g6_ahat"))
    f = synth.mgr_f_indices(2, s.n_cells)[0]
    part = type("Part", (), {"f_points": f, "c_points": np.setdiff1d(np.arange(s.n), f)})
    r, p = gmgr.build_rp(ahat, part, gmgr.RpKind.NONINJECTIVE)
    assert_bitwise(r.to_scipy(), mat("g6_r"))
    assert_bitwise(p.to_scipy(), mat("g6_p"))
    assert_bitwise(gsp.triple_product(r, ahat, p).to_scipy(), mat("g6_ac"))
