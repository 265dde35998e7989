"""Generate golden fixtures from the reference package (run in the build container).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array here is an output of the UNMODIFIED reference (ncpflow) on seeded
inputs; tests/test_golden.py checks the oracle (CPU) and the GPU path against
them without needing /root/reference at run time.
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from ncpflow import amg as ramg  # noqa: E402
from ncpflow import krylov as rkr  # noqa: E402
from ncpflow import mgr as rmgr  # noqa: E402
from ncpflow.sparse import CsrMatrix, IndexPartition, triple_product  # noqa: E402

from paper_1801_08464_b200 import synth  # noqa: E402
from oracle import blockscale as obs  # noqa: E402


def put(d, name, m):
    m = m.m if hasattr(m, "m") else m
    m = sp.csr_matrix(m)
    d[name + "_indptr"] = m.indptr.astype(np.int64)
    d[name + "_indices"] = m.indices.astype(np.int64)
    d[name + "_data"] = m.data
    d[name + "_shape"] = np.array(m.shape)


def random_system(rng, n):
    a = rng.standard_normal((n, n)) * 0.3
    a += np.diag(rng.uniform(2.0, 4.0, n)) * np.sqrt(n)
    return a


def main():
    out = {}
    rng = np.random.default_rng(20240)
    # G1: products (scipy semantics through the reference's own functions)
    a = sp.random(60, 50, density=0.15, random_state=1, data_rvs=rng.standard_normal).tocsr()
    b = sp.random(50, 70, density=0.15, random_state=2, data_rvs=rng.standard_normal).tocsr()
    r = sp.random(30, 60, density=0.2, random_state=3, data_rvs=rng.standard_normal).tocsr()
    sq = sp.random(60, 60, density=0.1, random_state=4, data_rvs=rng.standard_normal).tocsr() + sp.identity(60)
    p = sp.random(60, 40, density=0.1, random_state=5, data_rvs=rng.standard_normal).tocsr()
    put(out, "g1_a", a)
    put(out, "g1_b", b)
    put(out, "g1_ab", rmgr.triple_product(CsrMatrix(sp.identity(60, format="csr")), CsrMatrix(a), CsrMatrix(b)))
    put(out, "g1_r", r)
    put(out, "g1_sq", sq)
    put(out, "g1_p", p)
    put(out, "g1_rap", triple_product(CsrMatrix(r), CsrMatrix(sq), CsrMatrix(p)))
    # G2: build_rp, all kinds (reference test_mgr.py:50-65 inputs)
    rng2 = np.random.default_rng(0)
    a2 = random_system(rng2, 12)
    f2 = np.sort(rng2.choice(12, 5, replace=False))
    mask = np.zeros(12, dtype=bool)
    mask[f2] = True
    part = IndexPartition.from_f_mask(mask)
    put(out, "g2_a", a2)
    out["g2_f"] = f2
    for kind in rmgr.RpKind:
        rr, pp = rmgr.build_rp(CsrMatrix.from_dense(a2), part, kind)
        put(out, f"g2_r_{kind.value}", rr)
        put(out, f"g2_p_{kind.value}", pp)
    # G3: MGR apply (jacobi F-relax, exact coarse), both orders
    rng3 = np.random.default_rng(4)
    a3 = random_system(rng3, 30)
    f3 = np.sort(rng3.choice(30, 12, replace=False))
    r3 = rng3.standard_normal(30)
    put(out, "g3_a", a3)
    out["g3_f"] = f3
    out["g3_r"] = r3
    for kind in ("injective", "noninjective"):
        for post in (False, True):
            spec = rmgr.MgrLevelSpec((), rmgr.RpKind(kind), rmgr.FRelax("jacobi", sweeps=2))
            h = rmgr.setup_from_matrix(CsrMatrix.from_dense(a3), [(f3, spec)], coarse="exact",
                                       post_smoothing=post)
            out[f"g3_e_{kind}_{int(post)}"] = rmgr.mgr_apply(h, r3)
            put(out, f"g3_ac_{kind}_{int(post)}", h.levels[0].coarse_a)
    # G4: GMRES, identity and none preconditioner, two restarts
    rng4 = np.random.default_rng(11)
    a4 = random_system(rng4, 80) / np.sqrt(80)
    b4 = rng4.standard_normal(80)
    put(out, "g4_a", a4)
    out["g4_b"] = b4
    for tag, opts in (("r30", rkr.GmresOptions(rel_tol=1e-10)), ("r5", rkr.GmresOptions(rel_tol=1e-10, restart=5))):
        res = rkr.gmres(lambda v: a4 @ v, None, b4, opts)
        out[f"g4_x_{tag}"] = res.x
        out[f"g4_its_{tag}"] = np.array(res.iterations)
        out[f"g4_res_{tag}"] = np.array(res.residual_norm)
    # G5: strength graph
    e = np.ones(20)
    t = sp.diags([-e[:-1], 2 * e, -e[:-1]], [-1, 0, 1])
    poi = (sp.kron(t, sp.identity(20)) + sp.kron(sp.identity(20), t)).tocsr()
    rng5 = np.random.default_rng(5)
    ns = sp.random(200, 200, density=0.05, random_state=6, data_rvs=rng5.standard_normal).tocsr() \
        + sp.diags(rng5.uniform(1, 2, 200))
    ns = ns.tocsr()
    ns.sort_indices()
    for nm, m in (("poi", poi), ("ns", ns)):
        put(out, f"g5_{nm}", m)
        for th in (0.25, 0.5):
            out[f"g5_s_{nm}_{th}"] = ramg.strength_graph(CsrMatrix(m), th).data.astype(np.int8)
    # G6: synthetic config-1 16x16: reference MGR level on the block-scaled matrix
    s6 = synth.make_config(1, 16)
    _, ahat6 = obs.block_scale(s6)
    put(out, "g6_ahat", ahat6)
    f6 = synth.mgr_f_indices(2, s6.n_cells)[0]
    spec6 = rmgr.MgrLevelSpec((), rmgr.RpKind.NONINJECTIVE, rmgr.FRelax("jacobi"))
    h6 = rmgr.setup_from_matrix(CsrMatrix(ahat6), [(f6, spec6)], coarse="exact")
    put(out, "g6_r", h6.levels[0].r)
    put(out, "g6_p", h6.levels[0].p)
    put(out, "g6_ac", h6.levels[0].coarse_a)
    # G7: reference per-cell block inverses (_BlockDiagSolver) on config-4 8^3 (b=3) and config-1
    for tag, (cfg, edge) in (("c1", (1, 12)), ("c4", (4, 6))):
        s7 = synth.make_config(cfg, edge)
        a7 = synth.to_scalar_csr(s7, "cell", drop_zeros=False)
        cells = np.repeat(np.arange(s7.n_cells), s7.b)
        bd = rmgr._BlockDiagSolver(CsrMatrix(a7), cells)
        (idx, inv), = bd.batches
        out[f"g7_inv_{tag}"] = inv
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
