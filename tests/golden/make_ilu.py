"""Golden fixtures for the ILU(k) comparator, from the reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_ilu.py

Records the UNMODIFIED reference's ilu_factor (combined L\\U pattern and values)
and ilu_apply on seeded random diagonally dominant matrices at fill levels 0-2,
and GmresSolver(preconditioner='ilu') / ZeroPivot behaviour on the
reference-assembled Newton systems of tests/golden/physics.npz.
"""
import os
import sys

import numpy as np
import scipy.sparse as sp

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from ncpflow import ilu as rilu  # noqa: E402
from ncpflow import linsolve as rls  # noqa: E402
from ncpflow.assembly import ActiveSet  # noqa: E402
from ncpflow.krylov import GmresOptions  # noqa: E402
from ncpflow.sparse import CsrMatrix  # noqa: E402


def random_dd(rng, n, fill):
    dense = rng.standard_normal((n, n)) * (rng.random((n, n)) < fill)
    np.fill_diagonal(dense, np.abs(dense).sum(axis=1) + 1.0)
    return dense


def put_csr(d, name, m):
    m = sp.csr_matrix(m.m if hasattr(m, "m") else m)
    m.sort_indices()
    d[name + "_indptr"] = m.indptr.astype(np.int64)
    d[name + "_indices"] = m.indices.astype(np.int64)
    d[name + "_data"] = m.data
    d[name + "_shape"] = np.array(m.shape)


class System:
    def __init__(self, g, name):
        self.a = CsrMatrix(sp.csr_matrix((g[name + "_a_data"], g[name + "_a_indices"], g[name + "_a_indptr"]),
                                         shape=tuple(g[name + "_a_shape"])))
        self.rhs = g[name + "_rhs"]
        self.n_cells = int(g[name + "_ncells"])
        self.active_set = ActiveSet(g[name + "_active"], g[name + "_inactive"])


def main():
    out = {}
    rng = np.random.default_rng(7)
    for case, (n, fill) in enumerate([(40, 0.1), (60, 0.05), (30, 0.3)]):
        a = CsrMatrix.from_dense(random_dd(rng, n, fill))
        put_csr(out, f"r{case}_a", a)
        r = rng.standard_normal(n)
        out[f"r{case}_r"] = r
        for k in (0, 1, 2):
            f = rilu.ilu_factor(a, k)
            put_csr(out, f"r{case}_lu{k}", f.matrix)
            out[f"r{case}_x{k}"] = rilu.ilu_apply(f, r)
    g = np.load(os.path.join(HERE, "physics.npz"))
    for name in ["s3x3", "m12x10", "f12x10", "f8x8x4"]:
        system = System(g, name)
        for k in (0, 1):
            try:
                rilu.ilu_factor(system.a, k)
            except rilu.ZeroPivot as err:
                out[f"{name}_ilu{k}_zero_row"] = np.array(err.row)
            solver = rls.GmresSolver("ilu", GmresOptions(rel_tol=1e-10, max_iter=400, restart=30), ilu_level=k)
            try:
                res = solver.solve(system)
            except Exception as err:  # noqa: BLE001
                out[f"{name}_gsilu{k}_fail"] = np.array(str(err))
                print(name, k, "failed:", err)
                continue
            out[f"{name}_gsilu{k}_x"] = res.x
            out[f"{name}_gsilu{k}_its"] = np.array(res.iterations)
            out[f"{name}_gsilu{k}_conv"] = np.array(bool(res.converged))
            print(name, k, res.iterations, res.converged, res.residual_norm)
    np.savez_compressed(os.path.join(HERE, "ilu.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
