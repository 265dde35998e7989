"""Oracle restatement of ncpflow/sparse.py semantics (test infrastructure only).

* CSR with int32 indices, f64 values, sorted columns; explicit zeros are
  legal stored entries (sparse.py:35-50).
* ``matmul`` / ``triple_product`` use scipy's csr_matmat, which DROPS exact
  zero results after each product (probe p1; contrary
  to the docstring at sparse.py:4-6,200) and accumulates each output in
  left-operand column order with a separate multiply and add (probe p2).
* ``extract`` keeps stored zeros (sparse.py:181-190).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import clib


class DimensionMismatch(ValueError):
    pass


class CsrMatrix:
    """Minimal carrier with the attribute surface the reference MGR uses."""

    __slots__ = ("m",)

    def __init__(self, m):
        m = sp.csr_matrix(m) if not sp.isspmatrix_csr(m) else m
        if not m.has_sorted_indices:
            m = m.copy()
            m.sort_indices()
        self.m = m

    nrows = property(lambda s: s.m.shape[0])
    ncols = property(lambda s: s.m.shape[1])
    shape = property(lambda s: s.m.shape)
    nnz = property(lambda s: s.m.nnz)
    row_offsets = property(lambda s: s.m.indptr)
    col_indices = property(lambda s: s.m.indices)
    values = property(lambda s: s.m.data)

    def diagonal(self):
        return self.m.diagonal()

    def to_dense(self):
        return self.m.toarray()

    def transpose(self):
        return CsrMatrix(self.m.T.tocsr())


def as_scipy(a):
    """Accept an ncpflow/oracle CsrMatrix (has ``.m``) or any scipy matrix."""
    if hasattr(a, "m"):
        return a.m
    return sp.csr_matrix(a)


def spmv(a, x):
    m = as_scipy(a)
    x = np.asarray(x, dtype=float)
    if x.shape != (m.shape[1],):
        raise DimensionMismatch("spmv dimension mismatch")
    return m @ x


def extract(a, rows, cols):
    m = as_scipy(a)
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    return CsrMatrix(m[rows][:, cols].tocsr())


def matmul(a, b):
    am, bm = as_scipy(a), as_scipy(b)
    if am.shape[1] != bm.shape[0]:
        raise DimensionMismatch("matmul")
    return CsrMatrix((am @ bm).tocsr())


def triple_product(r, a, p):
    """R*(A*P) with scipy semantics (ncpflow/sparse.py:199-203)."""
    rm, am, pm = as_scipy(r), as_scipy(a), as_scipy(p)
    if rm.shape[1] != am.shape[0] or am.shape[1] != pm.shape[0]:
        raise DimensionMismatch("triple_product")
    return CsrMatrix((rm @ (am @ pm)).tocsr())


def spgemm_c(a, b):
    """The same product through the pinned C loop (cross-check of scipy's order)."""
    am, bm = as_scipy(a), as_scipy(b)
    L = clib.lib()
    m, k = am.shape[0], bm.shape[1]
    ap, aj = clib.c32(am.indptr), clib.c32(am.indices)
    ax = np.ascontiguousarray(am.data, dtype=float)
    bp, bj = clib.c32(bm.indptr), clib.c32(bm.indices)
    bx = np.ascontiguousarray(bm.data, dtype=float)
    cnt = np.zeros(m, dtype=np.int32)
    L.spgemm_count(m, k, clib.ptr(ap), clib.ptr(aj), clib.ptr(ax), clib.ptr(bp),
                   clib.ptr(bj), clib.ptr(bx), clib.ptr(cnt))
    cp = np.zeros(m + 1, dtype=np.int64)
    np.cumsum(cnt, out=cp[1:])
    cj = np.zeros(int(cp[-1]), dtype=np.int32)
    cx = np.zeros(int(cp[-1]))
    L.spgemm_fill(m, k, clib.ptr(ap), clib.ptr(aj), clib.ptr(ax), clib.ptr(bp),
                  clib.ptr(bj), clib.ptr(bx), clib.ptr(cp), clib.ptr(cj), clib.ptr(cx))
    return CsrMatrix(sp.csr_matrix((cx, cj, cp), shape=(m, k)))
