"""Device sparse matrices and the reference's sparse-kernel entry points.

Mirrors ncpflow/sparse.py (``spmv`` :174-178, ``extract`` :181-190,
``matmul`` :193-196, ``triple_product`` :199-203) with the same argument
meaning and error types, computed by libmgrgpu's sm_100a kernels.  Inputs may
be ``DeviceMatrix`` handles or any host CSR (an ``ncpflow.sparse.CsrMatrix``
— anything with ``.m`` — or a scipy sparse matrix), which is uploaded.
Products follow scipy's csr_matmat semantics bit for bit (exact zeros are
dropped).
"""
from __future__ import annotations

import numpy as np

from . import _lib
from .errors import DimensionMismatch


class DeviceMatrix:
    """Scalar CSR (b=1) or block CSR (b=2,3) matrix resident in HBM."""

    __slots__ = ("ctx", "h", "_info", "_keep")

    def __init__(self, ctx, handle, keep=None):
        self.ctx = ctx
        self.h = handle
        self._info = None
        self._keep = keep  # host arrays an asynchronous upload may still be reading

    # -- construction -----------------------------------------------------
    @classmethod
    def from_csr(cls, indptr, indices, data, shape, ctx=None):
        ctx = ctx or _lib.ctx()
        ip, ix, dv = _lib.i32(indptr), _lib.i32(indices), _lib.f64(data)
        h = _lib.P()
        ctx.call("mg_mat_upload_csr", int(shape[0]), int(shape[1]), _lib.ptr(ip), _lib.ptr(ix),
                 _lib.ptr(dv), _lib.ctypes.byref(h))
        return cls(ctx, h)

    @classmethod
    def from_bsr(cls, rowptr, colind, blocks, nbcols=None, ctx=None, asynchronous=False):
        """Upload a block CSR matrix.  ``asynchronous=True`` returns at once and
        copies on the context's copy stream (mg_mat_upload_bsr_async), so the
        next system can be uploaded while the current one is solved; the
        arrays must then be pinned to overlap, and are kept referenced by the
        returned matrix."""
        ctx = ctx or _lib.ctx()
        blocks = _lib.f64(blocks)
        b = blocks.shape[-1]
        rp, ci = _lib.i32(rowptr), _lib.i32(colind)
        nb = rp.size - 1
        h = _lib.P()
        fn = "mg_mat_upload_bsr_async" if asynchronous else "mg_mat_upload_bsr"
        ctx.call(fn, nb, int(nbcols if nbcols is not None else nb), int(b), _lib.ptr(rp),
                 _lib.ptr(ci), _lib.ptr(blocks), _lib.ctypes.byref(h))
        return cls(ctx, h, (rp, ci, blocks) if asynchronous else None)

    @classmethod
    def from_csr_varmajor(cls, indptr, indices, data, b, ctx=None):
        """The reference's variable-major scalar CSR (unknown var * N + cell,
        assembly.py:95-120) as the cell-major b x b block CSR the block kernels
        use (mg_mat_upload_csr_varmajor; conversion on the device).  Vectors for
        the result are cell-major: see to_cell_major / to_var_major."""
        ctx = ctx or _lib.ctx()
        ip, ix, dv = _lib.i32(indptr), _lib.i32(indices), _lib.f64(data)
        h = _lib.P()
        ctx.call("mg_mat_upload_csr_varmajor", int(ip.size - 1), int(b), _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv),
                 _lib.ctypes.byref(h))
        return cls(ctx, h)

    @classmethod
    def from_host(cls, a, ctx=None):
        if isinstance(a, DeviceMatrix):
            return a
        import scipy.sparse as sp
        m = a.m if hasattr(a, "m") else a
        if not sp.issparse(m):
            m = sp.csr_matrix(np.asarray(m, dtype=float))
        m = m.tocsr()
        if not m.has_sorted_indices:
            m = m.copy()
            m.sort_indices()
        return cls.from_csr(m.indptr, m.indices, m.data, m.shape, ctx)

    # -- info ---------------------------------------------------------------
    def _load_info(self):
        if self._info is None:
            nr, nc, b = _lib.c_int(), _lib.c_int(), _lib.c_int()
            nnz = _lib.c_int64()
            self.ctx.call("mg_mat_info", self.h, _lib.ctypes.byref(nr), _lib.ctypes.byref(nc),
                          _lib.ctypes.byref(nnz), _lib.ctypes.byref(b))
            self._info = (nr.value, nc.value, nnz.value, b.value)
        return self._info

    def spmv_layout(self):
        """(sell, index_bytes, sorted) of the solve-phase SpMV copy (mg_spmv_layout)."""
        sell, ib, srt = _lib.c_int(), _lib.c_int(), _lib.c_int()
        self.ctx.call("mg_spmv_layout", self.h, _lib.ctypes.byref(sell), _lib.ctypes.byref(ib),
                      _lib.ctypes.byref(srt))
        return bool(sell.value), ib.value, bool(srt.value)

    @property
    def block_size(self):
        return self._load_info()[3]

    @property
    def nrows(self):
        nr, _, _, b = self._load_info()
        return nr * b

    @property
    def ncols(self):
        _, nc, _, b = self._load_info()
        return nc * b

    @property
    def shape(self):
        return (self.nrows, self.ncols)

    @property
    def nnz(self):
        return self._load_info()[2]

    def download(self):
        nr, nc, nnz, b = self._load_info()
        ip = np.zeros(nr + 1, dtype=np.int32)
        ix = np.zeros(nnz, dtype=np.int32)
        dv = np.zeros(nnz * b * b)
        self.ctx.call("mg_mat_download", self.h, _lib.ptr(ip), _lib.ptr(ix), _lib.ptr(dv))
        return ip, ix, dv

    def to_scipy(self):
        import scipy.sparse as sp
        ip, ix, dv = self.download()
        nr, nc, nnz, b = self._load_info()
        if b == 1:
            m = sp.csr_matrix((dv, ix, ip), shape=(nr, nc))
            m.has_sorted_indices = True
            return m
        return sp.bsr_matrix((dv.reshape(nnz, b, b), ix, ip), shape=(nr * b, nc * b)).tocsr()

    @property
    def m(self):
        """scipy view (host copy), the attribute the reference's CsrMatrix exposes."""
        return self.to_scipy()

    def to_dense(self):
        return self.to_scipy().toarray()

    def diagonal(self):
        return self.to_scipy().diagonal()

    def transpose(self):
        h = _lib.P()
        self.ctx.call("mg_transpose", self.h, _lib.ctypes.byref(h))
        return DeviceMatrix(self.ctx, h)

    def __matmul__(self, x):
        return spmv(self, x)

    def free(self):
        if self.h:
            self.ctx.lib.mg_mat_free(self.ctx.h, self.h)
            self.h = None
            if self._keep is not None:  # copies of an asynchronous upload have landed before the arrays go
                self.ctx.sync()
                self._keep = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # noqa: BLE001
            pass

    def __repr__(self):
        return f"DeviceMatrix({self.nrows}x{self.ncols}, nnz={self.nnz}, b={self.block_size})"


def as_device(a, ctx=None) -> DeviceMatrix:
    return DeviceMatrix.from_host(a, ctx)


def spmv(a, x) -> np.ndarray:
    """y = A x (sparse.py:174-178)."""
    d = as_device(a)
    x = _lib.f64(x)
    if x.shape != (d.ncols,):
        raise DimensionMismatch(f"spmv: matrix is {d.nrows}x{d.ncols}, vector has length {x.shape}")
    y = np.empty(d.nrows)
    d.ctx.call("mg_spmv", d.h, _lib.ptr(x), _lib.ptr(y))
    return y


def matmul(a, b) -> DeviceMatrix:
    da, db = as_device(a), as_device(b)
    if da.ncols != db.nrows:
        raise DimensionMismatch(f"matmul: {da.shape} x {db.shape}")
    h = _lib.P()
    da.ctx.call("mg_matmul", da.h, db.h, _lib.ctypes.byref(h))
    return DeviceMatrix(da.ctx, h)


def triple_product(r, a, p) -> DeviceMatrix:
    dr, da, dp = as_device(r), as_device(a), as_device(p)
    if dr.ncols != da.nrows or da.ncols != dp.nrows:
        raise DimensionMismatch(f"triple_product: {dr.shape} x {da.shape} x {dp.shape}")
    h = _lib.P()
    da.ctx.call("mg_triple_product", dr.h, da.h, dp.h, _lib.ctypes.byref(h))
    return DeviceMatrix(da.ctx, h)


def extract(a, rows, cols) -> DeviceMatrix:
    """A[rows][:, cols] keeping stored zeros (sparse.py:181-190)."""
    d = as_device(a)
    rows, cols = _lib.i64(rows), _lib.i64(cols)
    for idx, limit, what in ((rows, d.nrows, "row"), (cols, d.ncols, "column")):
        if idx.size and (idx.min() < 0 or idx.max() >= limit):
            raise IndexError(f"{what} index out of range")
        if np.any(np.diff(idx) <= 0):
            raise ValueError(f"{what} indices must be sorted and duplicate-free")
    h = _lib.P()
    d.ctx.call("mg_extract", d.h, _lib.ptr(rows), int(rows.size), _lib.ptr(cols), int(cols.size),
               _lib.ctypes.byref(h))
    return DeviceMatrix(d.ctx, h)


def block_scale(a_bsr: DeviceMatrix, equilibrate: bool = True):
    """(G, Ahat = G A), G = Lambda D^-1 per cell, diagonal blocks exactly diag(Lambda)
    (SURVEY.md §7 D2/D3 plus the row equilibration of DESIGN.md §4)."""
    d, ah = _lib.P(), _lib.P()
    a_bsr.ctx.call("mg_block_scale", a_bsr.h, int(bool(equilibrate)), _lib.ctypes.byref(d),
                   _lib.ctypes.byref(ah))
    return DeviceMatrix(a_bsr.ctx, d), DeviceMatrix(a_bsr.ctx, ah)


def block_apply(dinv: DeviceMatrix, v) -> np.ndarray:
    v = _lib.f64(v)
    z = np.empty_like(v)
    dinv.ctx.call("mg_block_apply", dinv.h, _lib.ptr(v), _lib.ptr(z))
    return z


def equilibrate(a: DeviceMatrix):
    """Symmetric infinity-norm equilibration on the device (linsolve.py:107-122).

    Returns (scaled DeviceMatrix, row, col_scale): scaled = (diag(1/row) A) diag(col_scale)
    with exact zeros dropped; divide the rhs by ``row``, multiply the solution by
    ``col_scale``."""
    n = a.nrows
    row = np.empty(n)
    col = np.empty(n)
    h = _lib.P()
    a.ctx.call("mg_equilibrate", a.h, _lib.ctypes.byref(h), _lib.ptr(row), _lib.ptr(col))
    return DeviceMatrix(a.ctx, h), row, col


def abs_row_sum_max(a: DeviceMatrix) -> float:
    """max_i sum_j |a_ij| (the ``a_norm`` GmresSolver passes to gmres, linsolve.py:97-98)."""
    out = _lib.ctypes.c_double()
    a.ctx.call("mg_abs_row_sum_max", a.h, _lib.ctypes.byref(out))
    return float(out.value)


# -- Matrix Market I/O (sparse.py:256-264) -------------------------------------
def read_matrix_market(path, ctx=None) -> DeviceMatrix:
    """Load a Matrix Market file (e.g. the Jacobians _DumpingSolver writes,
    bench.py:286-300) straight into a device matrix."""
    import scipy.io
    import scipy.sparse as sp
    return DeviceMatrix.from_host(sp.csr_matrix(scipy.io.mmread(path, spmatrix=False)), ctx)


def write_matrix_market(path, a, comment=""):
    """Write a device (or host) matrix as a Matrix Market coordinate file."""
    import scipy.io
    m = a.to_scipy() if isinstance(a, DeviceMatrix) else (a.m if hasattr(a, "m") else a)
    scipy.io.mmwrite(path, m.tocoo(), comment=comment)


def to_cell_major(v, b):
    """x_cell[cell * b + var] = x_var[var * N + cell]"""
    v = np.asarray(v)
    return np.ascontiguousarray(v.reshape(b, -1).T).reshape(-1)


def to_var_major(v, b):
    """inverse of to_cell_major"""
    v = np.asarray(v)
    return np.ascontiguousarray(v.reshape(-1, b).T).reshape(-1)
