"""Oracle per-cell block inverse and block scaling (test infrastructure only).

Pins SURVEY.md §7 D2/D3 (the reference has no such step; its closest piece
is ``_BlockDiagSolver`` (mgr.py:212-242) which inverts per-cell blocks with
np.linalg.inv — tests compare against that at <= 1e-12):

* block inverse, closed form with a fixed operation order (no FMA):
  b=2  det = a00*a11 - a01*a10; inv = [[a11, -a01], [-a10, a00]] / det
  b=3  cofactor expansion along row 0, det = (a00*c00 + a01*c01) + a02*c02,
       inv_ij = adj_ij / det.
* scaled off-diagonal blocks  Ahat_ij[r][c] = sum_k Dinv_i[r][k]*A_ij[k][c]
  (k ascending, separate multiply/add); diagonal blocks are the exact
  identity (D3); the scalar CSR (cell-major unknown cell*b+var) keeps the
  diagonal 1.0 entries and drops off-diagonal-block entries equal to 0.0.
* prescale z_i = Dinv_i v_i (k ascending) — the first stage of
  M^-1 v = MGR_Ahat(D^-1 v).
* equilibration (default on): every "Dinv" above is G_i = Lambda_i D_i^-1,
  g[r][k] = lambda_r * dinv[r][k] with lambda_r = |A_ii[0][r]| (else the
  column max |A_ii[k][r]|); the pinned diagonal blocks become diag(lambda_i).
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp


class SingularBlock(RuntimeError):
    def __init__(self, cell):
        super().__init__(f"singular per-cell block at cell {cell}")
        self.cell = cell


def diag_blocks(sysm):
    N = sysm.n_cells
    brow = np.repeat(np.arange(N), np.diff(sysm.rowptr))
    is_d = sysm.col == brow
    if np.count_nonzero(is_d) != N:
        raise ValueError("every block row needs a diagonal block")
    return sysm.vals[is_d]


def block_inverse(blocks):
    a = blocks
    b = a.shape[1]
    inv = np.empty_like(a)
    if b == 2:
        det = a[:, 0, 0] * a[:, 1, 1] - a[:, 0, 1] * a[:, 1, 0]
        bad = np.where(det == 0.0)[0]
        if bad.size:
            raise SingularBlock(int(bad[0]))
        inv[:, 0, 0] = a[:, 1, 1] / det
        inv[:, 0, 1] = (-a[:, 0, 1]) / det
        inv[:, 1, 0] = (-a[:, 1, 0]) / det
        inv[:, 1, 1] = a[:, 0, 0] / det
        return inv
    if b == 3:
        g = lambda i, j: a[:, i, j]  # noqa: E731
        c00 = g(1, 1) * g(2, 2) - g(1, 2) * g(2, 1)
        c01 = g(1, 2) * g(2, 0) - g(1, 0) * g(2, 2)
        c02 = g(1, 0) * g(2, 1) - g(1, 1) * g(2, 0)
        det = (g(0, 0) * c00 + g(0, 1) * c01) + g(0, 2) * c02
        bad = np.where(det == 0.0)[0]
        if bad.size:
            raise SingularBlock(int(bad[0]))
        inv[:, 0, 0] = c00 / det
        inv[:, 1, 0] = c01 / det
        inv[:, 2, 0] = c02 / det
        inv[:, 0, 1] = (g(0, 2) * g(2, 1) - g(0, 1) * g(2, 2)) / det
        inv[:, 1, 1] = (g(0, 0) * g(2, 2) - g(0, 2) * g(2, 0)) / det
        inv[:, 2, 1] = (g(0, 1) * g(2, 0) - g(0, 0) * g(2, 1)) / det
        inv[:, 0, 2] = (g(0, 1) * g(1, 2) - g(0, 2) * g(1, 1)) / det
        inv[:, 1, 2] = (g(0, 2) * g(1, 0) - g(0, 0) * g(1, 2)) / det
        inv[:, 2, 2] = (g(0, 0) * g(1, 1) - g(0, 1) * g(1, 0)) / det
        return inv
    raise ValueError("b must be 2 or 3")


def _bmul(dl, a):
    """Per-block product with k ascending, separate multiply/add."""
    b = a.shape[1]
    out = np.empty_like(a)
    for r in range(b):
        for c in range(b):
            s = dl[:, r, 0] * a[:, 0, c]
            for k in range(1, b):
                s = s + dl[:, r, k] * a[:, k, c]
            out[:, r, c] = s
    return out


def row_scale(db):
    """Equilibration lambda_{i,r}: |A_ii[0][r]| (the pressure row's coefficient of
    variable r) when nonzero, else max_k |A_ii[k][r]|."""
    cm = np.abs(db).max(axis=1)
    pr = np.abs(db[:, 0, :])
    return np.where(pr != 0.0, pr, cm)


def prescale_blocks(sysm, equilibrate=True):
    """G_i = Lambda_i D_i^-1 (g[r][k] = lambda_r * dinv[r][k]); plain D^-1 without equilibration."""
    db = diag_blocks(sysm)
    dinv = block_inverse(db)
    if not equilibrate:
        return dinv, np.ones(db.shape[:2])
    lam = row_scale(db)
    return lam[:, :, None] * dinv, lam


def block_scale(sysm, equilibrate=True):
    """(G [N,b,b], Ahat scalar CSR cell-major) per the pinned rules.

    Ahat = G A with G = Lambda D^-1: off-diagonal blocks G_i A_ij (k ascending,
    separate multiply/add), diagonal blocks exactly diag(lambda_i) (D3).  The
    equilibration Lambda undoes the row normalisation of D^-1 so each row keeps
    its physical scale; without it the row-normalised Laplacian blocks make
    Galerkin R = P^T AMG diverge on config 3.
    """
    N, b = sysm.n_cells, sysm.b
    g, lam = prescale_blocks(sysm, equilibrate)
    dinv = g
    brow = np.repeat(np.arange(N), np.diff(sysm.rowptr))
    scaled = _bmul(dinv[brow], sysm.vals)
    is_d = sysm.col == brow
    scaled[is_d] = lam[:, :, None] * np.eye(b)[None]
    rr = np.arange(b)
    rows = (brow[:, None, None] * b + rr[None, :, None]) + 0 * rr[None, None, :]
    cols = (sysm.col.astype(np.int64)[:, None, None] * b + rr[None, None, :]) + 0 * rr[None, :, None]
    keep = scaled != 0.0
    keep[is_d] = np.eye(b, dtype=bool)
    m = sp.csr_matrix((scaled[keep], (rows[keep], cols[keep])), shape=(N * b, N * b))
    m.sort_indices()
    return dinv, m


def prescale(dinv, v):
    N, b = dinv.shape[0], dinv.shape[1]
    vv = np.asarray(v, dtype=float).reshape(N, b)
    out = np.empty_like(vv)
    for r in range(b):
        s = dinv[:, r, 0] * vv[:, 0]
        for k in range(1, b):
            s = s + dinv[:, r, k] * vv[:, k]
        out[:, r] = s
    return out.reshape(-1)
