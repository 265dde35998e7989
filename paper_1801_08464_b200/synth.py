"""Seeded synthetic block-sparse NCP Jacobians (BASELINE.json configs 1-5).

The reference has no generator for these systems; BASELINE.json describes
them in prose and SURVEY.md §8(d) / §7 D1-D4 pins the readings it leaves
open.  Every pin is restated here because each one changes bits:

* Cells are numbered x-fastest, ``cell = ix + nx*iy + nx*ny*iz`` (as
  ``ncpflow/grid.py:3-5``); unit spacing; a face's transmissibility is the
  harmonic mean of the two cell permeabilities (``grid.py:131-138``),
  times 0.01 on z-faces for config 3.
* Draw order from ``np.random.default_rng(seed)``: k, lambda_t, lambda_g,
  p-noise, [D for b=3], rhs (rhs drawn variable-major, length b*N).
  ``p = (ix + 0.5)/nx + N(0, 0.01)`` (0.01 is the standard deviation).
* Face mobilities: arithmetic mean of the two cells for A_pp/A_ps/A_ss
  (and D for the rho rows); A_sp uses the upwind lambda_g (the cell with
  the larger p; ties pick the lower-index cell).
* D1: A_ps(i,i) = +0.1*sum_j T_ij lg_ij and, for gas cells,
  A_sp(i,i) = +sum_j T_ij lg_up (negated off-diagonal row sums) so per-cell
  blocks are nonsingular.
* Gas-absent S rows (b=2): only A_sp(i,i) = -0.01.  b=3: only A_srho(i,i)=1.
* Gas regions: configs 1/2/5 centred disc/sphere of radius 0.35*E (config-5
  sequence: + step cells); config 3 gas-absent where
  z < 0.3E + 0.05E sin(2 pi x/E) sin(2 pi y/E) (cell-centre coordinates,
  zero phase); config 4 gas-absent outside a centred sphere r = 0.4924*E.

The output is the cell-major block-CSR (b x b row-major blocks, block
columns ascending) that the GPU path consumes, plus the rhs in cell-major
order.  ``to_scalar_csr`` gives the equivalent scalar CSR in either the
cell-major or the reference's variable-major unknown order.

No public dataset is involved: these seeded systems stand in for the
BASELINE configs (DESIGN.md says so).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["BlockSystem", "make_config", "make_system", "to_scalar_csr",
           "CONFIG_EDGES", "mgr_f_indices"]


@dataclass
class BlockSystem:
    """Cell-major BCSR system ``A x = rhs``."""

    nx: int
    ny: int
    nz: int
    b: int
    rowptr: np.ndarray          # int32 [N+1]
    col: np.ndarray             # int32 [nnzb]
    vals: np.ndarray            # float64 [nnzb, b, b]
    rhs: np.ndarray             # float64 [N*b] cell-major
    gas: np.ndarray             # bool [N]
    meta: dict = field(default_factory=dict)

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz

    @property
    def n(self):
        return self.n_cells * self.b

    @property
    def nnzb(self):
        return int(self.col.size)


CONFIG_EDGES = {1: (64, 64, 1), 2: (64, 64, 64), 3: (128, 128, 128), 4: (96, 96, 96)}


def _harmonic(a, b):
    s = a + b
    out = np.zeros(np.broadcast(a, b).shape)
    nz = s != 0.0
    out[nz] = 2.0 * (a * b)[nz] / s[nz]
    return out


def _shift_lo(arr, ax):
    sl = [slice(None)] * 3
    sl[ax] = slice(0, -1)
    return arr[tuple(sl)]


def _shift_hi(arr, ax):
    sl = [slice(None)] * 3
    sl[ax] = slice(1, None)
    return arr[tuple(sl)]


def _pad(face, ax, where):
    """Embed a face array (len-1 along ax) into a cell array, zero-padded."""
    pad = [(0, 0)] * 3
    pad[ax] = (0, 1) if where == "plus" else (1, 0)
    return np.pad(face, pad)


def make_system(nx, ny, nz, *, b=2, seed=0, sigma=1.0, zfac=1.0,
                region="sphere", radius=None, step=0) -> BlockSystem:
    """Generate one seeded synthetic system (see module docstring)."""
    if b not in (2, 3):
        raise ValueError("b must be 2 or 3")
    shape = (nz, ny, nx)                    # numpy axes (z, y, x): x fastest
    N = nx * ny * nz
    rng = np.random.default_rng(seed + step)
    k = np.exp(sigma * rng.standard_normal(N)).reshape(shape)
    lt = rng.uniform(0.5, 2.0, N).reshape(shape)
    lg = rng.uniform(0.0, 1.0, N).reshape(shape)
    pnoise = rng.normal(0.0, 0.01, N).reshape(shape)
    dd = rng.uniform(0.1, 1.0, N).reshape(shape) if b == 3 else None
    rhs_var = rng.uniform(-1.0, 1.0, b * N)

    iz, iy, ix = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    xc, yc, zc = ix + 0.5, iy + 0.5, iz + 0.5
    p = xc / nx + pnoise

    E = float(nx)
    if region == "sphere":
        r = (0.35 * E if radius is None else radius * E) + step
        d2 = (xc - nx / 2) ** 2 + (yc - ny / 2) ** 2
        if nz > 1:
            d2 = d2 + (zc - nz / 2) ** 2
        gas = d2 < r * r
    elif region == "interface":
        zi = 0.3 * nz + 0.05 * nz * np.sin(2 * np.pi * xc / nx) * np.sin(2 * np.pi * yc / ny)
        gas = ~(zc < zi)
    else:
        raise ValueError(f"unknown region {region!r}")

    dims = (nx, ny, nz)
    # axis id (x=0,y=1,z=2) -> numpy axis
    np_ax = {0: 2, 1: 1, 2: 0}
    steps = {0: 1, 1: nx, 2: nx * ny}
    active_axes = [a for a in (0, 1, 2) if dims[a] > 1]
    # slot order gives ascending block columns: -z,-y,-x,self,+x,+y,+z
    slots = [(a, "minus") for a in reversed(active_axes)] + [(None, "self")] + \
            [(a, "plus") for a in active_axes]
    S = len(slots)
    mask = np.zeros((S,) + shape, dtype=bool)
    T = np.zeros((S,) + shape)
    LT = np.zeros((S,) + shape)
    LG = np.zeros((S,) + shape)
    UP = np.zeros((S,) + shape)
    DF = np.zeros((S,) + shape) if b == 3 else None
    for s, (a, side) in enumerate(slots):
        if a is None:
            continue
        ax = np_ax[a]
        t_face = _harmonic(_shift_lo(k, ax), _shift_hi(k, ax))
        if a == 2:
            t_face = t_face * zfac
        lt_face = 0.5 * (_shift_lo(lt, ax) + _shift_hi(lt, ax))
        lg_face = 0.5 * (_shift_lo(lg, ax) + _shift_hi(lg, ax))
        up_face = np.where(_shift_lo(p, ax) >= _shift_hi(p, ax),
                           _shift_lo(lg, ax), _shift_hi(lg, ax))
        ones = np.ones_like(t_face, dtype=bool)
        mask[s] = _pad(ones, ax, side)
        T[s] = _pad(t_face, ax, side)
        LT[s] = _pad(lt_face, ax, side)
        LG[s] = _pad(lg_face, ax, side)
        UP[s] = _pad(up_face, ax, side)
        if b == 3:
            d_face = 0.5 * (_shift_lo(dd, ax) + _shift_hi(dd, ax))
            DF[s] = _pad(d_face, ax, side)
    self_slot = len(active_axes)
    mask[self_slot] = True

    blk = np.zeros((S,) + shape + (b, b))
    tl, tg, tu = T * LT, T * LG, T * UP
    nb = [s for s in range(S) if s != self_slot]
    sum_tl = np.sum(tl[nb], axis=0)
    sum_tg = np.sum(tg[nb], axis=0)
    sum_tu = np.sum(tu[nb], axis=0)
    gas_s = gas[None]
    for s in nb:
        blk[s, ..., 0, 0] = -tl[s]
        blk[s, ..., 0, 1] = -0.1 * tg[s]
        blk[s, ..., 1, 0] = np.where(gas, -tu[s], 0.0)
        blk[s, ..., 1, 1] = np.where(gas, -tg[s], 0.0)
    blk[self_slot, ..., 0, 0] = sum_tl + 1e-3
    blk[self_slot, ..., 0, 1] = 0.1 * sum_tg
    if b == 2:
        blk[self_slot, ..., 1, 0] = np.where(gas, sum_tu, -0.01)
        blk[self_slot, ..., 1, 1] = np.where(gas, 1.0 + sum_tg, 0.0)
    else:
        blk[self_slot, ..., 1, 0] = np.where(gas, sum_tu, 0.0)
        blk[self_slot, ..., 1, 1] = np.where(gas, 1.0 + sum_tg, 0.0)
        blk[self_slot, ..., 1, 2] = np.where(gas, 0.0, 1.0)
        td = T * DF
        for s in nb:
            blk[s, ..., 2, 2] = -td[s]
        blk[self_slot, ..., 2, 2] = 1.0 + np.sum(td[nb], axis=0)
        blk[self_slot, ..., 2, 0] = -0.01
    del gas_s

    # flatten to cell-major BCSR: iterate cells, then slots
    mask_c = mask.reshape(S, N).T                      # (N, S)
    offsets = np.array([(-steps[a] if side == "minus" else steps[a]) if a is not None else 0
                        for a, side in slots], dtype=np.int64)
    cell = np.arange(N, dtype=np.int64)
    colm = cell[:, None] + offsets[None, :]
    col = colm[mask_c].astype(np.int32)
    vals = blk.reshape(S, N, b, b).transpose(1, 0, 2, 3)[mask_c]
    counts = mask_c.sum(axis=1)
    rowptr = np.zeros(N + 1, dtype=np.int32)
    np.cumsum(counts, out=rowptr[1:])
    rhs = rhs_var.reshape(b, N).T.reshape(-1).copy()
    return BlockSystem(nx=nx, ny=ny, nz=nz, b=b, rowptr=rowptr, col=col,
                       vals=np.ascontiguousarray(vals), rhs=rhs,
                       gas=gas.reshape(-1).copy(),
                       meta=dict(seed=seed, step=step, sigma=sigma, zfac=zfac,
                                 region=region, radius=radius))


def make_config(config: int, edge: int | None = None, *, seed=0, step=0) -> BlockSystem:
    """BASELINE.json config 1..5 (config 5 = config-2 generator at cube ``edge``).

    ``edge`` overrides the grid size (same generator, smaller/larger grid),
    which the parity tests use to get oracle-sized cases of each config.
    """
    if config == 1:
        e = edge or 64
        return make_system(e, e, 1, b=2, seed=seed, step=step)
    if config in (2, 5):
        e = edge or 64
        return make_system(e, e, e, b=2, seed=seed, step=step)
    if config == 3:
        e = edge or 128
        return make_system(e, e, e, b=2, seed=seed, step=step, sigma=2.0, zfac=0.01,
                           region="interface")
    if config == 4:
        e = edge or 96
        return make_system(e, e, e, b=3, seed=seed, step=step, region="sphere",
                           radius=0.4924)
    raise ValueError(f"unknown config {config}")


def to_scalar_csr(sysm: BlockSystem, order="cell", drop_zeros=True):
    """Scalar CSR (indptr int32, indices int32, data f64) of the block matrix.

    ``order='cell'``: unknown ``cell*b + var``; ``order='var'``: the
    reference layout ``var*N + cell`` (``assembly.py:95-120``).
    """
    import scipy.sparse as sp
    N, b = sysm.n_cells, sysm.b
    nnzb = sysm.nnzb
    brow = np.repeat(np.arange(N, dtype=np.int64), np.diff(sysm.rowptr))
    bcol = sysm.col.astype(np.int64)
    r = np.arange(b)
    rows = (brow[:, None, None] * b + r[None, :, None]) + 0 * r[None, None, :]
    cols = (bcol[:, None, None] * b + r[None, None, :]) + 0 * r[None, :, None]
    vals = sysm.vals
    rows, cols, vals = rows.reshape(-1), cols.reshape(-1), vals.reshape(-1)
    if drop_zeros:
        keep = vals != 0.0
        rows, cols, vals = rows[keep], cols[keep], vals[keep]
    if order == "var":
        rows = (rows % b) * N + rows // b
        cols = (cols % b) * N + cols // b
    elif order != "cell":
        raise ValueError(order)
    m = sp.csr_matrix((vals, (rows, cols)), shape=(N * b, N * b))
    m.sum_duplicates()
    m.sort_indices()
    return m


def mgr_f_indices(b: int, N: int, order="cell"):
    """Level plan F sets for the synthetic systems (current-level local indices).

    b=2: [S].  b=3: [S, then rho].  Cell-major: S = cell*b+1; after S is
    removed the level is (p, rho) pairs, rho at odd local index.
    Variable-major: S = N..2N-1; then rho at N..2N-1 of the [p; rho] level.
    """
    cells = np.arange(N, dtype=np.int64)
    if order == "cell":
        if b == 2:
            return [cells * 2 + 1]
        return [cells * 3 + 1, cells * 2 + 1]
    if b == 2:
        return [N + cells]
    return [N + cells, N + cells]
