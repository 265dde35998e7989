"""Throughput of the GPU Newton assembly (residual + Jacobian + COO merge) on a
structured grid (no-flux boundaries, Van Genuchten models, mixed gas state).

usage: python tools/asm_bench.py [EDGE] [reps]
The static problem mirrors ncpflow.grid.build_grid / interior_transmissibilities
(x-faces, then y, then z; harmonic-mean transmissibilities) so it runs without
the reference; parity is covered by tests/test_assembly_gpu.py.
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_1801_08464_b200 import _lib  # noqa: E402
from paper_1801_08464_b200.assembly import AssemblyProblem, GpuAssembler  # noqa: E402


def structured(nx, ny, nz, perm=1e-16):
    n = nx * ny * nz
    dx = dy = dz = 1.0
    cells = np.arange(n)
    i, j, k = cells % nx, (cells // nx) % ny, cells // (nx * ny)
    fa, fb, ta, tg = [], [], [], []
    for ax, (idx, lim, step, area, dist) in enumerate(((i, nx, 1, dy * dz, dx), (j, ny, nx, dx * dz, dy),
                                                       (k, nz, nx * ny, dx * dy, dz))):
        a = cells[idx < lim - 1]
        fa.append(a)
        fb.append(a + step)
        ta.append(np.full(a.size, perm * area / dist))
        tg.append(np.full(a.size, area / dist))
    z = np.zeros(0)
    zi = np.zeros(0, np.int32)
    mu_l, mu_g = 1e-9, 9e-6
    henry, molar_h, temp, r_gas = 7.65e-6, 2e-3, 303.0, 8.314
    return AssemblyProblem(
        n_cells=n, cell_volume=dx * dy * dz, phi=0.3, diff_lh=3e-9, mu_l=mu_l, mu_g=mu_g, rho_w_std=1e3,
        c_h=henry * molar_h, c_v=molar_h / (r_gas * temp),
        rp_van_genuchten=1, s_lr=0.01, s_gr=0.0, rp_m=1.0 - 1.0 / 1.54, rp_eps=1e-5,
        cp_van_genuchten=1, p_entry=2e6, cp_n=1.54, cp_m=1.0 - 1.0 / 1.54, cp_eps=1e-5,
        face_a=np.concatenate(fa).astype(np.int32), face_b=np.concatenate(fb).astype(np.int32),
        trans=np.concatenate(ta), tgeo=np.concatenate(tg), gdx=np.zeros(sum(x.size for x in fa)),
        dir_cell=zi, dir_rule=zi, dir_trans=z, dir_tgeo=z, dir_gdx=z, rule_p=z, rule_s=z, rule_rho=z, rule_pc=z,
        rule_dpc=z, rule_lam_l=z, rule_lam_g=z, neu_cell=zi, neu_w=z, neu_h=z)


class _S:
    def __init__(self, p, s, r):
        self.p_l, self.s_l, self.rho_lh = p, s, r


def main():
    edge = int(sys.argv[1]) if len(sys.argv) > 1 else 128
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    pb = structured(edge, edge, edge)
    n = pb.n_cells
    rng = np.random.default_rng(0)
    p = 1e6 + rng.uniform(-5e4, 5e4, n)
    s = rng.uniform(0.7, 0.9, n)
    inactive = rng.random(n) < 0.4
    s[inactive] = 1.0 + rng.uniform(0.0005, 0.002, inactive.sum())
    rho = np.where(inactive, 0.3 * pb.c_h * p, pb.c_h * p - 3e-4)
    st, old = _S(p, s, rho), _S(p - 100.0, s - 1e-3, rho * 0.99)
    ctx = _lib.ctx()
    asm = GpuAssembler(pb, ctx)
    for _ in range(2):
        sysm = asm.jacobian(st, old, 10.0)
        sysm.a.free()
    ctx.sync()
    t0 = time.perf_counter()
    for _ in range(reps):
        sysm = asm.jacobian(st, old, 10.0)
        ctx.sync()
        nnz = sysm.a.nnz
        sysm.a.free()
    ms = (time.perf_counter() - t0) * 1e3 / reps
    print(f"assembly {edge}^3: {n} cells, {3 * n} unknowns, Jacobian nnz {nnz}: {ms:.1f} ms per residual+Jacobian "
          f"(host state upload and residual download included), {3 * n / (ms * 1e-3) / 1e6:.1f} M unknowns/s")


if __name__ == "__main__":
    main()
