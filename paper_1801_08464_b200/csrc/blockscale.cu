// Per-cell block kernels: batched b x b inverses of the diagonal blocks held
// in registers, block scaling Ahat = D^-1 A (scalar CSR, cell-major), and the
// per-apply prescale z = D^-1 v.
//
// Reference counterpart: _BlockDiagSolver (mgr.py:212-242; np.linalg.inv per
// cell, batched einsum apply).  The pinned operation order (closed-form
// adjugate, k-ascending products, no FMA) is the one restated in
// oracle/blockscale.py, so Dinv and Ahat are bit-identical to the oracle
// (SURVEY.md §7 D2/D3).  HBM-bound: read 8 b^2 N (diagonal blocks) + write
// 8 b^2 N; scaling reads/writes every block once.
#include "ops.cuh"
#include "blockscale.cuh"

namespace mg {

template <int B>
__device__ __forceinline__ bool invert_block(const double *a, double *inv) {
  if (B == 2) {
    double det = __dsub_rn(__dmul_rn(a[0], a[3]), __dmul_rn(a[1], a[2]));
    if (det == 0.0) return false;
    inv[0] = __ddiv_rn(a[3], det);
    inv[1] = __ddiv_rn(-a[1], det);
    inv[2] = __ddiv_rn(-a[2], det);
    inv[3] = __ddiv_rn(a[0], det);
    return true;
  } else {
#define G(i, j) a[(i) * 3 + (j)]
    double c00 = __dsub_rn(__dmul_rn(G(1, 1), G(2, 2)), __dmul_rn(G(1, 2), G(2, 1)));
    double c01 = __dsub_rn(__dmul_rn(G(1, 2), G(2, 0)), __dmul_rn(G(1, 0), G(2, 2)));
    double c02 = __dsub_rn(__dmul_rn(G(1, 0), G(2, 1)), __dmul_rn(G(1, 1), G(2, 0)));
    double det = __dadd_rn(__dadd_rn(__dmul_rn(G(0, 0), c00), __dmul_rn(G(0, 1), c01)), __dmul_rn(G(0, 2), c02));
    if (det == 0.0) return false;
    inv[0 * 3 + 0] = __ddiv_rn(c00, det);
    inv[1 * 3 + 0] = __ddiv_rn(c01, det);
    inv[2 * 3 + 0] = __ddiv_rn(c02, det);
    inv[0 * 3 + 1] = __ddiv_rn(__dsub_rn(__dmul_rn(G(0, 2), G(2, 1)), __dmul_rn(G(0, 1), G(2, 2))), det);
    inv[1 * 3 + 1] = __ddiv_rn(__dsub_rn(__dmul_rn(G(0, 0), G(2, 2)), __dmul_rn(G(0, 2), G(2, 0))), det);
    inv[2 * 3 + 1] = __ddiv_rn(__dsub_rn(__dmul_rn(G(0, 1), G(2, 0)), __dmul_rn(G(0, 0), G(2, 1))), det);
    inv[0 * 3 + 2] = __ddiv_rn(__dsub_rn(__dmul_rn(G(0, 1), G(1, 2)), __dmul_rn(G(0, 2), G(1, 1))), det);
    inv[1 * 3 + 2] = __ddiv_rn(__dsub_rn(__dmul_rn(G(0, 2), G(1, 0)), __dmul_rn(G(0, 0), G(1, 2))), det);
    inv[2 * 3 + 2] = __ddiv_rn(__dsub_rn(__dmul_rn(G(0, 0), G(1, 1)), __dmul_rn(G(0, 1), G(1, 0))), det);
#undef G
    return true;
  }
}

// equilibration lambda_r = |a[0][r]| if nonzero else max_k |a[k][r]| (oracle row_scale)
template <int B>
__device__ __forceinline__ double lambda_of(const double *a, int r) {
  double p = fabs(a[r]);
  if (p != 0.0) return p;
  double m = 0.0;
#pragma unroll
  for (int k = 0; k < B; ++k) m = fmax(m, fabs(a[k * B + r]));
  return m;
}

// G_i = Lambda_i D_i^-1 (or D_i^-1 when !equil), one thread per cell
template <int B>
__global__ void k_block_inv(int N, const int *rp, const int *ci, const double *v, double *dinv,
                            int *bad, int equil) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  int dp = -1;
  for (int q = rp[i]; q < rp[i + 1]; ++q)
    if (ci[q] == i) { dp = q; break; }
  double a[B * B], inv[B * B];
  if (dp < 0) { atomicMin(bad, i); return; }
#pragma unroll
  for (int t = 0; t < B * B; ++t) a[t] = v[(int64_t)dp * B * B + t];
  if (!invert_block<B>(a, inv)) { atomicMin(bad, i); return; }
#pragma unroll
  for (int r = 0; r < B; ++r) {
    double lam = equil ? lambda_of<B>(a, r) : 1.0;
#pragma unroll
    for (int k = 0; k < B; ++k)
      dinv[(int64_t)i * B * B + r * B + k] = equil ? __dmul_rn(lam, inv[r * B + k]) : inv[r * B + k];
  }
}

// scaled entry (r, c) of block q in block row i: sum_k Dinv_i[r][k] * A_q[k][c]
template <int B>
__device__ __forceinline__ double scaled(const double *d, const double *a, int r, int c) {
  double s = __dmul_rn(d[r * B + 0], a[0 * B + c]);
#pragma unroll
  for (int k = 1; k < B; ++k) s = __dadd_rn(s, __dmul_rn(d[r * B + k], a[k * B + c]));
  return s;
}

// VS lanes per scalar row t = (cell i, var r), lane l takes blocks rp[i] + l,
// + VS, ...; entries keep (block, column) order through a group scan of the
// per-lane kept counts.  mode 0 count, mode 1 fill.
template <int B, int VS>
__global__ void k_scale_rows(int N, const int *rp, const int *ci, const double *v, const double *dinv,
                             int mode, int *cnt, const int *orp, int *oci, double *ov, int equil) {
  for (RowGroup<VS> g; g.row < (int64_t)N * B; g.next()) {
    const int64_t t = g.row;
    const int i = (int)(t / B), r = (int)(t % B);
    double d[B * B];
  #pragma unroll
    for (int q = 0; q < B * B; ++q) d[q] = dinv[(int64_t)i * B * B + q];
    const int qb = rp[i], qe = rp[i + 1];
    int64_t o = mode ? orp[t] : 0;
    int c0 = 0;
    for (int q0 = qb; q0 < qe; q0 += VS) {
      const int q = q0 + g.lane;
      int kept = 0;
      int cols[B];
      double vals[B];
      if (q < qe) {
        const int j = ci[q];
        const double *a = v + (int64_t)q * B * B;
        if (j == i) {
          cols[0] = i * B + r;
          vals[0] = equil ? lambda_of<B>(a, r) : 1.0;
          kept = 1;
        } else {
  #pragma unroll
          for (int c = 0; c < B; ++c) {
            double s = scaled<B>(d, a, r, c);
            if (s != 0.0) { cols[kept] = j * B + c; vals[kept] = s; ++kept; }
          }
        }
      }
      int incl = kept;
  #pragma unroll
      for (int off = 1; off < VS; off <<= 1) {
        int y = __shfl_up_sync(g.mask, incl, off, VS);
        if (g.lane >= off) incl += y;
      }
      if (mode) {
        const int64_t p = o + c0 + incl - kept;
  #pragma unroll
        for (int e = 0; e < B; ++e)
          if (e < kept) { oci[p + e] = cols[e]; ov[p + e] = vals[e]; }
      }
      c0 += g.bcast(incl, VS - 1);
    }
    if (!mode && g.lane == 0) cnt[t] = c0;
  }
}

template <int B>
__global__ void k_block_apply(int N, const double *__restrict__ dinv, const double *__restrict__ x,
                              double *__restrict__ z) {
  PDL_ENTRY();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  double d[B * B], xv[B];
#pragma unroll
  for (int q = 0; q < B * B; ++q) d[q] = dinv[(int64_t)i * B * B + q];
#pragma unroll
  for (int q = 0; q < B; ++q) xv[q] = x[(int64_t)i * B + q];
#pragma unroll
  for (int r = 0; r < B; ++r) {
    double s = __dmul_rn(d[r * B + 0], xv[0]);
#pragma unroll
    for (int k = 1; k < B; ++k) s = __dadd_rn(s, __dmul_rn(d[r * B + k], xv[k]));
    z[(int64_t)i * B + r] = s;
  }
}

template <int B>
__global__ void k_block_apply_ind(int N, const double *__restrict__ dinv, const double *const *xslot,
                                  double *__restrict__ z) {
  PDL_ENTRY();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const double *__restrict__ x = *xslot;
  double d[B * B], xv[B];
#pragma unroll
  for (int q = 0; q < B * B; ++q) d[q] = dinv[(int64_t)i * B * B + q];
#pragma unroll
  for (int q = 0; q < B; ++q) xv[q] = x[(int64_t)i * B + q];
#pragma unroll
  for (int r = 0; r < B; ++r) {
    double s = __dmul_rn(d[r * B + 0], xv[0]);
#pragma unroll
    for (int k = 1; k < B; ++k) s = __dadd_rn(s, __dmul_rn(d[r * B + k], xv[k]));
    z[(int64_t)i * B + r] = s;
  }
}

__global__ void k_set_ptr(const double **slot, const double *value) {
  PDL_ENTRY();
  *slot = value;
}

__global__ void k_diag_pattern(int N, int *rp, int *ci) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N) { rp[i] = i; ci[i] = i; }
  if (i == N) rp[N] = N;
}

void block_scale(const Csr &a, Csr &dinv, Csr &ahat, bool equil) {
  const int B = a.b;
  if (B != 2 && B != 3) throw MgError(MG_ERR_UNSUPPORTED, "block_scale: b must be 2 or 3");
  if (a.nr != a.nc) throw MgError(MG_ERR_DIM_MISMATCH, "block_scale: square block matrix required");
  int N = a.nr;
  int eq = equil ? 1 : 0;
  dinv.alloc(N, N, N, B);
  k_diag_pattern<<<grid_for((int64_t)N + 1, 256), 256, 0, stream()>>>(N, dinv.rp.p, dinv.ci.p);
  check_launch("diag_pattern");
  DBuf<int> bad(1);
  const int big = 0x7fffffff;
  dset_i32(bad.p, {big});
  if (B == 2)
    k_block_inv<2><<<grid_for(N, 256), 256, 0, stream()>>>(N, a.rp.p, a.ci.p, a.v.p, dinv.v.p, bad.p, eq);
  else
    k_block_inv<3><<<grid_for(N, 256), 256, 0, stream()>>>(N, a.rp.p, a.ci.p, a.v.p, dinv.v.p, bad.p, eq);
  check_launch("block_inv");
  int hb = 0;
  d2h(&hb, bad.p, sizeof(int));
  if (hb != big) throw MgError(MG_ERR_SINGULAR, "singular (or missing) diagonal block at cell " + std::to_string(hb), hb);
  int64_t n = (int64_t)N * B;
  DBuf<int> cnt((size_t)n);
  ahat.nr = ahat.nc = (int)n;
  ahat.b = 1;
  ahat.rp.alloc((size_t)n + 1);
  auto launch = [&](int mode, int *c, const int *orp, int *oci, double *ov) {
    if (B == 2)
      k_scale_rows<2, 8><<<rowgroup_grid(n * 8), 256, 0, stream()>>>(N, a.rp.p, a.ci.p, a.v.p, dinv.v.p, mode, c, orp,
                                                                    oci, ov, eq);
    else
      k_scale_rows<3, 8><<<rowgroup_grid(n * 8), 256, 0, stream()>>>(N, a.rp.p, a.ci.p, a.v.p, dinv.v.p, mode, c, orp,
                                                                    oci, ov, eq);
    check_launch("scale_rows");
  };
  launch(0, cnt.p, nullptr, nullptr, nullptr);
  ahat.nnz = exclusive_scan_i32_to_i32(cnt.p, ahat.rp.p, (int)n);
  ahat.ci.alloc((size_t)ahat.nnz);
  ahat.v.alloc((size_t)ahat.nnz);
  launch(1, nullptr, ahat.rp.p, ahat.ci.p, ahat.v.p);
}

void block_apply(const Csr &dinv, const double *x, double *z) {
  int N = dinv.nr;
  if (!N) return;
  if (dinv.b == 2)
    launch_pdl(k_block_apply<2>, grid_for(N, 256), 256, 0, N, dinv.v.p, x, z);
  else if (dinv.b == 3)
    launch_pdl(k_block_apply<3>, grid_for(N, 256), 256, 0, N, dinv.v.p, x, z);
  else
    throw MgError(MG_ERR_UNSUPPORTED, "block_apply: b must be 2 or 3");
  check_launch("block_apply");
}

void block_apply_indirect(const Csr &dinv, const double *const *xslot, double *z) {
  int N = dinv.nr;
  if (!N) return;
  if (dinv.b == 2)
    launch_pdl(k_block_apply_ind<2>, grid_for(N, 256), 256, 0, N, dinv.v.p, xslot, z);
  else if (dinv.b == 3)
    launch_pdl(k_block_apply_ind<3>, grid_for(N, 256), 256, 0, N, dinv.v.p, xslot, z);
  else
    throw MgError(MG_ERR_UNSUPPORTED, "block_apply: b must be 2 or 3");
  check_launch("block_apply_indirect");
}

void set_device_ptr(const double **slot, const double *value) {
  launch_pdl(k_set_ptr, 1, 1, 0, slot, value);
  check_launch("set_ptr");
}

}  // namespace mg

// ---- symmetric infinity-norm equilibration (GmresSolver._equilibrated) --------------
// Replaces linsolve.py:107-122 (scipy):
//   row = max_j |a_ij| (0 -> 1);  col = max_i (1/row_i) |a_ij| (0 -> 1)
//   scaled = (diags(1/row) @ a) @ diags(1/col): each value ((1/row_i) a_ij) (1/col_j),
//   two rounded products, exact zeros dropped after each product (csr_matmat)
namespace mg {
namespace {
__global__ void k_row_absmax(int n, const int *rp, const double *v, double *row) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  double m = 0.0;
  for (int q = rp[wid] + lane; q < rp[wid + 1]; q += 32) m = fmax(m, fabs(v[q]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) row[wid] = m == 0.0 ? 1.0 : m;
}
__global__ void k_col_absmax(int n, const int *rp, const int *ci, const double *v, const double *row,
                             unsigned long long *colbits) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  const double dr = __ddiv_rn(1.0, row[wid]);
  for (int q = rp[wid] + lane; q < rp[wid + 1]; q += 32) {
    double t = __dmul_rn(dr, fabs(v[q]));  // non-negative: bit order == value order
    if (t > 0.0) atomicMax(colbits + ci[q], (unsigned long long)__double_as_longlong(t));
  }
}
__global__ void k_col_scale(int n, const unsigned long long *colbits, double *colscale) {
  int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  double c = __longlong_as_double((long long)colbits[j]);
  colscale[j] = __ddiv_rn(1.0, c == 0.0 ? 1.0 : c);
}
__device__ __forceinline__ double eq_value(double a, double dr, double dc) {
  double t = __dmul_rn(dr, a);
  return t == 0.0 ? 0.0 : __dmul_rn(t, dc);
}
__global__ void k_eq_count(int n, const int *rp, const int *ci, const double *v, const double *row,
                           const double *colscale, int *cnt) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  const double dr = __ddiv_rn(1.0, row[wid]);
  int c = 0;
  for (int q = rp[wid] + lane; q < rp[wid + 1]; q += 32) c += eq_value(v[q], dr, colscale[ci[q]]) != 0.0;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if (lane == 0) cnt[wid] = c;
}
__global__ void k_eq_fill(int n, const int *rp, const int *ci, const double *v, const double *row,
                          const double *colscale, const int *orp, int *oci, double *ov) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  const double dr = __ddiv_rn(1.0, row[wid]);
  int o = orp[wid];
  for (int q0 = rp[wid]; q0 < rp[wid + 1]; q0 += 32) {
    int q = q0 + lane;
    double val = q < rp[wid + 1] ? eq_value(v[q], dr, colscale[ci[q]]) : 0.0;
    unsigned bal = __ballot_sync(0xffffffffu, val != 0.0);
    if (val != 0.0) {
      int p = o + __popc(bal & ((1u << lane) - 1));
      oci[p] = ci[q];
      ov[p] = val;
    }
    o += __popc(bal);
  }
}
__global__ void k_abs_row_sum_max(int n, const int *rp, const double *v, unsigned long long *out) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  double s = 0.0;
  for (int q = rp[wid] + lane; q < rp[wid + 1]; q += 32) s += fabs(v[q]);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0 && s > 0.0) atomicMax(out, (unsigned long long)__double_as_longlong(s));
}
}  // namespace

void equilibrate(const Csr &a, Csr &out, double *row_dev, double *colscale_dev) {
  if (a.b != 1 || a.nr != a.nc) throw MgError(MG_ERR_UNSUPPORTED, "equilibrate: square scalar CSR required");
  const int n = a.nr;
  out.nr = out.nc = n;
  out.b = 1;
  out.rp.alloc((size_t)n + 1);
  if (!n) {
    dzero(out.rp.p, sizeof(int));
    return;
  }
  const int g = grid_for((int64_t)n * 32, 256);
  k_row_absmax<<<g, 256, 0, stream()>>>(n, a.rp.p, a.v.p, row_dev);
  check_launch("row_absmax");
  DBuf<unsigned long long> colbits(n);
  dzero(colbits.p, sizeof(unsigned long long) * n);
  k_col_absmax<<<g, 256, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, row_dev, colbits.p);
  check_launch("col_absmax");
  k_col_scale<<<grid_for(n, 256), 256, 0, stream()>>>(n, colbits.p, colscale_dev);
  check_launch("col_scale");
  DBuf<int> cnt(n);
  k_eq_count<<<g, 256, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, row_dev, colscale_dev, cnt.p);
  check_launch("eq_count");
  out.nnz = exclusive_scan_i32_to_i32(cnt.p, out.rp.p, n);
  out.ci.alloc((size_t)out.nnz);
  out.v.alloc((size_t)out.nnz);
  k_eq_fill<<<g, 256, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, row_dev, colscale_dev, out.rp.p, out.ci.p,
                                     out.v.p);
  check_launch("eq_fill");
}

double abs_row_sum_max(const Csr &a) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "abs_row_sum_max: scalar CSR required");
  if (!a.nr) return 0.0;
  DBuf<unsigned long long> m(1);
  dzero(m.p, sizeof(unsigned long long));
  k_abs_row_sum_max<<<grid_for((int64_t)a.nr * 32, 256), 256, 0, stream()>>>(a.nr, a.rp.p, a.v.p, m.p);
  check_launch("abs_row_sum_max");
  unsigned long long h = 0;
  d2h(&h, m.p, sizeof(h));
  double r;
  memcpy(&r, &h, sizeof(r));
  return r;
}
}  // namespace mg
