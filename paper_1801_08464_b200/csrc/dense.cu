// Dense coarsest-level solve: explicit inverse at setup (blocked Gauss-Jordan for
// n > 256, Gauss-Jordan with partial pivoting otherwise or when the blocked form
// meets a bad pivot), one dense matvec per apply.
//
// Replaces scipy.linalg.lu_factor / lu_solve at the AMG coarsest level
// (amg.py:330-343, n <= max(cutoff, 200)) and the small direct solves of
// coarse="exact" / FRelax("exact") / RpKind.IDEAL (mgr.py:127-131, 204-209,
// 306-307).  Pivot choice follows LAPACK getrf (first index of max |a_ik|).
#include "ops.cuh"

namespace mg {

// ---- single-CTA Gauss-Jordan for small n (augmented [A | I] in global) ----
__global__ void __launch_bounds__(1024) k_gj_small(double *aug, int n, int *bad) {
  const int w = 2 * n;
  __shared__ double sval[32];
  __shared__ int sidx[32];
  __shared__ int piv;
  __shared__ double pval;
  for (int k = 0; k < n; ++k) {
    // argmax |aug[i][k]|, i in [k, n)
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      double v = fabs(aug[(int64_t)i * w + k]);
      if (v > best) { best = v; bi = i; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_down_sync(0xffffffffu, best, off);
      int oi = __shfl_down_sync(0xffffffffu, bi, off);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { sval[threadIdx.x >> 5] = best; sidx[threadIdx.x >> 5] = bi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = -1.0; int ii = n;
      int nw = (blockDim.x + 31) / 32;
      for (int q = 0; q < nw; ++q)
        if (sval[q] > b || (sval[q] == b && sidx[q] < ii)) { b = sval[q]; ii = sidx[q]; }
      piv = ii;
      pval = (ii < n) ? aug[(int64_t)ii * w + k] : 0.0;
      if (!(fabs(pval) > 1e-300) && *bad < 0) *bad = k;
    }
    __syncthreads();
    if (*bad >= 0) return;
    int p = piv;
    double pv = pval;
    if (p != k)
      for (int j = threadIdx.x; j < w; j += blockDim.x) {
        double t = aug[(int64_t)k * w + j];
        aug[(int64_t)k * w + j] = aug[(int64_t)p * w + j];
        aug[(int64_t)p * w + j] = t;
      }
    __syncthreads();
    for (int j = threadIdx.x; j < w; j += blockDim.x) aug[(int64_t)k * w + j] /= pv;
    __syncthreads();
    // eliminate column k from every other row
    for (int64_t t = threadIdx.x; t < (int64_t)n * w; t += blockDim.x) {
      int i = (int)(t / w), j = (int)(t % w);
      if (i == k || j == k) continue;
      double f = aug[(int64_t)i * w + k];
      if (f != 0.0) aug[(int64_t)i * w + j] -= f * aug[(int64_t)k * w + j];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x)
      if (i != k) aug[(int64_t)i * w + k] = 0.0;
    __syncthreads();
  }
}

// ---- multi-block variant for larger n: one launch per elimination phase ----
__global__ void k_gj_pivot(double *aug, int n, int k, int *pivot, int *bad, double *pvbuf) {
  const int w = 2 * n;
  __shared__ double sval[32];
  __shared__ int sidx[32];
  double best = -1.0;
  int bi = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    double v = fabs(aug[(int64_t)i * w + k]);
    if (v > best) { best = v; bi = i; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_down_sync(0xffffffffu, best, off);
    int oi = __shfl_down_sync(0xffffffffu, bi, off);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if ((threadIdx.x & 31) == 0) { sval[threadIdx.x >> 5] = best; sidx[threadIdx.x >> 5] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double b = -1.0; int ii = n;
    for (int q = 0; q < (int)(blockDim.x + 31) / 32; ++q)
      if (sval[q] > b || (sval[q] == b && sidx[q] < ii)) { b = sval[q]; ii = sidx[q]; }
    *pivot = ii;
    double pv = ii < n ? aug[(int64_t)ii * w + k] : 0.0;
    *pvbuf = pv;
    if (!(fabs(pv) > 1e-300) && *bad < 0) *bad = k;
  }
}
__global__ void k_gj_swapscale(double *aug, int n, int k, const int *pivot, const int *bad,
                               const double *pvbuf) {
  if (*bad >= 0) return;
  const int w = 2 * n;
  int p = *pivot;
  double pv = *pvbuf;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < w; j += gridDim.x * blockDim.x) {
    double a = aug[(int64_t)k * w + j], b = aug[(int64_t)p * w + j];
    if (p != k) aug[(int64_t)p * w + j] = a;
    aug[(int64_t)k * w + j] = b / pv;
  }
}
__global__ void k_gj_elim(double *aug, const double *rowk, const double *colk, int n, int k, const int *bad) {
  if (*bad >= 0) return;
  const int w = 2 * n;
  int64_t total = (int64_t)n * w;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / w), j = (int)(t % w);
    if (i == k) continue;
    double f = colk[i];
    if (j == k) aug[t] = 0.0;
    else if (f != 0.0) aug[t] -= f * rowk[j];
  }
}
__global__ void k_gj_snap(const double *aug, double *rowk, double *colk, int n, int k) {
  const int w = 2 * n;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < w; j += gridDim.x * blockDim.x) {
    rowk[j] = aug[(int64_t)k * w + j];
    if (j < n) colk[j] = aug[(int64_t)j * w + k];
  }
}

__global__ void k_aug_init(const double *a, double *aug, int n) {
  int64_t total = (int64_t)n * 2 * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / (2 * n)), j = (int)(t % (2 * n));
    aug[t] = j < n ? a[(int64_t)i * n + j] : (j - n == i ? 1.0 : 0.0);
  }
}
__global__ void k_aug_extract(const double *aug, double *inv, int n) {
  int64_t total = (int64_t)n * n;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    int i = (int)(t / n), j = (int)(t % n);
    inv[t] = aug[(int64_t)i * 2 * n + n + j];
  }
}

// ---- blocked in-place Gauss-Jordan without pivoting (n > 256) --------------------
// Block pivot K = [k0, k0 + 32):  D = M_KK^-1 (one CTA, in shared memory);
// M_Kj <- D M_Kj (j not in K);  M_ij -= M_iK M_Kj (i, j not in K);
// M_iK <- -M_iK D (i not in K);  M_KK <- D.  After the last panel M = A^-1.
// A 32-column rank update per panel instead of one full pass over [A | I] per
// column: ~2n^3 flops and n/32 x 4 launches (n = 2048: 64 panels) instead of
// 4n launches.  No pivoting: a pivot that is tiny against its row in the
// diagonal block (|p| < 1e-10 max|row|) aborts, and dense_inverse falls back to
// the partially pivoted Gauss-Jordan above (the AMG coarsest operators and
// the small MGR F blocks are diagonally dominant in practice).
constexpr int BGJ = 32;

// the diagonal block D = M_KK inverted by one CTA of 32 x 32 threads, one element
// each, held in a register (warp r = row r).  Step k: warp k alone forms 1/p and its
// scaled row rks = D[k][c] / p and publishes both in shared memory (double-buffered:
// one barrier per step, 32 divisions per step instead of 1024 on the FP64 pipe); every
// thread takes its column entry D[r][k] from lane k of its own warp.  The arithmetic
// per element is unchanged (rks = D[k][c] * (1/p), D[r][c] -= D[r][k] * rks).
__global__ void __launch_bounds__(BGJ * BGJ) k_bgj_diag(const double *m, int n, int k0, double *dinv, int *bad) {
  PDL_ENTRY();
  __shared__ double prow[2][BGJ + 1];
  const int c = threadIdx.x, r = threadIdx.y;
  const int nb = min(BGJ, n - k0);
  double a = (r < nb && c < nb) ? m[(int64_t)(k0 + r) * n + k0 + c] : (r == c ? 1.0 : 0.0);
#pragma unroll 1
  for (int k = 0; k < BGJ; ++k) {
    double *pr = prow[k & 1];
    if (r == k) {  // warp k holds row k: the pivot test against the row's largest entry
      const double p = __shfl_sync(0xffffffffu, a, k);
      double amax = fabs(a);
      for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      if (c == 0 && (!(fabs(p) > 1e-10 * amax) || !(fabs(p) > 1e-300))) atomicCAS(bad, -1, k0 + k);
      const double ip = 1.0 / p;
      pr[c] = a * ip;
      if (c == 0) pr[BGJ] = ip;
    }
    __syncthreads();
    const double rks = pr[c];
    const double ip = pr[BGJ];
    const double ci = __shfl_sync(0xffffffffu, a, k);  // D[r][k]
    if (c == k) a = (r == k) ? ip : -ci * ip;
    else if (r == k) a = rks;
    else a = a - ci * rks;
  }
  dinv[r * BGJ + c] = a;
}

// M_Kj <- D M_Kj for j outside K: one thread per column j (coalesced across j);
// 64-thread CTAs so that the panel's FP64 work spreads over n / 64 SMs
constexpr int BGJ_PT = 64;
__global__ void __launch_bounds__(BGJ_PT) k_bgj_rowpanel(double *m, int n, int k0, const double *dinv,
                                                         const int *bad) {
  PDL_ENTRY();
  if (*bad >= 0) return;
  __shared__ double d[BGJ][BGJ];
  for (int t = threadIdx.x; t < BGJ * BGJ; t += blockDim.x) d[t / BGJ][t % BGJ] = dinv[t];
  __syncthreads();
  const int nb = min(BGJ, n - k0);
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n || (j >= k0 && j < k0 + nb)) return;
  double x[BGJ];
#pragma unroll
  for (int k = 0; k < BGJ; ++k) x[k] = k < nb ? m[(int64_t)(k0 + k) * n + j] : 0.0;
#pragma unroll 4
  for (int r = 0; r < nb; ++r) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < BGJ; ++k) s += d[r][k] * x[k];
    m[(int64_t)(k0 + r) * n + j] = s;
  }
}

// M_ij -= M_iK M_Kj for i, j outside K: 64 x 64 output tile per CTA, 4 x 4 per thread
__global__ void __launch_bounds__(256) k_bgj_update(double *m, int n, int k0, const int *bad) {
  PDL_ENTRY();
  if (*bad >= 0) return;
  __shared__ double a[64][BGJ + 1];
  __shared__ double b[BGJ][64 + 1];
  const int nb = min(BGJ, n - k0);
  const int i0 = blockIdx.y * 64, j0 = blockIdx.x * 64;
  for (int t = threadIdx.x; t < 64 * BGJ; t += 256) {
    const int ii = t / BGJ, kk = t % BGJ;
    const int i = i0 + ii;
    a[ii][kk] = (i < n && kk < nb) ? m[(int64_t)i * n + k0 + kk] : 0.0;
    const int kb = t / 64, jj = t % 64;
    const int j = j0 + jj;
    b[kb][jj] = (j < n && kb < nb) ? m[(int64_t)(k0 + kb) * n + j] : 0.0;
  }
  __syncthreads();
  const int tr = threadIdx.x / 16, tc = threadIdx.x % 16;
  double acc[4][4] = {};
#pragma unroll 8
  for (int k = 0; k < BGJ; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { av[u] = a[tr + 16 * u][k]; bv[u] = b[k][tc + 16 * u]; }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] += av[u] * bv[v];
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + tr + 16 * u;
    if (i >= n || (i >= k0 && i < k0 + nb)) continue;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int j = j0 + tc + 16 * v;
      if (j >= n || (j >= k0 && j < k0 + nb)) continue;
      m[(int64_t)i * n + j] -= acc[u][v];
    }
  }
}

// M_iK <- -M_iK D (i outside K), M_KK <- D: one thread per row
__global__ void __launch_bounds__(BGJ_PT) k_bgj_colpanel(double *m, int n, int k0, const double *dinv,
                                                         const int *bad) {
  PDL_ENTRY();
  if (*bad >= 0) return;
  __shared__ double d[BGJ][BGJ];
  for (int t = threadIdx.x; t < BGJ * BGJ; t += blockDim.x) d[t / BGJ][t % BGJ] = dinv[t];
  __syncthreads();
  const int nb = min(BGJ, n - k0);
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double *row = m + (int64_t)i * n + k0;
  if (i >= k0 && i < k0 + nb) {
    for (int c = 0; c < nb; ++c) row[c] = d[i - k0][c];
    return;
  }
  double x[BGJ];
#pragma unroll
  for (int k = 0; k < BGJ; ++k) x[k] = k < nb ? row[k] : 0.0;
  for (int c = 0; c < nb; ++c) {
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < BGJ; ++k) s += x[k] * d[k][c];
    row[c] = -s;
  }
}

// n > 256: returns -1 on success, else the global index of a rejected pivot
static int blocked_gj(const double *a_dev, double *inv_dev, int n) {
  DBuf<double> dinv(BGJ * BGJ);
  DBuf<int> bad(1);
  dset_i32(bad.p, {-1});
  MG_CUDA(cudaMemcpyAsync(inv_dev, a_dev, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, stream()));
  const dim3 tiles((n + 63) / 64, (n + 63) / 64);
  for (int k0 = 0; k0 < n; k0 += BGJ) {
    // programmatic dependent launch: each kernel waits for its predecessor's
    // completion on the device, its launch latency hidden behind it
    launch_pdl(k_bgj_diag, dim3(1), dim3(BGJ, BGJ), 0, (const double *)inv_dev, n, k0, dinv.p, bad.p);
    launch_pdl(k_bgj_rowpanel, dim3((n + BGJ_PT - 1) / BGJ_PT), dim3(BGJ_PT), 0, inv_dev, n, k0,
               (const double *)dinv.p, (const int *)bad.p);
    launch_pdl(k_bgj_update, tiles, dim3(256), 0, inv_dev, n, k0, (const int *)bad.p);
    launch_pdl(k_bgj_colpanel, dim3((n + BGJ_PT - 1) / BGJ_PT), dim3(BGJ_PT), 0, inv_dev, n, k0,
               (const double *)dinv.p, (const int *)bad.p);
    check_launch("blocked gj");
    count_launch(3);
  }
  int hb = -1;
  d2h(&hb, bad.p, sizeof(int));
  return hb;
}

int dense_inverse(const double *a_dev, double *inv_dev, int n) {
  if (n == 0) return -1;
  if (n > 256 && blocked_gj(a_dev, inv_dev, n) < 0) return -1;
  // small n, or a pivot the unpivoted blocked form rejected: Gauss-Jordan on
  // [A | I] with partial pivoting
  DBuf<double> aug((size_t)n * 2 * n);
  DBuf<int> flags(2);
  dset_i32(flags.p, {0, -1});
  k_aug_init<<<grid_for((int64_t)n * 2 * n, 256, 4096), 256, 0, stream()>>>(a_dev, aug.p, n);
  check_launch("aug_init");
  if (n <= 256) {
    k_gj_small<<<1, 1024, 0, stream()>>>(aug.p, n, flags.p + 1);
    check_launch("gj_small");
  } else {
    DBuf<double> rowk((size_t)2 * n), colk((size_t)n), pvbuf(1);
    int gb = grid_for((int64_t)n * 2 * n, 256, g_ctx->num_sms * 8);
    for (int k = 0; k < n; ++k) {
      k_gj_pivot<<<1, 1024, 0, stream()>>>(aug.p, n, k, flags.p, flags.p + 1, pvbuf.p);
      k_gj_swapscale<<<grid_for(2 * n, 256), 256, 0, stream()>>>(aug.p, n, k, flags.p, flags.p + 1,
                                                                  pvbuf.p);
      k_gj_snap<<<grid_for(2 * n, 256), 256, 0, stream()>>>(aug.p, rowk.p, colk.p, n, k);
      k_gj_elim<<<gb, 256, 0, stream()>>>(aug.p, rowk.p, colk.p, n, k, flags.p + 1);
      check_launch("gj step");
      count_launch(3);
    }
  }
  int hf[2];
  d2h(hf, flags.p, sizeof(hf));
  if (hf[1] >= 0) return hf[1];
  k_aug_extract<<<grid_for((int64_t)n * n, 256, 4096), 256, 0, stream()>>>(aug.p, inv_dev, n);
  check_launch("aug_extract");
  return -1;
}

// y = M x: small n one warp per row; larger n (the coarsest levels of a few
// thousand rows, L2-resident) four warps per row with the partial sums combined
// in shared memory, so the grid fills the SMs.
__global__ void k_dense_mv(const double *__restrict__ m, const double *__restrict__ x, double *y, int n) {
  PDL_ENTRY();
  int row = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  double s = 0.0;
  if (row < n)
    for (int j = lane; j < n; j += 32) s += m[(int64_t)row * n + j] * x[j];
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (row < n && lane == 0) y[row] = s;
}
__global__ void __launch_bounds__(256) k_dense_mv4(const double *__restrict__ m, const double *__restrict__ x,
                                                   double *y, int n) {
  PDL_ENTRY();
  __shared__ double part[8];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 2 + (w >> 2), seg = w & 3;
  double s = 0.0;
  if (row < n) {
    const double *mr = m + (int64_t)row * n;
    for (int j = seg * 32 + lane; j < n; j += 128) s += mr[j] * x[j];
  }
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) part[w] = s;
  __syncthreads();
  if (threadIdx.x < 2) {
    const int r = blockIdx.x * 2 + threadIdx.x;
    if (r < n) y[r] = (part[threadIdx.x * 4] + part[threadIdx.x * 4 + 1]) + (part[threadIdx.x * 4 + 2] + part[threadIdx.x * 4 + 3]);
  }
}

void dense_matvec(const double *m_dev, const double *x, double *y, int n) {
  if (!n) return;
  if (n >= 512) launch_pdl(k_dense_mv4, (n + 1) / 2, 256, 0, m_dev, x, y, n);
  else launch_pdl(k_dense_mv, grid_for((int64_t)n * 32, 256), 256, 0, m_dev, x, y, n);
  check_launch("dense_mv");
}

}  // namespace mg
