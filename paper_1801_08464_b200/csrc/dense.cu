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

// ---- blocked Gauss-Jordan without pivoting (n > 256) -----------------------------
// Block pivot K = [k0, k0 + 32), D = M_KK^-1.  One panel step maps M to M':
//   M'_Kj = D M_Kj (j not in K);      M'_ij = M_ij - M_iK (D M_Kj) (i, j not in K);
//   M'_iK = -M_iK D (i not in K);     M'_KK = D.
// After the last panel M = A^-1.  A panel step is ONE launch, out of place between
// two n x n buffers (no read / write hazards between CTAs, so no separate row-panel,
// update and column-panel launches): every CTA forms its own 32 x 64 slice of
// D M_Kj in shared memory.  The next panel's diagonal block is updated and inverted
// by one extra CTA of the same launch (look-ahead), so the 32-step dependent chain of
// the small inverse runs beside the rank-32 update instead of between two launches:
// n / 32 dependent launches in all (n = 1708: 54 x ~20 us), chained by programmatic
// dependent launch.  ~3 n^3 FP64 multiply-adds, explicit fma (the inverse is compared
// with the oracle's LU solve to 1e-12, not bit for bit).  No pivoting: a pivot that is
// tiny against its row in the diagonal block (|p| < 1e-10 max|row|) aborts, and
// dense_inverse falls back to the partially pivoted Gauss-Jordan above (the AMG
// coarsest operators and the small MGR F blocks are diagonally dominant in practice).
constexpr int BGJ = 32;

// the first diagonal block D = M_KK inverted by one CTA of 32 x 32 threads, one element
// each, held in a register (warp r = row r).  Step k: warp k alone forms 1/p and its
// scaled row rks = D[k][c] / p and publishes both in shared memory (double-buffered:
// one barrier per step, 32 divisions per step instead of 1024 on the FP64 pipe); every
// thread takes its column entry D[r][k] from lane k of its own warp.
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
      // |p| > 1e-10 max_c |a_c|  <=>  |p| > 1e-10 |a_c| on every lane: one vote
      const bool ok = __all_sync(0xffffffffu, fabs(p) > 1e-10 * fabs(a)) && fabs(p) > 1e-300;
      if (c == 0 && !ok) atomicCAS(bad, -1, k0 + k);
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

// One panel step src -> dst (see above).  Block 0: look-ahead (the next diagonal
// block of dst, inverted into dnext); blocks 1..: 64 x 64 output tiles, 4 x 4 per
// thread.  256 threads.
__global__ void __launch_bounds__(256, 3) k_bgj_panel(const double *__restrict__ src, double *__restrict__ dst, int n,
                                                   int k0, const double *__restrict__ dcur, double *dnext,
                                                   int tiles_x, int *bad) {
  PDL_ENTRY();
  // the flag can be raised by this launch's own look-ahead CTA: one read per CTA,
  // so that a CTA leaves as a whole
  __shared__ int sbad;
  if (threadIdx.x == 0) sbad = *(volatile int *)bad;
  __syncthreads();
  if (sbad >= 0) return;
  __shared__ double sa[64][BGJ + 1];   // M_iK
  __shared__ double sb[BGJ][64 + 1];   // M_Kj, then D M_Kj (columns of K: D)
  __shared__ double sd[BGJ][BGJ + 1];  // D
  const int tid = threadIdx.x;
  const int nb = min(BGJ, n - k0);
  for (int t = tid; t < BGJ * BGJ; t += 256) sd[t / BGJ][t % BGJ] = dcur[t];
  if (blockIdx.x == 0) {
    // ---- look-ahead: U = M_R'R' - M_R'K (D M_KR'), R' = [k0 + 32, k0 + 32 + nbn), then U^-1
    const int r0 = k0 + BGJ;
    const int nbn = min(BGJ, n - r0);
    if (nbn <= 0) return;
    __shared__ double prow[2][BGJ + 1];
    for (int t = tid; t < BGJ * BGJ; t += 256) {
      const int r = t / BGJ, c = t % BGJ;
      sa[r][c] = (r < nbn && c < nb) ? src[(int64_t)(r0 + r) * n + k0 + c] : 0.0;
      sb[r][c] = (r < nb && c < nbn) ? src[(int64_t)(k0 + r) * n + r0 + c] : 0.0;
    }
    __syncthreads();
    const int w = tid >> 5, c = tid & 31;  // thread (w, c) holds rows q * 8 + w, column c
    double t4[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < BGJ; ++k) s = fma(sd[q * 8 + w][k], sb[k][c], s);
      t4[q] = s;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 4; ++q) sb[q * 8 + w][c] = t4[q];
    __syncthreads();
    double a[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int r = q * 8 + w;
      double s = 0.0;
#pragma unroll
      for (int k = 0; k < BGJ; ++k) s = fma(sa[r][k], sb[k][c], s);
      a[q] = (r < nbn && c < nbn) ? src[(int64_t)(r0 + r) * n + r0 + c] - s : (r == c ? 1.0 : 0.0);
    }
    // register-resident Gauss-Jordan (as k_bgj_diag, four rows per thread); fully
    // unrolled so that the owner slot k / 8 is a compile-time register index
#pragma unroll
    for (int k = 0; k < BGJ; ++k) {
      double *pr = prow[k & 1];
      if (w == (k & 7)) {
        const double ak = a[k >> 3];
        const double p = __shfl_sync(0xffffffffu, ak, k);
        const bool ok = __all_sync(0xffffffffu, fabs(p) > 1e-10 * fabs(ak)) && fabs(p) > 1e-300;
        if (c == 0 && !ok) atomicCAS(bad, -1, r0 + k);
        const double ip = 1.0 / p;
        pr[c] = ak * ip;
        if (c == 0) pr[BGJ] = ip;
      }
      __syncthreads();
      const double rks = pr[c];
      const double ip = pr[BGJ];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int r = q * 8 + w;
        const double ci = __shfl_sync(0xffffffffu, a[q], k);
        if (c == k) a[q] = (r == k) ? ip : -ci * ip;
        else if (r == k) a[q] = rks;
        else a[q] = a[q] - ci * rks;
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) dnext[(q * 8 + w) * BGJ + c] = a[q];
    return;
  }
  // ---- a 64 x 64 tile of dst
  const int tile = blockIdx.x - 1;
  const int i0 = (tile / tiles_x) * 64, j0 = (tile % tiles_x) * 64;
  for (int t = tid; t < 64 * BGJ; t += 256) {
    const int ii = t / BGJ, kk = t % BGJ;
    const int i = i0 + ii;
    sa[ii][kk] = (i < n && kk < nb) ? src[(int64_t)i * n + k0 + kk] : 0.0;
    const int kb = t / 64, jj = t % 64;
    const int j = j0 + jj;
    sb[kb][jj] = (j < n && kb < nb) ? src[(int64_t)(k0 + kb) * n + j] : 0.0;
  }
  __syncthreads();
  {
    // column jj of sb <- D * (column jj), columns of K <- D: 4 threads per column, 8 rows each
    const int jj = tid & 63, rg = tid >> 6;
    const int j = j0 + jj;
    const bool in_k = j >= k0 && j < k0 + nb;
    double out[8] = {};
#pragma unroll 8
    for (int k = 0; k < BGJ; ++k) {
      const double ck = sb[k][jj];
#pragma unroll
      for (int q = 0; q < 8; ++q) out[q] = fma(sd[rg * 8 + q][k], ck, out[q]);
    }
    if (in_k) {
#pragma unroll
      for (int q = 0; q < 8; ++q) out[q] = sd[rg * 8 + q][j - k0];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 8; ++q) sb[rg * 8 + q][jj] = out[q];
  }
  __syncthreads();
  const int tr = tid / 16, tc = tid % 16;
  double acc[4][4] = {};
#pragma unroll 8
  for (int k = 0; k < BGJ; ++k) {
    double av[4], bv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) { av[u] = sa[tr + 16 * u][k]; bv[u] = sb[k][tc + 16 * u]; }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int v = 0; v < 4; ++v) acc[u][v] = fma(av[u], bv[v], acc[u][v]);
  }
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int i = i0 + tr + 16 * u;
    if (i >= n) continue;
    const bool i_in_k = i >= k0 && i < k0 + nb;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int jj = tc + 16 * v, j = j0 + jj;
      if (j >= n) continue;
      const bool j_in_k = j >= k0 && j < k0 + nb;
      double o;
      if (i_in_k) o = sb[i - k0][jj];
      else o = (j_in_k ? 0.0 : src[(int64_t)i * n + j]) - acc[u][v];
      dst[(int64_t)i * n + j] = o;
    }
  }
}

// n > 256: returns -1 on success, else the global index of a rejected pivot
static int blocked_gj(const double *a_dev, double *inv_dev, int n) {
  DBuf<double> dinv(2 * BGJ * BGJ), tmp((size_t)n * n);
  DBuf<int> bad(1);
  dset_i32(bad.p, {-1});
  const int npan = (n + BGJ - 1) / BGJ;
  // panel p reads buf[p & 1] and writes buf[(p + 1) & 1]: the last one lands in inv_dev
  double *buf[2] = {(npan & 1) ? tmp.p : inv_dev, (npan & 1) ? inv_dev : tmp.p};
  MG_CUDA(cudaMemcpyAsync(buf[0], a_dev, sizeof(double) * (size_t)n * n, cudaMemcpyDeviceToDevice, stream()));
  launch_pdl(k_bgj_diag, dim3(1), dim3(BGJ, BGJ), 0, (const double *)buf[0], n, 0, dinv.p, bad.p);
  check_launch("blocked gj diag");
  const int tx = (n + 63) / 64;
  for (int p = 0; p < npan; ++p) {
    // programmatic dependent launch: each panel waits for its predecessor's
    // completion on the device, its launch latency hidden behind it
    launch_pdl(k_bgj_panel, dim3(1 + tx * tx), dim3(256), 0, (const double *)buf[p & 1], buf[(p + 1) & 1], n,
               p * BGJ, (const double *)(dinv.p + (p & 1) * BGJ * BGJ), dinv.p + ((p + 1) & 1) * BGJ * BGJ, tx,
               bad.p);
    check_launch("blocked gj panel");
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
