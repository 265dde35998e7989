// Dense coarsest-level solve: explicit inverse by Gauss-Jordan with partial
// pivoting at setup, one dense matvec per apply.
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

int dense_inverse(const double *a_dev, double *inv_dev, int n) {
  if (n == 0) return -1;
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

// y = M x, one warp per row
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

void dense_matvec(const double *m_dev, const double *x, double *y, int n) {
  if (!n) return;
  launch_pdl(k_dense_mv, grid_for((int64_t)n * 32, 256), 256, 0, m_dev, x, y, n);
  check_launch("dense_mv");
}

}  // namespace mg
