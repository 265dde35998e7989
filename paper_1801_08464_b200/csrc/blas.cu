// Vector kernels and the fused CGS2 Arnoldi kernels for GMRES
// (krylov.py:101-109: c = V w; w -= c V; c' = V w; w -= c' V; h = ||w||).
//
// Reductions are two-stage with a fixed block count and fixed order, so every
// result is bitwise reproducible run to run.  The projection of step j reads
// the j+1 basis vectors once per pass: update_mdot fuses "w -= cV" with the
// re-orthogonalisation dot products and update_norm2 fuses the second
// subtraction with ||w||^2 (3 basis passes per Arnoldi step instead of 5).
#include "ops.cuh"

namespace mg {

static const int RB = 256;           // threads per reduction block
static int red_blocks(int64_t n) {
  int64_t b = (n + RB * 4 - 1) / (RB * 4);
  int cap = g_ctx->num_sms * 4;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

__global__ void k_fill(double *x, double val, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = val;
}
__global__ void k_mul(double *y, const double *a, const double *x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a[i] * x[i];
}
__global__ void k_axpy(double *y, double a, const double *x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = y[i] + a * x[i];
}
__global__ void k_add(double *y, const double *x, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = y[i] + x[i];
}
__global__ void k_divs(double *y, const double *x, double d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}
__global__ void k_sub(double *r, const double *b, const double *ax, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - ax[i];
}
__global__ void k_gather(double *d, const double *s, const int *idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[idx[i]];
}
__global__ void k_scatter_add(double *d, const double *s, const int *idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[idx[i]] = d[idx[i]] + s[i];
}
__global__ void k_scatter_set(double *d, const double *s, const int *idx, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[idx[i]] = s[i];
}

static int ew_grid(int64_t n) { return grid_for(n, 256, g_ctx->num_sms * 8); }

void vfill(double *x, double val, int64_t n) {
  if (!n) return;
  k_fill<<<ew_grid(n), 256, 0, stream()>>>(x, val, n);
  check_launch("fill");
}
void vcopy(double *dst, const double *src, int64_t n) { d2d(dst, src, n * sizeof(double)); }
void vmul(double *y, const double *a, const double *x, int64_t n) {
  if (!n) return;
  k_mul<<<ew_grid(n), 256, 0, stream()>>>(y, a, x, n);
  check_launch("mul");
}
void vaxpy(double *y, double a, const double *x, int64_t n) {
  if (!n) return;
  k_axpy<<<ew_grid(n), 256, 0, stream()>>>(y, a, x, n);
  check_launch("axpy");
}
void vadd(double *y, const double *x, int64_t n) {
  if (!n) return;
  k_add<<<ew_grid(n), 256, 0, stream()>>>(y, x, n);
  check_launch("add");
}
void vdiv_scalar(double *y, const double *x, double d, int64_t n) {
  if (!n) return;
  k_divs<<<ew_grid(n), 256, 0, stream()>>>(y, x, d, n);
  check_launch("div");
}
void vsub(double *r, const double *b, const double *ax, int64_t n) {
  if (!n) return;
  k_sub<<<ew_grid(n), 256, 0, stream()>>>(r, b, ax, n);
  check_launch("sub");
}
void gather(double *dst, const double *src, const int *idx, int64_t n) {
  if (!n) return;
  k_gather<<<ew_grid(n), 256, 0, stream()>>>(dst, src, idx, n);
  check_launch("gather");
}
void scatter_add(double *dst, const double *src, const int *idx, int64_t n) {
  if (!n) return;
  k_scatter_add<<<ew_grid(n), 256, 0, stream()>>>(dst, src, idx, n);
  check_launch("scatter_add");
}
void scatter_set(double *dst, const double *src, const int *idx, int64_t n) {
  if (!n) return;
  k_scatter_set<<<ew_grid(n), 256, 0, stream()>>>(dst, src, idx, n);
  check_launch("scatter_set");
}

// ---- block-level reduction of K values per thread -> partial[blockIdx][k] ----
template <int KM>
__device__ __forceinline__ void block_reduce_store(double (&acc)[KM], int K, double *partial) {
  __shared__ double sm[RB / 32][KM];
  int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    double s = acc[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
    if (lane == 0) sm[wid][k] = s;
  }
  __syncthreads();
  if (threadIdx.x < KM && (int)threadIdx.x < K) {
    double s = 0.0;
#pragma unroll
    for (int w = 0; w < RB / 32; ++w) s += sm[w][threadIdx.x];
    partial[(int64_t)blockIdx.x * K + threadIdx.x] = s;
  }
}

// out[k] = sum_b partial[b*K + k], one warp per k, fixed order
__global__ void k_finish(const double *partial, int nb, int K, double *out) {
  int k = blockIdx.x;
  int lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += partial[(int64_t)b * K + k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) out[k] = s;
}

__global__ void __launch_bounds__(RB) k_dot(const double *x, const double *y, int64_t n, double *partial) {
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
    acc[0] += x[i] * y[i];
  block_reduce_store<1>(acc, 1, partial);
}

static double reduce_finish(double *partial, int nb, int K, double *out_dev) {
  k_finish<<<K, 32, 0, stream()>>>(partial, nb, K, out_dev);
  check_launch("finish");
  return 0.0;
}

double dot(const double *x, const double *y, int64_t n) {
  int nb = red_blocks(n);
  double *part = red_scratch((size_t)nb + 8);
  double *out = part + nb;
  k_dot<<<nb, RB, 0, stream()>>>(x, y, n, part);
  check_launch("dot");
  reduce_finish(part, nb, 1, out);
  double h = 0.0;
  d2h(&h, out, sizeof(double));
  return h;
}

double nrm2(const double *x, int64_t n) { return sqrt(dot(x, x, n)); }

// partial projections of w onto V_0..V_{K-1} (K <= 32 per pass)
template <int KM>
__global__ void __launch_bounds__(RB) k_mdot(const double *__restrict__ V, int64_t ldv, int K,
                                            const double *__restrict__ w, int64_t n,
                                            double *partial) {
  double acc[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double wi = w[i];
#pragma unroll
    for (int k = 0; k < KM; ++k)
      if (k < K) acc[k] += V[k * ldv + i] * wi;
  }
  block_reduce_store<KM>(acc, K, partial);
}

// w -= sum c_k V_k ; then partial V^T w
template <int KM>
__global__ void __launch_bounds__(RB) k_update_mdot(const double *__restrict__ V, int64_t ldv, int K,
                                                   const double *__restrict__ c, double *w,
                                                   int64_t n, double *partial) {
  __shared__ double cc[KM];
  double acc[KM];
  if (threadIdx.x < KM) cc[threadIdx.x] = (int)threadIdx.x < K ? c[threadIdx.x] : 0.0;
  __syncthreads();
#pragma unroll
  for (int k = 0; k < KM; ++k) acc[k] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double vk[KM];
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < KM; ++k) {
      vk[k] = k < K ? V[k * ldv + i] : 0.0;
      t += cc[k] * vk[k];
    }
    double wi = w[i] - t;
    w[i] = wi;
#pragma unroll
    for (int k = 0; k < KM; ++k) acc[k] += vk[k] * wi;
  }
  block_reduce_store<KM>(acc, K, partial);
}

// w -= sum c_k V_k ; partial ||w||^2
template <int KM>
__global__ void __launch_bounds__(RB) k_update_norm(const double *__restrict__ V, int64_t ldv, int K,
                                                   const double *__restrict__ c, double *w,
                                                   int64_t n, double *partial) {
  double cc[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) cc[k] = k < K ? c[k] : 0.0;
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double t = 0.0;
#pragma unroll
    for (int k = 0; k < KM; ++k)
      if (k < K) t += cc[k] * V[k * ldv + i];
    double wi = w[i] - t;
    w[i] = wi;
    acc[0] += wi * wi;
  }
  block_reduce_store<1>(acc, 1, partial);
}

// u = sum y_k V_k (or u += when accumulate)
template <int KM>
__global__ void __launch_bounds__(RB) k_combine(const double *__restrict__ V, int64_t ldv, int K,
                                               const double *__restrict__ y, double *u, int64_t n,
                                               int accumulate) {
  double cc[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) cc[k] = k < K ? y[k] : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double t = accumulate ? u[i] : 0.0;
#pragma unroll
    for (int k = 0; k < KM; ++k)
      if (k < K) t += cc[k] * V[k * ldv + i];
    u[i] = t;
  }
}

#define KSEL(K, CALL16, CALL32) \
  do { if ((K) <= 16) { CALL16; } else { CALL32; } } while (0)

void mdot(const double *V, int64_t ldv, int K, const double *w, int64_t n, double *out_dev) {
  int nb = red_blocks(n);
  for (int k0 = 0; k0 < K; k0 += 32) {
    int kk = K - k0 < 32 ? K - k0 : 32;
    double *part = red_scratch((size_t)nb * 32);
    const double *Vk = V + (int64_t)k0 * ldv;
    KSEL(kk, (k_mdot<16><<<nb, RB, 0, stream()>>>(Vk, ldv, kk, w, n, part)),
         (k_mdot<32><<<nb, RB, 0, stream()>>>(Vk, ldv, kk, w, n, part)));
    check_launch("mdot");
    reduce_finish(part, nb, kk, out_dev + k0);
  }
}

void update_mdot(const double *V, int64_t ldv, int K, const double *c_dev, double *w, int64_t n,
                 double *out_dev) {
  int nb = red_blocks(n);
  if (K <= 32) {
    double *part = red_scratch((size_t)nb * 32);
    KSEL(K, (k_update_mdot<16><<<nb, RB, 0, stream()>>>(V, ldv, K, c_dev, w, n, part)),
         (k_update_mdot<32><<<nb, RB, 0, stream()>>>(V, ldv, K, c_dev, w, n, part)));
    check_launch("update_mdot");
    reduce_finish(part, nb, K, out_dev);
    return;
  }
  // long restarts: unfused (w -= cV chunk by chunk, then projections)
  DBuf<double> t((size_t)n);
  combine(V, ldv, K, c_dev, t.p, n);
  vaxpy(w, -1.0, t.p, n);
  mdot(V, ldv, K, w, n, out_dev);
}

void update_norm2(const double *V, int64_t ldv, int K, const double *c_dev, double *w, int64_t n,
                  double *out_dev) {
  int nb = red_blocks(n);
  double *part = red_scratch((size_t)nb + 8);
  if (K <= 32) {
    KSEL(K, (k_update_norm<16><<<nb, RB, 0, stream()>>>(V, ldv, K, c_dev, w, n, part)),
         (k_update_norm<32><<<nb, RB, 0, stream()>>>(V, ldv, K, c_dev, w, n, part)));
    check_launch("update_norm");
    reduce_finish(part, nb, 1, out_dev);
    return;
  }
  DBuf<double> t((size_t)n);
  combine(V, ldv, K, c_dev, t.p, n);
  vaxpy(w, -1.0, t.p, n);
  k_dot<<<nb, RB, 0, stream()>>>(w, w, n, part);
  check_launch("dot");
  reduce_finish(part, nb, 1, out_dev);
}

void combine(const double *V, int64_t ldv, int K, const double *y_dev, double *u, int64_t n) {
  int nb = grid_for(n, RB, g_ctx->num_sms * 8);
  if (K == 0) { vfill(u, 0.0, n); return; }
  for (int k0 = 0; k0 < K; k0 += 32) {
    int kk = K - k0 < 32 ? K - k0 : 32;
    const double *Vk = V + (int64_t)k0 * ldv;
    KSEL(kk, (k_combine<16><<<nb, RB, 0, stream()>>>(Vk, ldv, kk, y_dev + k0, u, n, k0 > 0)),
         (k_combine<32><<<nb, RB, 0, stream()>>>(Vk, ldv, kk, y_dev + k0, u, n, k0 > 0)));
    check_launch("combine");
  }
}

}  // namespace mg
