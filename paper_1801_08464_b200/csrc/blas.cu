// Vector kernels and the fused CGS2 Arnoldi kernels for GMRES
// (krylov.py:101-109: c = V w; w -= c V; c' = V w; w -= c' V; h = ||w||).
//
// Reductions are two-stage with a fixed block count and fixed order, so every
// result is bitwise reproducible run to run.  An Arnoldi step makes four
// streaming passes over its j+1 basis vectors: mdot (c = V w), update
// (w -= c V), mdot (c' = V w), update_norm2 (w -= c' V fused with ||w||^2).
// The register-light mdot (4 accumulators, w shared through L1) measured
// faster than a 3-pass variant that kept all j+1 vectors in registers or
// shared memory (202 registers / 12% occupancy, resp. 37% occupancy).
#include "ops.cuh"

namespace mg {

static const int RB = 256;           // threads per reduction block
static int red_blocks(int64_t n) {
  int64_t b = (n + RB * 4 - 1) / (RB * 4);
  int cap = g_ctx->num_sms * 8;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

__global__ void k_fill(double *x, double val, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = val;
}
__global__ void k_mul(double *y, const double *a, const double *x, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = a[i] * x[i];
}
__global__ void k_axpy(double *y, double a, const double *x, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = y[i] + a * x[i];
}
__global__ void k_add(double *y, const double *x, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = y[i] + x[i];
}
__global__ void k_divs(double *y, const double *x, double d, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}
__global__ void k_sub(double *r, const double *b, const double *ax, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    r[i] = b[i] - ax[i];
}
__global__ void k_gather(double *d, const double *s, const int *idx, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[i] = s[idx[i]];
}
// dst = src[idx]; bs = sign .* dst (when sign); xo = d .* (bs or dst): the gather of
// the F-residual fused with the first pre-sweep from zero of the F-relaxation AMG
__global__ void k_gather_scale(double *dst, const double *src, const int *idx, int64_t n, const double *sign,
                               double *bs, const double *dv, double *xo) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    double v = src[idx[i]];
    dst[i] = v;
    if (sign) {
      v = sign[i] * v;
      bs[i] = v;
    }
    xo[i] = dv[i] * v;
  }
}
__global__ void k_scatter_add(double *d, const double *s, const int *idx, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[idx[i]] = d[idx[i]] + s[i];
}
__global__ void k_scatter_set(double *d, const double *s, const int *idx, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    d[idx[i]] = s[i];
}

__global__ void k_fc_merge(double *e, const double *ef, const int *fmap, int64_t n) {
  PDL_ENTRY();
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int f = fmap[i];
    e[i] = f >= 0 ? ef[f] : 0.0;
  }
}

static int ew_grid(int64_t n) { return grid_for(n, 256, g_ctx->num_sms * 8); }

void fc_merge(double *e, const double *ef, const int *fmap, int64_t n) {
  if (!n) return;
  launch_pdl(k_fc_merge, ew_grid(n), 256, 0, e, ef, fmap, n);
  check_launch("fc_merge");
}

void vfill(double *x, double val, int64_t n) {
  if (!n) return;
  launch_pdl(k_fill, ew_grid(n), 256, 0, x, val, n);
  check_launch("fill");
}
void vcopy(double *dst, const double *src, int64_t n) { d2d(dst, src, n * sizeof(double)); }
void vmul(double *y, const double *a, const double *x, int64_t n) {
  if (!n) return;
  launch_pdl(k_mul, ew_grid(n), 256, 0, y, a, x, n);
  check_launch("mul");
}
void vaxpy(double *y, double a, const double *x, int64_t n) {
  if (!n) return;
  launch_pdl(k_axpy, ew_grid(n), 256, 0, y, a, x, n);
  check_launch("axpy");
}
void vadd(double *y, const double *x, int64_t n) {
  if (!n) return;
  launch_pdl(k_add, ew_grid(n), 256, 0, y, x, n);
  check_launch("add");
}
void vdiv_scalar(double *y, const double *x, double d, int64_t n) {
  if (!n) return;
  launch_pdl(k_divs, ew_grid(n), 256, 0, y, x, d, n);
  check_launch("div");
}
void vsub(double *r, const double *b, const double *ax, int64_t n) {
  if (!n) return;
  launch_pdl(k_sub, ew_grid(n), 256, 0, r, b, ax, n);
  check_launch("sub");
}
void gather(double *dst, const double *src, const int *idx, int64_t n) {
  if (!n) return;
  launch_pdl(k_gather, ew_grid(n), 256, 0, dst, src, idx, n);
  check_launch("gather");
}
void gather_scale(double *dst, const double *src, const int *idx, int64_t n, const double *sign, double *bs,
                  const double *d, double *xo) {
  if (!n) return;
  launch_pdl(k_gather_scale, ew_grid(n), 256, 0, dst, src, idx, n, sign, bs, d, xo);
  check_launch("gather_scale");
}
void scatter_add(double *dst, const double *src, const int *idx, int64_t n) {
  if (!n) return;
  launch_pdl(k_scatter_add, ew_grid(n), 256, 0, dst, src, idx, n);
  check_launch("scatter_add");
}
void scatter_set(double *dst, const double *src, const int *idx, int64_t n) {
  if (!n) return;
  launch_pdl(k_scatter_set, ew_grid(n), 256, 0, dst, src, idx, n);
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
  PDL_ENTRY();
  int k = blockIdx.x;
  int lane = threadIdx.x;
  double s = 0.0;
  for (int b = lane; b < nb; b += 32) s += partial[(int64_t)b * K + k];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) s += __shfl_down_sync(0xffffffffu, s, off);
  if (lane == 0) out[k] = s;
}

__global__ void __launch_bounds__(RB) k_dot(const double *x, const double *y, int64_t n, double *partial) {
  PDL_ENTRY();
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB)
    acc[0] += x[i] * y[i];
  block_reduce_store<1>(acc, 1, partial);
}

static double reduce_finish(double *partial, int nb, int K, double *out_dev) {
  launch_pdl(k_finish, K, 32, 0, partial, nb, K, out_dev);
  check_launch("finish");
  return 0.0;
}

double dot(const double *x, const double *y, int64_t n) {
  int nb = red_blocks(n);
  double *part = red_scratch((size_t)nb + 8);
  double *out = part + nb;
  launch_pdl(k_dot, nb, RB, 0, x, y, n, part);
  check_launch("dot");
  reduce_finish(part, nb, 1, out);
  double h = 0.0;
  d2h(&h, out, sizeof(double));
  return h;
}

double nrm2(const double *x, int64_t n) { return sqrt(dot(x, x, n)); }

// c_k = V_k . w for k < K <= 32: warp q of the block owns vectors q, q+8,
// q+16, q+24 over the block's chunk of CH elements; w is re-read from L1 by
// the 8 warps, V streams once; 4 accumulators per thread, full occupancy.
static const int MCH = 2048;
__global__ void __launch_bounds__(256) k_mdot2(const double *__restrict__ V, int64_t ldv, int K,
                                              const double *__restrict__ w, int64_t n, double *partial) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t c0 = (int64_t)blockIdx.x * MCH; c0 < n; c0 += (int64_t)gridDim.x * MCH) {
    int64_t cend = c0 + MCH < n ? c0 + MCH : n;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int k = wid + 8 * q;
      if (k >= K) break;
      const double *vk = V + k * ldv;
      double a = 0.0;
      int64_t i = c0 + lane;
      for (; i + 96 < cend; i += 128) {
        double v0 = __ldcs(vk + i), v1 = __ldcs(vk + i + 32), v2 = __ldcs(vk + i + 64), v3 = __ldcs(vk + i + 96);
        double w0 = __ldg(w + i), w1 = __ldg(w + i + 32), w2 = __ldg(w + i + 64), w3 = __ldg(w + i + 96);
        a += v0 * w0 + v1 * w1 + v2 * w2 + v3 * w3;
      }
      for (; i < cend; i += 32) a += __ldcs(vk + i) * __ldg(w + i);
      acc[q] += a;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double a = acc[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) a += __shfl_down_sync(0xffffffffu, a, off);
    int k = wid + 8 * q;
    if (lane == 0 && k < K) partial[(int64_t)blockIdx.x * K + k] = a;
  }
}

// w -= sum_k c_k V_k (streaming, two elements per thread)
__global__ void __launch_bounds__(RB) k_update(const double *__restrict__ V, int64_t ldv, int K,
                                              const double *__restrict__ c, double *w, int64_t n) {
  PDL_ENTRY();
  __shared__ double cc[32];
  if (threadIdx.x < 32) cc[threadIdx.x] = (int)threadIdx.x < K ? c[threadIdx.x] : 0.0;
  __syncthreads();
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double t = 0.0;
    for (int k0 = 0; k0 < K; k0 += 8) {
      double vk[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) vk[u] = k0 + u < K ? __ldcs(V + (k0 + u) * ldv + i) : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) t += cc[(k0 + u) & 31] * vk[u];
    }
    w[i] = w[i] - t;
  }
}

// w -= sum c_k V_k ; partial ||w||^2  (c staged in shared memory, low registers)
__global__ void __launch_bounds__(RB) k_update_norm(const double *__restrict__ V, int64_t ldv, int K,
                                                   const double *__restrict__ c, double *w, int64_t n,
                                                   double *partial) {
  PDL_ENTRY();
  __shared__ double cc[32];
  if (threadIdx.x < 32) cc[threadIdx.x] = (int)threadIdx.x < K ? c[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[1] = {0.0};
  // two consecutive elements per thread (16-byte loads) when ldv and n are even
  if ((ldv & 1) == 0) {
    const int64_t n2 = n >> 1;
    const double2 *V2 = reinterpret_cast<const double2 *>(V);
    double2 *w2 = reinterpret_cast<double2 *>(w);
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n2; i += (int64_t)gridDim.x * RB) {
      double tx = 0.0, ty = 0.0;
      for (int k0 = 0; k0 < K; k0 += 8) {
        double2 vk[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          vk[u] = k0 + u < K ? __ldcs(V2 + (k0 + u) * (ldv >> 1) + i) : make_double2(0.0, 0.0);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          tx += cc[k0 + u < 32 ? k0 + u : 31] * vk[u].x;
          ty += cc[k0 + u < 32 ? k0 + u : 31] * vk[u].y;
        }
      }
      double2 wv = w2[i];
      wv.x -= tx;
      wv.y -= ty;
      w2[i] = wv;
      acc[0] += wv.x * wv.x + wv.y * wv.y;
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
      int64_t i = n - 1;
      double t = 0.0;
      for (int k = 0; k < K; ++k) t += cc[k] * V[k * ldv + i];
      double wi = w[i] - t;
      w[i] = wi;
      acc[0] += wi * wi;
    }
  } else {
    for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
      double t = 0.0;
#pragma unroll 8
      for (int k = 0; k < K; ++k) t += cc[k] * V[k * ldv + i];
      double wi = w[i] - t;
      w[i] = wi;
      acc[0] += wi * wi;
    }
  }
  block_reduce_store<1>(acc, 1, partial);
}

// u = sum y_k V_k (or u += when accumulate)
template <int KM>
__global__ void __launch_bounds__(RB) k_combine(const double *__restrict__ V, int64_t ldv, int K,
                                               const double *__restrict__ y, double *u, int64_t n,
                                               int accumulate) {
  PDL_ENTRY();
  double cc[KM];
#pragma unroll
  for (int k = 0; k < KM; ++k) cc[k] = k < K ? y[k] : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double t = accumulate ? u[i] : 0.0;
    // eight basis loads issued before their products (the compiler otherwise
    // interleaves each load with the dependent add chain: one load in flight)
#pragma unroll
    for (int k0 = 0; k0 < KM; k0 += 8) {
      double v[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) v[q] = k0 + q < K ? __ldcs(V + (int64_t)(k0 + q) * ldv + i) : 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (k0 + q < K) t += cc[k0 + q] * v[q];
    }
    u[i] = t;
  }
}

// ---- one-reduction CGS2 with delayed reorthogonalisation (DCGS2) -------------------
// Dot pass: out = [V^T u, V^T w] for the K = j+1 stored vectors (V[j] = u, the
// provisional new basis vector) against u and the new Krylov vector w, reading
// V once: each warp owns vectors k, k + nw, ... over a chunk of MCH elements
// (u and w shared through L1); blocks of nw = min(K, 8) warps keep every warp
// busy for small K.
__global__ void __launch_bounds__(256) k_mdot2x(const double *__restrict__ V, int64_t ldv, int K,
                                               const double *__restrict__ u, const double *__restrict__ w,
                                               int64_t n, double *partial) {
  PDL_ENTRY();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  double au[4] = {0.0, 0.0, 0.0, 0.0}, aw[4] = {0.0, 0.0, 0.0, 0.0};
  for (int64_t c0 = (int64_t)blockIdx.x * MCH; c0 < n; c0 += (int64_t)gridDim.x * MCH) {
    int64_t cend = c0 + MCH < n ? c0 + MCH : n;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      int k = wid + nw * q;
      if (k >= K) break;
      const double *vk = V + k * ldv;
      double a = 0.0, b = 0.0;
      int64_t i = c0 + lane;
      for (; i + 32 < cend; i += 64) {
        double v0 = __ldcs(vk + i), v1 = __ldcs(vk + i + 32);
        double u0 = __ldg(u + i), u1 = __ldg(u + i + 32);
        double w0 = __ldg(w + i), w1 = __ldg(w + i + 32);
        a += v0 * u0 + v1 * u1;
        b += v0 * w0 + v1 * w1;
      }
      for (; i < cend; i += 32) {
        double v0 = __ldcs(vk + i);
        a += v0 * __ldg(u + i);
        b += v0 * __ldg(w + i);
      }
      au[q] += a;
      aw[q] += b;
    }
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    double a = au[q], b = aw[q];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_down_sync(0xffffffffu, a, off);
      b += __shfl_down_sync(0xffffffffu, b, off);
    }
    int k = wid + nw * q;
    if (lane == 0 && k < K) {
      partial[(int64_t)blockIdx.x * 2 * K + k] = a;
      partial[(int64_t)blockIdx.x * 2 * K + K + k] = b;
    }
  }
}

// Update pass, one read of the j finalised vectors Q = V[0..j):
//   q_j     = (sigma u - Q s) / alpha             -> V[j]   (u read from V[j])
//   u_{j+1} = (sigma w - Q e - gamma sigma u) / alpha -> V[j+1]; partial ||u_{j+1}||^2
// coef = [s (j), e (j), sigma, 1/alpha, gamma]
__global__ void __launch_bounds__(RB) k_dcgs2_update(double *V, int64_t ldv, int j,
                                                    const double *__restrict__ coef,
                                                    const double *__restrict__ w, int64_t n,
                                                    double *partial) {
  PDL_ENTRY();
  __shared__ double cs[32], ce[32], sc[3];
  if (threadIdx.x < 32) {
    cs[threadIdx.x] = (int)threadIdx.x < j ? coef[threadIdx.x] : 0.0;
    ce[threadIdx.x] = (int)threadIdx.x < j ? coef[j + threadIdx.x] : 0.0;
  }
  if (threadIdx.x < 3) sc[threadIdx.x] = coef[2 * j + threadIdx.x];
  __syncthreads();
  const double sigma = sc[0], inva = sc[1], gamma = sc[2];
  double *uj = V + (int64_t)j * ldv, *un = V + (int64_t)(j + 1) * ldv;
  double acc[1] = {0.0};
  for (int64_t i = blockIdx.x * (int64_t)RB + threadIdx.x; i < n; i += (int64_t)gridDim.x * RB) {
    double a = 0.0, b = 0.0;
    for (int k0 = 0; k0 < j; k0 += 8) {
      double vk[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) vk[t] = k0 + t < j ? __ldcs(V + (k0 + t) * ldv + i) : 0.0;
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        a += cs[(k0 + t) & 31] * vk[t];
        b += ce[(k0 + t) & 31] * vk[t];
      }
    }
    const double u = sigma * uj[i];
    const double nu = (sigma * __ldg(w + i) - b - gamma * u) * inva;
    uj[i] = (u - a) * inva;
    un[i] = nu;
    acc[0] += nu * nu;
  }
  block_reduce_store<1>(acc, 1, partial);
}

// Thread per element, KT basis vectors per tile: u_i and w_i are loaded once per
// tile and each thread keeps KT independent basis loads in flight (the warp-per-
// vector kernel above re-reads u, w from L1 per vector and keeps two loads in
// flight).  2 KT accumulators per thread, block-reduced once at the end.
template <int KT>
__global__ void __launch_bounds__(256) k_mdot2x_t(const double *__restrict__ V, int64_t ldv, int K,
                                                  const double *__restrict__ u, const double *__restrict__ w,
                                                  int64_t n, double *partial) {
  PDL_ENTRY();
  __shared__ double sm[8][2 * KT];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int k0 = 0; k0 < K; k0 += KT) {
    double au[KT], aw[KT];
#pragma unroll
    for (int t = 0; t < KT; ++t) au[t] = aw[t] = 0.0;
    const int kt = K - k0 < KT ? K - k0 : KT;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
      const double ui = __ldg(u + i), wi = __ldg(w + i);
      double v[KT];
#pragma unroll
      for (int t = 0; t < KT; ++t) v[t] = t < kt ? __ldcs(V + (int64_t)(k0 + t) * ldv + i) : 0.0;
#pragma unroll
      for (int t = 0; t < KT; ++t) {
        au[t] += v[t] * ui;
        aw[t] += v[t] * wi;
      }
    }
#pragma unroll
    for (int t = 0; t < KT; ++t) {
      double a = au[t], b = aw[t];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
      }
      if (lane == 0) {
        sm[wid][t] = a;
        sm[wid][KT + t] = b;
      }
    }
    __syncthreads();
    if ((int)threadIdx.x < 2 * KT) {
      const int t = threadIdx.x % KT;
      if (t < kt) {
        double s = 0.0;
        for (int q = 0; q < 8; ++q) s += sm[q][threadIdx.x];
        const int k = k0 + t + (threadIdx.x >= KT ? K : 0);
        partial[(int64_t)blockIdx.x * 2 * K + k] = s;
      }
    }
    __syncthreads();
  }
}

static bool mdot2x_tiled() {  // MG_MDOT2X_TILED=0: warp-per-vector kernel (A/B)
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_MDOT2X_TILED");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

void mdot2x(const double *V, int64_t ldv, int K, const double *u, const double *w, int64_t n, double *out_dev) {
  if (K > 32) throw MgError(MG_ERR_UNSUPPORTED, "mdot2x: at most 32 vectors");
  if (mdot2x_tiled()) {
    int64_t want = (n + 255) / 256;
    int cap = g_ctx->num_sms * (K <= 8 ? 3 : 2);  // resident blocks (80 / 128 registers)
    int nb = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
    double *part = red_scratch((size_t)nb * 64);
    if (K <= 8) launch_pdl(k_mdot2x_t<8>, nb, 256, 0, V, ldv, K, u, w, n, part);
    else launch_pdl(k_mdot2x_t<16>, nb, 256, 0, V, ldv, K, u, w, n, part);
    check_launch("mdot2x");
    reduce_finish(part, nb, 2 * K, out_dev);
    return;
  }
  const int nw = K < 8 ? K : 8;
  int64_t want = (n + MCH - 1) / MCH;
  int64_t cap = (int64_t)g_ctx->num_sms * 8 * (8 / nw);
  int nb = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  double *part = red_scratch((size_t)nb * 64);
  launch_pdl(k_mdot2x, nb, 32 * nw, 0, V, ldv, K, u, w, n, part);
  check_launch("mdot2x");
  reduce_finish(part, nb, 2 * K, out_dev);
}

void dcgs2_update(double *V, int64_t ldv, int j, const double *coef_dev, const double *w, int64_t n,
                  double *norm2_dev) {
  if (j > 32) throw MgError(MG_ERR_UNSUPPORTED, "dcgs2_update: at most 32 vectors");
  int nb = red_blocks(n);
  double *part = red_scratch((size_t)nb + 8);
  launch_pdl(k_dcgs2_update, nb, RB, 0, V, ldv, j, coef_dev, w, n, part);
  check_launch("dcgs2_update");
  reduce_finish(part, nb, 1, norm2_dev);
}

#define KSEL(K, CALL16, CALL32) \
  do { if ((K) <= 16) { CALL16; } else { CALL32; } } while (0)

void mdot(const double *V, int64_t ldv, int K, const double *w, int64_t n, double *out_dev) {
  int64_t want = (n + MCH - 1) / MCH;
  int nb = (int)(want < g_ctx->num_sms * 8 ? (want < 1 ? 1 : want) : g_ctx->num_sms * 8);
  for (int k0 = 0; k0 < K; k0 += 32) {
    int kk = K - k0 < 32 ? K - k0 : 32;
    double *part = red_scratch((size_t)nb * 32);
    const double *Vk = V + (int64_t)k0 * ldv;
    launch_pdl(k_mdot2, nb, 256, 0, Vk, ldv, kk, w, n, part);
    check_launch("mdot");
    reduce_finish(part, nb, kk, out_dev + k0);
  }
}

void update_mdot(const double *V, int64_t ldv, int K, const double *c_dev, double *w, int64_t n,
                 double *out_dev) {
  if (K <= 32) {
    // w -= cV (one streaming pass), then the projections of the updated w
    launch_pdl(k_update, grid_for(n, RB, g_ctx->num_sms * 8), RB, 0, V, ldv, K, c_dev, w, n);
    check_launch("update");
    mdot(V, ldv, K, w, n, out_dev);
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
    launch_pdl(k_update_norm, nb, RB, 0, V, ldv, K, c_dev, w, n, part);
    check_launch("update_norm");
    reduce_finish(part, nb, 1, out_dev);
    return;
  }
  DBuf<double> t((size_t)n);
  combine(V, ldv, K, c_dev, t.p, n);
  vaxpy(w, -1.0, t.p, n);
  launch_pdl(k_dot, nb, RB, 0, w, w, n, part);
  check_launch("dot");
  reduce_finish(part, nb, 1, out_dev);
}

void combine(const double *V, int64_t ldv, int K, const double *y_dev, double *u, int64_t n) {
  int nb = grid_for(n, RB, g_ctx->num_sms * 8);
  if (K == 0) { vfill(u, 0.0, n); return; }
  for (int k0 = 0; k0 < K; k0 += 32) {
    int kk = K - k0 < 32 ? K - k0 : 32;
    const double *Vk = V + (int64_t)k0 * ldv;
    KSEL(kk, (launch_pdl(k_combine<16>, nb, RB, 0, Vk, ldv, kk, y_dev + k0, u, n, k0 > 0)),
         (launch_pdl(k_combine<32>, nb, RB, 0, Vk, ldv, kk, y_dev + k0, u, n, k0 > 0)));
    check_launch("combine");
  }
}

}  // namespace mg
