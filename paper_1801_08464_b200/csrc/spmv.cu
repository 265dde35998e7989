// SpMV family: scalar CSR (sub-warp per row, fused epilogues) and block-CSR
// b = 2 / 3 (lane group per block row, vectorised block loads).
//
// Replaces scipy csr_matvec at every hot call site:
// the GMRES operator `a @ v` (linsolve.py:100), MGR residual / R / P products
// (mgr.py:347,355,357) and the AMG residual / restriction / prolongation
// (amg.py:347,361-364).  HBM-bound: algorithmic bytes per launch
// nnz*(8 b^2 + 4) + 4 (nr + 1) + 8 b (nc + nr).
#include "ops.cuh"

namespace mg {

struct EpiStore {
  double *y;
  __device__ void operator()(int r, double s) const { y[r] = s; }
};
struct EpiResid {
  const double *b;
  double *r;
  __device__ void operator()(int i, double s) const { r[i] = b[i] - s; }
};
struct EpiAdd {
  double *y;
  __device__ void operator()(int r, double s) const { y[r] = y[r] + s; }
};
struct EpiJacobi {
  const double *x, *b, *dinv;
  double *xo;
  __device__ void operator()(int i, double s) const { xo[i] = x[i] + dinv[i] * (b[i] - s); }
};

// VS lanes cooperate on one row; each lane keeps U independent (value, column)
// loads in flight before the dependent x gathers, so a warp has VS*U*12 B of
// matrix traffic outstanding per round trip.  Groups stride over rows (grid
// sized to the resident capacity); every lane runs the shuffle (uniform loop).
template <int VS, int U, class Epi>
__global__ void __launch_bounds__(256) k_csr(int nr, const int *__restrict__ rp,
                                             const int *__restrict__ ci,
                                             const double *__restrict__ v,
                                             const double *__restrict__ x, Epi epi) {
  const int lane = threadIdx.x % VS;
  const int g0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / VS);
  const int ng = (int)((int64_t)gridDim.x * blockDim.x / VS);
  const int warp_first = (int)(((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / VS);
  for (int row = g0, wf = warp_first; wf < nr; row += ng, wf += ng) {
    double sum = 0.0;
    if (row < nr) {
      int s = __ldg(rp + row), e = __ldg(rp + row + 1);
      for (int k0 = s; k0 < e; k0 += VS * U) {
        double vv[U];
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int k = k0 + lane + u * VS;
          bool ok = k < e;
          vv[u] = ok ? __ldcs(v + k) : 0.0;
          cc[u] = ok ? __ldcs(ci + k) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (cc[u] >= 0) sum += vv[u] * __ldg(x + cc[u]);
      }
    }
#pragma unroll
    for (int off = VS / 2; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off, VS);
    if (row < nr && lane == 0) epi(row, sum);
  }
}

template <int B, int G, int U>
__global__ void __launch_bounds__(256) k_bsr(int nbr, const int *__restrict__ rp,
                                             const int *__restrict__ ci,
                                             const double *__restrict__ v,
                                             const double *__restrict__ x,
                                             double *__restrict__ y) {
  const int lane = threadIdx.x % G;
  const int g0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / G);
  const int ng = (int)((int64_t)gridDim.x * blockDim.x / G);
  const int warp_first = (int)(((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / G);
  for (int row = g0, wf = warp_first; wf < nbr; row += ng, wf += ng) {
    double acc[B];
#pragma unroll
    for (int r = 0; r < B; ++r) acc[r] = 0.0;
    if (row < nbr) {
      int s = __ldg(rp + row), e = __ldg(rp + row + 1);
      for (int k0 = s; k0 < e; k0 += G * U) {
        double a[U][B * B];
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int k = k0 + lane + u * G;
          cc[u] = k < e ? __ldcs(ci + k) : -1;
          if (B == 2) {
            const double2 *vb = reinterpret_cast<const double2 *>(v) + (int64_t)(k < e ? k : s) * 2;
            double2 r0 = __ldcs(vb), r1 = __ldcs(vb + 1);
            a[u][0] = r0.x; a[u][1] = r0.y; a[u][2] = r1.x; a[u][3] = r1.y;
          } else {
            const double *vb = v + (int64_t)(k < e ? k : s) * B * B;
#pragma unroll
            for (int q = 0; q < B * B; ++q) a[u][q] = __ldcs(vb + q);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (cc[u] < 0) continue;
          double xc[B];
          if (B == 2) {
            double2 t = __ldg(reinterpret_cast<const double2 *>(x) + cc[u]);
            xc[0] = t.x; xc[1] = t.y;
          } else {
#pragma unroll
            for (int q = 0; q < B; ++q) xc[q] = __ldg(x + (int64_t)cc[u] * B + q);
          }
#pragma unroll
          for (int r = 0; r < B; ++r) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < B; ++q) t += a[u][r * B + q] * xc[q];
            acc[r] += t;
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < B; ++r)
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) acc[r] += __shfl_down_sync(0xffffffffu, acc[r], off, G);
    if (row < nbr && lane == 0) {
      if (B == 2) {
        reinterpret_cast<double2 *>(y)[row] = make_double2(acc[0], acc[1]);
      } else {
#pragma unroll
        for (int r = 0; r < B; ++r) y[(int64_t)row * B + r] = acc[r];
      }
    }
  }
}

// resident-capacity grid for the row-striding SpMV kernels
static int spmv_grid(int64_t threads_needed) {
  int64_t want = (threads_needed + 255) / 256;
  int64_t cap = (int64_t)g_ctx->num_sms * 8;
  if (want > cap) want = cap;
  return (int)(want < 1 ? 1 : want);
}

template <class Epi>
static void launch_csr(const Csr &a, const double *x, Epi epi) {
  if (a.nr == 0) return;
  double avg = a.nr ? (double)a.nnz / a.nr : 0.0;
  const int T = 256;
  cudaStream_t s = stream();
  (void)T;
#define LAUNCH(VS, U)                                                               \
  k_csr<VS, U, Epi><<<spmv_grid((int64_t)a.nr * VS), 256, 0, s>>>(a.nr, a.rp.p, a.ci.p, \
                                                                  a.v.p, x, epi)
  if (avg <= 2.5) LAUNCH(2, 2);
  else if (avg <= 5) LAUNCH(4, 2);
  else if (avg <= 9) LAUNCH(4, 3);
  else if (avg <= 18) LAUNCH(8, 3);
  else if (avg <= 36) LAUNCH(16, 3);
  else if (avg <= 72) LAUNCH(16, 5);
  else LAUNCH(32, 4);
#undef LAUNCH
  check_launch("csr spmv");
}

void spmv(const Csr &a, const double *x, double *y) {
  if (a.b == 1) {
    launch_csr(a, x, EpiStore{y});
    return;
  }
  if (a.nr == 0) return;
  const int T = 256;
  double avg = (double)a.nnz / a.nr;
  cudaStream_t s = stream();
  (void)T;
  if (a.b == 2) {
    if (avg <= 4.5) k_bsr<2, 2, 3><<<spmv_grid((int64_t)a.nr * 2), 256, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
    else k_bsr<2, 4, 2><<<spmv_grid((int64_t)a.nr * 4), 256, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
  } else if (a.b == 3) {
    if (avg <= 4.5) k_bsr<3, 2, 3><<<spmv_grid((int64_t)a.nr * 2), 256, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
    else k_bsr<3, 4, 2><<<spmv_grid((int64_t)a.nr * 4), 256, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
  } else {
    throw MgError(MG_ERR_UNSUPPORTED, "block size must be 1, 2 or 3");
  }
  check_launch("bsr spmv");
}

void residual(const Csr &a, const double *x, const double *b, double *r) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "residual: scalar CSR only");
  launch_csr(a, x, EpiResid{b, r});
}

void spmv_add(const Csr &a, const double *x, double *y) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "spmv_add: scalar CSR only");
  launch_csr(a, x, EpiAdd{y});
}

void jacobi_sweep(const Csr &a, const double *x, const double *b, const double *dinv, double *xo) {
  launch_csr(a, x, EpiJacobi{x, b, dinv, xo});
}

}  // namespace mg
