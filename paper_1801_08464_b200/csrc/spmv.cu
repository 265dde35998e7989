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

// VS lanes cooperate on one row; every lane runs the shuffle (no early exit).
template <int VS, class Epi>
__global__ void __launch_bounds__(256) k_csr(int nr, const int *__restrict__ rp,
                                             const int *__restrict__ ci,
                                             const double *__restrict__ v,
                                             const double *__restrict__ x, Epi epi) {
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int row = (int)(tid / VS);
  int lane = (int)(tid % VS);
  double sum = 0.0;
  if (row < nr) {
    int s = __ldg(rp + row), e = __ldg(rp + row + 1);
#pragma unroll 4
    for (int k = s + lane; k < e; k += VS) sum += __ldg(v + k) * __ldg(x + __ldg(ci + k));
  }
#pragma unroll
  for (int off = VS / 2; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off, VS);
  if (row < nr && lane == 0) epi(row, sum);
}

template <int B, int G>
__global__ void __launch_bounds__(256) k_bsr(int nbr, const int *__restrict__ rp,
                                             const int *__restrict__ ci,
                                             const double *__restrict__ v,
                                             const double *__restrict__ x,
                                             double *__restrict__ y) {
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  int row = (int)(tid / G);
  int lane = (int)(tid % G);
  double acc[B];
#pragma unroll
  for (int r = 0; r < B; ++r) acc[r] = 0.0;
  if (row < nbr) {
    int s = __ldg(rp + row), e = __ldg(rp + row + 1);
    for (int k = s + lane; k < e; k += G) {
      int c = __ldg(ci + k);
      if (B == 2) {
        const double2 *vb = reinterpret_cast<const double2 *>(v) + (int64_t)k * 2;
        double2 r0 = __ldg(vb), r1 = __ldg(vb + 1);
        double2 xc = __ldg(reinterpret_cast<const double2 *>(x) + c);
        acc[0] += r0.x * xc.x + r0.y * xc.y;
        acc[1] += r1.x * xc.x + r1.y * xc.y;
      } else {
        const double *vb = v + (int64_t)k * B * B;
        double xc[B];
#pragma unroll
        for (int q = 0; q < B; ++q) xc[q] = __ldg(x + (int64_t)c * B + q);
#pragma unroll
        for (int r = 0; r < B; ++r) {
          double t = 0.0;
#pragma unroll
          for (int q = 0; q < B; ++q) t += __ldg(vb + r * B + q) * xc[q];
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

template <class Epi>
static void launch_csr(const Csr &a, const double *x, Epi epi) {
  if (a.nr == 0) return;
  double avg = a.nr ? (double)a.nnz / a.nr : 0.0;
  const int T = 256;
  cudaStream_t s = stream();
#define LAUNCH(VS)                                                                    \
  k_csr<VS, Epi><<<grid_for((int64_t)a.nr * VS, T), T, 0, s>>>(a.nr, a.rp.p, a.ci.p, \
                                                               a.v.p, x, epi)
  if (avg <= 2.5) LAUNCH(2);
  else if (avg <= 5) LAUNCH(4);
  else if (avg <= 12) LAUNCH(8);
  else if (avg <= 28) LAUNCH(16);
  else LAUNCH(32);
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
  if (a.b == 2) {
    if (avg <= 4.5) k_bsr<2, 4><<<grid_for((int64_t)a.nr * 4, T), T, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
    else k_bsr<2, 8><<<grid_for((int64_t)a.nr * 8, T), T, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
  } else if (a.b == 3) {
    if (avg <= 4.5) k_bsr<3, 4><<<grid_for((int64_t)a.nr * 4, T), T, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
    else k_bsr<3, 8><<<grid_for((int64_t)a.nr * 8, T), T, 0, s>>>(a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
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
