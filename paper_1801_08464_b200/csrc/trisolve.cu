// Gauss-Seidel F-relaxation: forward substitution with the lower triangle
// (diagonal included) of A_ff.
//
// Replaces _GaussSeidelF (ncpflow/mgr.py:175-188): SuperLU on
// tril(A_ff, k=0) with NATURAL ordering, x = L^-1 r, further sweeps
// x += L^-1 (r - A_ff x).  Row i computes
//     s = r_i;  s -= l_ij * x_j  for j < i ascending;  x_i = s / l_ii
// (separate multiply and subtract, the column-oriented substitution order).
//
// Sync-free schedule: warps take rows in increasing order from an atomic
// ticket; each lane spins (acquire) on the ready flag of the dependency it
// holds.  Every row a warp waits on was ticketed earlier to a running warp
// and rows never wait on later rows, so the schedule cannot deadlock; the
// parallelism is the wavefront structure of L (for a 3D 7-point block ~nx+ny+nz
// sequential steps).
#include "ops.cuh"
#include "solver.cuh"
#include "sparse_util.cuh"

namespace mg {

__device__ __forceinline__ int tri_ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void tri_st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// lower-triangular CSR rows (sorted columns, diagonal last)
__global__ void k_trsv_lower(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                             const double *__restrict__ v, const double *__restrict__ r, double *x, int *ctrl) {
  const int lane = threadIdx.x & 31;
  int *ready = ctrl + 1;
  while (true) {
    int row = 0;
    if (lane == 0) row = atomicAdd(ctrl, 1);
    row = __shfl_sync(0xffffffffu, row, 0);
    if (row >= n) return;
    const int s = rp[row], e = rp[row + 1] - 1;  // [s, e): off-diagonal entries, e: diagonal
    double acc = r[row];
    for (int q0 = s; q0 < e; q0 += 32) {
      const int q = q0 + lane;
      double prod = 0.0;
      if (q < e) {
        const int j = ci[q];
        MG_DCHECK(j >= 0 && j < row);  // strictly lower: a later row would never become ready
#ifdef MG_BOUNDS_CHECK
        long long spins = 0;
        while (tri_ld_acquire(ready + j) == 0) MG_DCHECK(++spins < (1LL << 32));
#else
        while (tri_ld_acquire(ready + j) == 0) {
        }
#endif
        prod = __dmul_rn(v[q], __ldcg(x + j));
      }
      const int cnt = min(32, e - q0);
      for (int l = 0; l < cnt; ++l) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, prod, l));
    }
    if (lane == 0) {
      MG_DCHECK(e >= s && ci[e] == row);  // diagonal stored last
      __stcg(x + row, __ddiv_rn(acc, v[e]));
      tri_st_release(ready + row, 1);
    }
    __syncwarp();
  }
}

__global__ void k_tril_count(int n, const int *rp, const int *ci, int *cnt) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  for (int q = rp[i]; q < rp[i + 1]; ++q) c += ci[q] <= i;
  cnt[i] = c;
}
__global__ void k_tril_fill(int n, const int *rp, const int *ci, const double *v, const int *orp, int *oci,
                            double *ov, int *bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int o = orp[i];
  bool diag = false;
  for (int q = rp[i]; q < rp[i + 1]; ++q) {
    if (ci[q] > i) continue;
    if (ci[q] == i) diag = v[q] != 0.0;
    oci[o] = ci[q];
    ov[o] = v[q];
    ++o;
  }
  if (!diag) atomicMin(bad, i);
}

void tril_setup(const Csr &a, Csr &l) {
  if (a.b != 1 || a.nr != a.nc) throw MgError(MG_ERR_UNSUPPORTED, "Gauss-Seidel: square scalar CSR required");
  const int n = a.nr;
  l.nr = l.nc = n;
  l.b = 1;
  l.rp.alloc((size_t)n + 1);
  DBuf<int> cnt((size_t)(n ? n : 1)), bad(1);
  const int big = 0x7fffffff;
  dset_i32(bad.p, {big});
  if (n) {
    k_tril_count<<<grid_for(n, 256), 256, 0, stream()>>>(n, a.rp.p, a.ci.p, cnt.p);
    check_launch("tril_count");
  }
  l.nnz = exclusive_scan_i32_to_i32(cnt.p, l.rp.p, n);
  l.ci.alloc((size_t)l.nnz);
  l.v.alloc((size_t)l.nnz);
  if (n) {
    k_tril_fill<<<grid_for(n, 256), 256, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, l.rp.p, l.ci.p, l.v.p, bad.p);
    check_launch("tril_fill");
  }
  int hb = 0;
  d2h(&hb, bad.p, sizeof(int));
  // the reference's zero-diagonal check (mgr.py:177-179) reports the first row
  if (hb != big) throw MgError(MG_ERR_ZERO_F_DIAG, "zero diagonal in A_ff at fine row " + std::to_string(hb), hb);
}

// x = L^-1 r; ctrl: n + 1 ints of scratch (ticket + ready flags)
void trsv_lower(const Csr &l, const double *r, double *x, int *ctrl) {
  const int n = l.nr;
  if (!n) return;
  dzero(ctrl, sizeof(int) * ((size_t)n + 1));
  static int grid = 0;
  if (!grid) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_trsv_lower, 256, 0);
    grid = g_ctx->num_sms * (per_sm > 0 ? per_sm : 1);
  }
  int g = std::min(grid, (n + 7) / 8);
  k_trsv_lower<<<g < 1 ? 1 : g, 256, 0, stream()>>>(n, l.rp.p, l.ci.p, l.v.p, r, x, ctrl);
  check_launch("trsv_lower");
}

}  // namespace mg
