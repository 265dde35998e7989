// ILU(k) preconditioner (the comparator of SURVEY.md §8(f) item 4): replaces
// ncpflow/ilu.py:53-174 (ilu_factor / ilu_apply).
//
// * Symbolic: level 0 = the pattern of A; level k >= 1 = the structural
//   level-of-fill closure of ilu.py:53-96 (a fill entry (i,j) created through
//   pivot p has level lev(i,p) + lev(p,j) + 1 and survives if <= k), computed
//   row by row on the host (inherently sequential in the row order, setup
//   only).
// * Numeric: IKJ elimination restricted to the pattern (ilu.py:113-149) on the
//   device, one warp per row, rows taken in increasing order from an atomic
//   ticket; row i waits (acquire) for each pivot row p < i, then
//   l_ip = w_p / u_pp and w_c -= l_ip u_pc over row p's upper part (lanes in
//   parallel, each c once per pivot, pivots in ascending order as the
//   reference).  No pivoting; a zero pivot reports the reference's
//   ZeroPivot(row) for the first failing row.
// * Apply: forward substitution with the unit lower factor, backward with the
//   upper factor (sync-free, as trisolve.cu; ilu.py:166-174).
#include <algorithm>
#include <queue>
#include <vector>
#include "ops.cuh"
#include "solver.cuh"

namespace mg {
namespace {

__device__ __forceinline__ int ilu_ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void ilu_st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// lower bound of c in the sorted cols[lo, hi)
__device__ __forceinline__ int find_col(const int *__restrict__ ci, int lo, int hi, int c) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (__ldg(ci + mid) < c) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// ctrl: [0] ticket, [1 + i] row i done.  err: first failing row (atomicMin) and
// the row reported by the reference (pivot row p, or i for its own diagonal)
__global__ void k_ilu_numeric(int n, const int *__restrict__ rp, const int *__restrict__ ci, double *v,
                              const int *__restrict__ dpos, int *ctrl, unsigned long long *err) {
  const int lane = threadIdx.x & 31;
  int *ready = ctrl + 1;
  while (true) {
    int row = 0;
    if (lane == 0) row = atomicAdd(ctrl, 1);
    row = __shfl_sync(0xffffffffu, row, 0);
    if (row >= n) return;
    const int s = rp[row], e = rp[row + 1], d = dpos[row];
    int failed = -1;  // reported row
    // pivots: the lower entries of the row, ascending (sequential dependency)
    for (int q = s; q < (d >= 0 ? d : e) && failed < 0; ++q) {
      const int p = ci[q];
      if (p >= row) break;
      if (lane == 0)
        while (ilu_ld_acquire(ready + p) == 0) {
        }
      __syncwarp();
      const int pd = __ldcg(dpos + p);
      const double piv = pd >= 0 ? __ldcg(v + pd) : 0.0;
      if (piv == 0.0) {
        failed = p;
        break;
      }
      const double lip = __ddiv_rn(v[q], piv);  // own row: written only by this warp
      __syncwarp();
      if (lane == 0) v[q] = lip;
      // w_c -= l_ip u_pc for c in row p's upper part and in this row's pattern
      const int pe = __ldg(rp + p + 1);
      for (int t = pd + 1 + lane; t < pe; t += 32) {
        const int c = __ldg(ci + t);
        const int pos = find_col(ci, q + 1, e, c);
        if (pos < e && __ldg(ci + pos) == c) v[pos] = __dsub_rn(v[pos], __dmul_rn(lip, __ldcg(v + t)));
      }
      __syncwarp();
    }
    if (failed < 0 && (d < 0 || v[d] == 0.0)) failed = row;
    if (lane == 0) {
      if (failed >= 0) atomicMin(err, ((unsigned long long)(unsigned)row << 32) | (unsigned)failed);
      __threadfence();
      ilu_st_release(ready + row, 1);  // published even on failure: no row waits forever
    }
    __syncwarp();
  }
}

__global__ void k_diag_pos(int n, const int *rp, const int *ci, int *dpos) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int lo = rp[i], hi = rp[i + 1];
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (ci[mid] < i) lo = mid + 1; else hi = mid;
  }
  dpos[i] = (lo < rp[i + 1] && ci[lo] == i) ? lo : -1;
}

// combined pattern rows (sorted), values from A at A's positions, zeros at fill
__global__ void k_ilu_scatter(int n, const int *arp, const int *aci, const double *av, const int *rp, const int *ci,
                              double *v) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  const int s = rp[wid], e = rp[wid + 1];
  for (int q = s + lane; q < e; q += 32) v[q] = 0.0;
  __syncwarp();
  for (int q = arp[wid] + lane; q < arp[wid + 1]; q += 32) {
    const int c = aci[q];
    int lo = s, hi = e;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (ci[mid] < c) lo = mid + 1; else hi = mid;
    }
    v[lo] = av[q];
  }
}

// sync-free substitution with the combined factor: lower (unit diagonal,
// entries left of dpos) forward, or upper (entries from dpos) backward
__global__ void k_ilu_trsv(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                           const double *__restrict__ v, const int *__restrict__ dpos, const double *__restrict__ r,
                           double *x, int *ctrl, int upper) {
  const int lane = threadIdx.x & 31;
  int *ready = ctrl + 1;
  while (true) {
    int t = 0;
    if (lane == 0) t = atomicAdd(ctrl, 1);
    t = __shfl_sync(0xffffffffu, t, 0);
    if (t >= n) return;
    const int row = upper ? n - 1 - t : t;
    const int d = dpos[row];
    int s, e;
    if (upper) { s = d + 1; e = rp[row + 1]; }
    else { s = rp[row]; e = d; }
    double acc = r[row];
    // reference order (column-oriented substitution): lower j ascending, upper j descending
    const int cnt = e - s;
    for (int c0 = 0; c0 < cnt; c0 += 32) {
      const int k = c0 + lane;
      double prod = 0.0;
      if (k < cnt) {
        const int q = upper ? e - 1 - k : s + k;
        const int j = ci[q];
        while (ilu_ld_acquire(ready + j) == 0) {
        }
        prod = __dmul_rn(v[q], __ldcg(x + j));
      }
      const int m = min(32, cnt - c0);
      for (int l = 0; l < m; ++l) acc = __dsub_rn(acc, __shfl_sync(0xffffffffu, prod, l));
    }
    if (lane == 0) {
      __stcg(x + row, upper ? __ddiv_rn(acc, v[d]) : acc);
      ilu_st_release(ready + row, 1);
    }
    __syncwarp();
  }
}

int persistent_grid(const void *kern) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, 0);
  return g_ctx->num_sms * (per_sm > 0 ? per_sm : 1);
}

// host: level-of-fill closure (ilu.py:53-96), row by row
void symbolic_fill(int n, const std::vector<int> &rp, const std::vector<int> &ci, int level,
                   std::vector<int> &orp, std::vector<int> &oci) {
  std::vector<std::vector<int>> ucols(n), ulevs(n);
  std::vector<int64_t> lev(n, -1);
  orp.assign(n + 1, 0);
  oci.clear();
  std::vector<int> touched;
  for (int i = 0; i < n; ++i) {
    touched.assign(ci.begin() + rp[i], ci.begin() + rp[i + 1]);
    std::priority_queue<int, std::vector<int>, std::greater<int>> heap;
    std::vector<int> queued;
    for (int q = rp[i]; q < rp[i + 1]; ++q) lev[ci[q]] = 0;
    for (int q = rp[i]; q < rp[i + 1]; ++q)
      if (ci[q] < i) {
        heap.push(ci[q]);
        queued.push_back(ci[q]);
      }
    auto is_queued = [&](int c) { return std::find(queued.begin(), queued.end(), c) != queued.end(); };
    while (!heap.empty()) {
      int p = heap.top();
      heap.pop();
      int64_t lip = lev[p];
      if (lip < 0 || lip > level) continue;
      const std::vector<int> &uc = ucols[p], &ul = ulevs[p];
      for (size_t t = 0; t < uc.size(); ++t) {
        int64_t lf = lip + ul[t] + 1;
        if (lf > level) continue;
        int c = uc[t];
        int64_t cur = lev[c];
        if (cur < 0) {
          lev[c] = lf;
          touched.push_back(c);
          if (c < i && !is_queued(c)) {
            heap.push(c);
            queued.push_back(c);
          }
        } else if (lf < cur) {
          lev[c] = lf;
        }
      }
    }
    std::sort(touched.begin(), touched.end());
    touched.erase(std::unique(touched.begin(), touched.end()), touched.end());
    for (int c : touched)
      if (lev[c] <= level) {
        oci.push_back(c);
        if (c > i) {
          ucols[i].push_back(c);
          ulevs[i].push_back((int)lev[c]);
        }
      }
    orp[i + 1] = (int)oci.size();
    for (int c : touched) lev[c] = -1;
  }
}

}  // namespace

std::unique_ptr<Ilu> ilu_factor(const Csr &a, int level) {
  if (a.b != 1 || a.nr != a.nc) throw MgError(MG_ERR_BAD_OPTION, "ILU expects a square matrix");
  if (level < 0) throw MgError(MG_ERR_BAD_OPTION, "fill level must be nonnegative");
  const int n = a.nr;
  auto f = std::make_unique<Ilu>();
  f->n = n;
  f->level = level;
  Csr &m = f->LU;
  if (level == 0) {
    m.alloc(n, n, a.nnz);
    d2d(m.rp.p, a.rp.p, sizeof(int) * ((size_t)n + 1));
    d2d(m.ci.p, a.ci.p, sizeof(int) * (size_t)a.nnz);
    d2d(m.v.p, a.v.p, sizeof(double) * (size_t)a.nnz);
  } else {
    std::vector<int> hrp(n + 1), hci(a.nnz), orp, oci;
    d2h(hrp.data(), a.rp.p, sizeof(int) * ((size_t)n + 1));
    d2h(hci.data(), a.ci.p, sizeof(int) * (size_t)a.nnz);
    symbolic_fill(n, hrp, hci, level, orp, oci);
    m.alloc(n, n, (int64_t)oci.size());
    h2d(m.rp.p, orp.data(), sizeof(int) * ((size_t)n + 1));
    h2d(m.ci.p, oci.data(), sizeof(int) * oci.size());
    if (n) {
      k_ilu_scatter<<<grid_for((int64_t)n * 32, 256), 256, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, m.rp.p, m.ci.p,
                                                                           m.v.p);
      check_launch("ilu_scatter");
    }
  }
  f->dpos.alloc((size_t)(n ? n : 1));
  f->ctrl.alloc((size_t)n + 1);
  f->t.alloc((size_t)(n ? n : 1));
  if (!n) return f;
  k_diag_pos<<<grid_for(n, 256), 256, 0, stream()>>>(n, m.rp.p, m.ci.p, f->dpos.p);
  check_launch("diag_pos");
  DBuf<unsigned long long> err(1);
  const unsigned long long none = ~0ULL;
  MG_CUDA(cudaMemsetAsync(err.p, 0xff, sizeof(none), stream()));
  dzero(f->ctrl.p, sizeof(int) * ((size_t)n + 1));
  static int grid = 0;
  if (!grid) grid = persistent_grid((const void *)k_ilu_numeric);
  k_ilu_numeric<<<std::min(grid, (n + 7) / 8), 256, 0, stream()>>>(n, m.rp.p, m.ci.p, m.v.p, f->dpos.p,
                                                                   f->ctrl.p, err.p);
  check_launch("ilu_numeric");
  unsigned long long he = none;
  d2h(&he, err.p, sizeof(he));
  if (he != none) {
    int prow = (int)(he & 0xffffffffu);
    throw MgError(MG_ERR_ZERO_PIVOT, "zero pivot encountered at row " + std::to_string(prow), prow);
  }
  return f;
}

void ilu_apply(Ilu &f, const double *r, double *x) {
  const int n = f.n;
  if (!n) return;
  static int grid = 0;
  if (!grid) grid = persistent_grid((const void *)k_ilu_trsv);
  const int g = std::min(grid, (n + 7) / 8);
  dzero(f.ctrl.p, sizeof(int) * ((size_t)n + 1));
  k_ilu_trsv<<<g, 256, 0, stream()>>>(n, f.LU.rp.p, f.LU.ci.p, f.LU.v.p, f.dpos.p, r, f.t.p, f.ctrl.p, 0);
  check_launch("ilu_lower");
  dzero(f.ctrl.p, sizeof(int) * ((size_t)n + 1));
  k_ilu_trsv<<<g, 256, 0, stream()>>>(n, f.LU.rp.p, f.LU.ci.p, f.LU.v.p, f.dpos.p, f.t.p, x, f.ctrl.p, 1);
  check_launch("ilu_upper");
}

}  // namespace mg
