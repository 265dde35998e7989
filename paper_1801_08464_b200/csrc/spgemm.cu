// Sparse-sparse kernels: SpGEMM with scipy csr_matmat semantics, transpose,
// submatrix extraction.
//
// SpGEMM (replaces scipy csr_matmat at triple_product, sparse.py:199-203 —
// MGR RAP mgr.py:288 and AMG Galerkin amg.py:318).
// Gustavson row by row, one warp per output row, two passes:
//   count: distinct columns per row (hash of keys only, table >= 2x the
//          row's product count), sizes the output;
//   fill:  table sized by the exact distinct count (>= 2x), accumulators per
//          hash slot, then the keys are sorted and written with their sums.
// Products are generated in windows of 32: a warp scan of |B_j| over 32
// entries of A's row and a per-lane binary search map window lane -> (j, k),
// so every lane issues its global loads at once.  Bit-exact with scipy
// (SURVEY.md §8(c) p2): each output column is accumulated as
// 0 + a_ij1*b_j1k + a_ij2*b_j2k + ... in (j, k) stored order with a separate
// multiply and add — within a window, lanes hitting the same column are
// serialised in lane order by __match_any_sync groups — and exact zeros are
// dropped after the product, columns sorted.
#include "ops.cuh"
#include "sparse_util.cuh"
#include "hash.cuh"
#include <cub/cub.cuh>

namespace mg {

// insert and return the slot; *fresh = 1 when this lane created it
__device__ __forceinline__ int hash_insert_slot(int *keys, unsigned mask, int k, int *fresh) {
  unsigned h = hash_k(k, mask);
#ifdef MG_BOUNDS_CHECK
  unsigned probes = 0;
#endif
  while (true) {
#ifdef MG_BOUNDS_CHECK
    MG_DCHECK(probes++ <= mask);
#endif
    int cur = keys[h];
    if (cur == k) { *fresh = 0; return (int)h; }
    if (cur == -1) {
      int old = atomicCAS(&keys[h], -1, k);
      if (old == -1) { *fresh = 1; return (int)h; }
      if (old == k) { *fresh = 0; return (int)h; }
    }
    h = (h + 1) & mask;
  }
}

// Walk the products of A row `row` (j ascending, B_j stored order) in windows
// of 32; calls f(valid, k, prod) with all lanes converged, in product order.
template <bool NEED_VAL, class F>
__device__ __forceinline__ void for_products(int row, int lane, const int *__restrict__ arp,
                                             const int *__restrict__ aci, const double *__restrict__ av,
                                             const int *__restrict__ brp, const int *__restrict__ bci,
                                             const double *__restrict__ bv, F &&f) {
  int s = arp[row], e = arp[row + 1];
  for (int q0 = s; q0 < e; q0 += 32) {
    int q = q0 + lane;
    int rb = 0, len = 0;
    double a = 0.0;
    if (q < e) {
      int j = __ldg(aci + q);
      if (NEED_VAL) a = __ldg(av + q);
      rb = __ldg(brp + j);
      len = __ldg(brp + j + 1) - rb;
    }
    int incl = len;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, off);
      if (lane >= off) incl += y;
    }
    int total = __shfl_sync(0xffffffffu, incl, 31);
    for (int w0 = 0; w0 < total; w0 += 32) {
      int p = w0 + lane;
      // src = first lane with incl > p
      int lo = 0, hi = 31;
#pragma unroll
      for (int it = 0; it < 5; ++it) {
        int mid = (lo + hi) >> 1;
        int v = __shfl_sync(0xffffffffu, incl, mid);
        if (p < v) hi = mid; else lo = mid + 1;
      }
      int src = lo;
      int s_incl = __shfl_sync(0xffffffffu, incl, src);
      int s_len = __shfl_sync(0xffffffffu, len, src);
      int s_rb = __shfl_sync(0xffffffffu, rb, src);
      double s_a = NEED_VAL ? __shfl_sync(0xffffffffu, a, src) : 0.0;
      bool valid = p < total;
      int k = -1;
      double prod = 0.0;
      if (valid) {
        int r = s_rb + (p - (s_incl - s_len));
        k = __ldg(bci + r);
        if (NEED_VAL) prod = __dmul_rn(s_a, __ldg(bv + r));
      }
      f(valid, k, prod);
    }
  }
}

// The same products, in the same order, but windows never span two A entries: the
// products of one window come from one row of B, whose columns are distinct, so no
// two lanes of a window share an output column (no conflict groups to serialise).
// For long B rows (the Galerkin R*(AP)); lanes idle in a row's last window.
template <bool NEED_VAL, class F>
__device__ __forceinline__ void for_products_rows(int row, int lane, const int *__restrict__ arp,
                                                  const int *__restrict__ aci, const double *__restrict__ av,
                                                  const int *__restrict__ brp, const int *__restrict__ bci,
                                                  const double *__restrict__ bv, F &&f) {
  int s = arp[row], e = arp[row + 1];
  for (int q0 = s; q0 < e; q0 += 32) {
    int q = q0 + lane;
    int rb = 0, len = 0;
    double a = 0.0;
    if (q < e) {
      int j = __ldg(aci + q);
      if (NEED_VAL) a = __ldg(av + q);
      rb = __ldg(brp + j);
      len = __ldg(brp + j + 1) - rb;
    }
    const int nq = min(32, e - q0);
    for (int src = 0; src < nq; ++src) {
      const int s_rb = __shfl_sync(0xffffffffu, rb, src);
      const int s_len = __shfl_sync(0xffffffffu, len, src);
      const double s_a = NEED_VAL ? __shfl_sync(0xffffffffu, a, src) : 0.0;
      for (int w0 = 0; w0 < s_len; w0 += 32) {
        const int p = w0 + lane;
        const bool valid = p < s_len;
        int k = -1;
        double prod = 0.0;
        if (valid) {
          k = __ldg(bci + s_rb + p);
          if (NEED_VAL) prod = __dmul_rn(s_a, __ldg(bv + s_rb + p));
        }
        f(valid, k, prod);
      }
    }
  }
}

// ---- count pass: keys only ------------------------------------------------------
template <int T, int WPB, bool RW>
__global__ void __launch_bounds__(WPB * 32, 2048 / (WPB * 32)) k_spgemm_count(int nrows, const int *rows, const int *arp,
                                                           const int *aci, const int *brp, const int *bci,
                                                           int *cnt) {
  __shared__ int skeys[WPB][T];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int *keys = skeys[wid];
  const unsigned mask = T - 1;
  for (int r = blockIdx.x * WPB + wid; r < nrows; r += gridDim.x * WPB) {
    int row = rows[r];
    for (int i = lane; i < T; i += 32) keys[i] = -1;
    __syncwarp();
    int mine = 0;
    auto ins = [&](bool valid, int k, double) {
      if (valid) mine += hash_insert(keys, mask, k);
    };
    if (RW) for_products_rows<false>(row, lane, arp, aci, nullptr, brp, bci, nullptr, ins);
    else for_products<false>(row, lane, arp, aci, nullptr, brp, bci, nullptr, ins);
    for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
    if (lane == 0) cnt[row] = mine;
    __syncwarp();
  }
}

// global-memory keys for rows beyond the largest smem bin
template <bool RW>
__global__ void k_spgemm_count_g(int nrows, const int *rows, const int64_t *goff, const int *gsize,
                                 unsigned char *pool, const int *arp, const int *aci, const int *brp,
                                 const int *bci, int *cnt) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= nrows) return;
  int T = gsize[wid];
  int *keys = (int *)(pool + goff[wid]);
  unsigned mask = (unsigned)T - 1;
  int row = rows[wid];
  for (int i = lane; i < T; i += 32) keys[i] = -1;
  __syncwarp();
  int mine = 0;
  auto ins = [&](bool valid, int k, double) {
    if (valid) mine += hash_insert(keys, mask, k);
  };
  if (RW) for_products_rows<false>(row, lane, arp, aci, nullptr, brp, bci, nullptr, ins);
  else for_products<false>(row, lane, arp, aci, nullptr, brp, bci, nullptr, ins);
  for (int off = 16; off > 0; off >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, off);
  if (lane == 0) cnt[row] = mine;
}

// ---- fill pass ------------------------------------------------------------------
struct FillTabs {
  int *keys;     // T
  double *acc;   // T (per slot)
  int *list;     // T/2 (sorted keys)
  double *win;   // 32 window values
};

// register sort of the u <= 32E compacted keys in list, then write (key, acc)
template <int E>
__device__ __forceinline__ int emit_sorted(const FillTabs &t, unsigned mask, int u, int lane, int *oci,
                                           double *ov) {
  int k[E], d[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int m = lane * E + e;
    k[e] = m < u ? t.list[m] : 0x7fffffff;
    d[e] = 0;
  }
  warp_sort_regs<E, false>(k, d, lane);
  int nzc = 0;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int m = lane * E + e;
    if (m < u) {
      double val = t.acc[hash_find(t.keys, mask, k[e])];
      oci[m] = k[e];
      ov[m] = val;
      nzc += val != 0.0;
    }
  }
  return nzc;
}

template <bool SORT, bool RW>
__device__ __forceinline__ void fill_row(int row, int T, FillTabs t, int lane, const int *arp, const int *aci,
                                         const double *av, const int *brp, const int *bci, const double *bv,
                                         const int64_t *base, int *oci, double *ov, int *nz) {
  const unsigned mask = (unsigned)T - 1;
  for (int i = lane; i < T; i += 32) t.keys[i] = -1;
  __syncwarp();
  int u = 0;
  if (RW) {
    // conflict-free windows (one B row each): every lane owns its slot in the window
    for_products_rows<true>(row, lane, arp, aci, av, brp, bci, bv, [&](bool valid, int k, double prod) {
      int fresh = 0;
      if (valid) {
        const int slot = hash_insert_slot(t.keys, mask, k, &fresh);
        t.acc[slot] = __dadd_rn(fresh ? 0.0 : t.acc[slot], prod);
      }
      u += __popc(__ballot_sync(0xffffffffu, fresh));
      __syncwarp();
    });
  } else {
    for_products<true>(row, lane, arp, aci, av, brp, bci, bv, [&](bool valid, int k, double prod) {
      int fresh = 0;
      int slot = valid ? hash_insert_slot(t.keys, mask, k, &fresh) : -1 - lane;
      if (fresh) t.acc[slot] = 0.0;
      t.win[lane] = prod;
      u += __popc(__ballot_sync(0xffffffffu, fresh));
      unsigned grp = __match_any_sync(0xffffffffu, slot);
      __syncwarp();
      if (valid && lane == __ffs(grp) - 1) {
        double sacc = t.acc[slot];
        unsigned m = grp;
        while (m) {
          int l = __ffs(m) - 1;
          sacc = __dadd_rn(sacc, t.win[l]);
          m &= m - 1;
        }
        t.acc[slot] = sacc;
      }
      __syncwarp();
    });
  }
  int64_t o = base[row];
  int nzc = 0;
  if (!SORT) {
    // unsorted output (a Galerkin intermediate A*P: R*(AP) accumulates each of its
    // output columns in R's row order whatever the column order inside AP's rows,
    // so only the final product needs scipy's sorted layout): slot order, values
    // straight from the table, no key list / sort / probe
    int filled = 0;
    for (int i0 = 0; i0 < T; i0 += 32) {
      const int k = t.keys[i0 + lane];
      const unsigned bal = __ballot_sync(0xffffffffu, k != -1);
      if (k != -1) {
        const int q = filled + __popc(bal & ((1u << lane) - 1));
        const double val = t.acc[i0 + lane];
        oci[o + q] = k;
        ov[o + q] = val;
        nzc += val != 0.0;
      }
      filled += __popc(bal);
    }
    MG_DCHECK(filled == u);
  } else {
    // sorted key list
    int filled = 0;
    for (int i0 = 0; i0 < T; i0 += 32) {
      int k = t.keys[i0 + lane];
      unsigned bal = __ballot_sync(0xffffffffu, k != -1);
      if (k != -1) t.list[filled + __popc(bal & ((1u << lane) - 1))] = k;
      filled += __popc(bal);
    }
    __syncwarp();
    MG_DCHECK(filled == u && u <= T / 2);  // list capacity; u = the count pass's size
    if (u <= 32) nzc = emit_sorted<1>(t, mask, u, lane, oci + o, ov + o);
    else if (u <= 64) nzc = emit_sorted<2>(t, mask, u, lane, oci + o, ov + o);
    else if (u <= 128) nzc = emit_sorted<4>(t, mask, u, lane, oci + o, ov + o);
    else if (T >= 512 && u <= 256) nzc = emit_sorted<8>(t, mask, u, lane, oci + o, ov + o);
    else {
      int P = 32;
      while (P < u) P <<= 1;
      MG_DCHECK(P <= T / 2);
      for (int i = u + lane; i < P; i += 32) t.list[i] = 0x7fffffff;
      __syncwarp();
      warp_bitonic(t.list, P, lane);
      for (int q = lane; q < u; q += 32) {
        int k = t.list[q];
        double val = t.acc[hash_find(t.keys, mask, k)];
        oci[o + q] = k;
        ov[o + q] = val;
        nzc += val != 0.0;
      }
    }
  }
  for (int off = 16; off > 0; off >>= 1) nzc += __shfl_xor_sync(0xffffffffu, nzc, off);
  if (lane == 0) nz[row] = nzc;
  __syncwarp();
}

template <int T>
__host__ __device__ constexpr size_t fill_bytes() { return (size_t)T * 4 + (size_t)T * 8 + (size_t)T * 2 + 256; }

template <int T, int WPB, bool SORT, bool RW>
__global__ void __launch_bounds__(WPB * 32, 2048 / (WPB * 32)) k_spgemm_fill(int nrows, const int *rows, const int *arp,
                                                          const int *aci, const double *av, const int *brp,
                                                          const int *bci, const double *bv, const int64_t *base,
                                                          int *oci, double *ov, int *nz) {
  extern __shared__ __align__(16) unsigned char smem[];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char *w = smem + fill_bytes<T>() * wid;
  FillTabs t;
  t.acc = (double *)w;
  t.win = t.acc + T;
  t.keys = (int *)(t.win + 32);
  t.list = t.keys + T;
  for (int r = blockIdx.x * WPB + wid; r < nrows; r += gridDim.x * WPB)
    fill_row<SORT, RW>(rows[r], T, t, lane, arp, aci, av, brp, bci, bv, base, oci, ov, nz);
}

template <bool SORT, bool RW>
__global__ void k_spgemm_fill_g(int nrows, const int *rows, const int64_t *goff, const int *gsize,
                                unsigned char *pool, const int *arp, const int *aci, const double *av,
                                const int *brp, const int *bci, const double *bv, const int64_t *base, int *oci,
                                double *ov, int *nz) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= nrows) return;
  int T = gsize[wid];
  unsigned char *w = pool + goff[wid];
  FillTabs t;
  t.acc = (double *)w;
  t.win = t.acc + T;
  t.keys = (int *)(t.win + 32);
  t.list = t.keys + T;
  fill_row<SORT, RW>(rows[wid], T, t, lane, arp, aci, av, brp, bci, bv, base, oci, ov, nz);
}

// compaction: drop exact zeros, keep order (VS-lane group per row)
template <int VS>
__global__ void k_compact(int m, const int64_t *tmp_rp, const int *tci, const double *tv, const int *rp,
                          int *ci, double *v) {
  for (RowGroup<VS> g; g.row < m; g.next()) {
    const int r = (int)g.row;
    int64_t s = tmp_rp[r], e = tmp_rp[r + 1];
    int o = rp[r];
    for (int64_t q0 = s; q0 < e; q0 += VS) {
      int64_t q = q0 + g.lane;
      double val = q < e ? tv[q] : 0.0;
      bool keep = q < e && val != 0.0;
      unsigned bal = g.ballot(keep);
      if (keep) {
        int p = o + g.rank(bal);
        ci[p] = tci[q];
        v[p] = val;
      }
      o += __popc(bal);
    }
  }
}

// per-row product upper bound
template <int VS>
__global__ void k_row_ub(int m, const int *arp, const int *aci, const int *brp, int *ub) {
  for (RowGroup<VS> g; g.row < m; g.next()) {
    const int r = (int)g.row;
    int64_t s = 0;
    for (int q = arp[r] + g.lane; q < arp[r + 1]; q += VS) {
      int j = aci[q];
      s += brp[j + 1] - brp[j];
    }
    s = g.sum(s);
    if (g.lane == 0) ub[r] = s > 0x3fffffff ? 0x3fffffff : (int)s;
  }
}

__device__ __forceinline__ int bin_of(int v) {
  int b = 0;
  while (b < NBIN && v > (32 << b)) ++b;
  return b;
}

// per-block bin histogram in shared memory, one global atomic per bin per block
__global__ void k_bin_count(int m, const int *ub, int *bin_cnt) {
  __shared__ int h[NBIN + 1];
  if (threadIdx.x <= NBIN) h[threadIdx.x] = 0;
  __syncthreads();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x)
    atomicAdd(&h[bin_of(ub[i])], 1);
  __syncthreads();
  if (threadIdx.x <= NBIN && h[threadIdx.x]) atomicAdd(&bin_cnt[threadIdx.x], h[threadIdx.x]);
}
__global__ void k_bin_fill(int m, const int *ub, int *fillpos, int *rows) {
  __shared__ int h[NBIN + 1], base[NBIN + 1];
  if (threadIdx.x <= NBIN) h[threadIdx.x] = 0;
  __syncthreads();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  int b = -1, r = 0;
  if (i < m) {
    b = bin_of(ub[i]);
    r = atomicAdd(&h[b], 1);
  }
  __syncthreads();
  if (threadIdx.x <= NBIN && h[threadIdx.x]) base[threadIdx.x] = atomicAdd(&fillpos[threadIdx.x], h[threadIdx.x]);
  __syncthreads();
  if (b >= 0) rows[base[b] + r] = i;
}
// global tables: T = pow2 >= 2 ub, bytes from the requested layout
__global__ void k_gmem_tabs(int nr, const int *rows, const int *ub, int *tsz, int *units, int layout) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr) return;
  int u = ub[rows[i]];
  int T = 64;
  while (T < 2 * u) T <<= 1;
  tsz[i] = T;
  size_t bytes = layout == 0 ? table_bytes(T, false) : layout == 1 ? (size_t)T * 4 : (size_t)T * 14 + 256;
  units[i] = (int)((bytes + 15) / 16);  // 16-byte units
}

__global__ void k_scale_i64(int64_t *a, int64_t s, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] *= s;
}
void scale_i64(int64_t *a, int64_t s, int n) {
  k_scale_i64<<<grid_for(n, 256), 256, 0, stream()>>>(a, s, n);
  check_launch("scale_i64");
}

void RowBins::build(const int *ub_dev, int m, int layout) {
  static_assert(NBIN + 1 == 8, "bin offsets are set from 8 kernel parameters");
  DBuf<int> bc(NBIN + 1);
  dzero(bc.p, sizeof(int) * (NBIN + 1));
  if (m) {
    k_bin_count<<<grid_for(m, 256, g_ctx->num_sms * 4), 256, 0, stream()>>>(m, ub_dev, bc.p);
    check_launch("bin_count");
  }
  d2h(cnt, bc.p, sizeof(int) * (NBIN + 1));
  off[0] = 0;
  for (int b = 1; b <= NBIN; ++b) off[b] = off[b - 1] + cnt[b - 1];
  dset_i32(bc.p, {off[0], off[1], off[2], off[3], off[4], off[5], off[6], off[7]});
  rows.alloc((size_t)(m ? m : 1));
  if (m) {
    k_bin_fill<<<grid_for(m, 256), 256, 0, stream()>>>(m, ub_dev, bc.p, rows.p);
    check_launch("bin_fill");
  }
  int ng = cnt[NBIN];
  if (ng) {
    gsize.alloc(ng);
    DBuf<int> units(ng);
    goff.alloc((size_t)ng + 1);
    k_gmem_tabs<<<grid_for(ng, 256), 256, 0, stream()>>>(ng, rows.p + off[NBIN], ub_dev, gsize.p, units.p, layout);
    check_launch("gmem_tabs");
    int64_t tot = exclusive_scan_i32_to_i64(units.p, goff.p, ng);
    pool.alloc((size_t)tot * 16);
    scale_i64(goff.p, 16, ng + 1);
  }
}

static int cap_grid(int nrows, int wpb) {
  int grid = (nrows + wpb - 1) / wpb;
  int cap = g_ctx->num_sms * 32;
  return grid > cap ? cap : grid;
}

template <int T, int WPB>
static void launch_count(int nrows, const int *rows, const Csr &a, const Csr &b, int *cnt, bool rw) {
  if (!nrows) return;
  auto kern = rw ? k_spgemm_count<T, WPB, true> : k_spgemm_count<T, WPB, false>;
  kern<<<cap_grid(nrows, WPB), WPB * 32, 0, stream()>>>(nrows, rows, a.rp.p, a.ci.p, b.rp.p, b.ci.p, cnt);
  check_launch("spgemm_count");
}

template <int T, int WPB, bool SORT, bool RW>
static void launch_fill_t(int nrows, const int *rows, const Csr &a, const Csr &b, const int64_t *base, int *oci,
                          double *ov, int *nz) {
  size_t sm = fill_bytes<T>() * WPB;
  MG_CUDA(cudaFuncSetAttribute(k_spgemm_fill<T, WPB, SORT, RW>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)sm));
  k_spgemm_fill<T, WPB, SORT, RW><<<cap_grid(nrows, WPB), WPB * 32, sm, stream()>>>(
      nrows, rows, a.rp.p, a.ci.p, a.v.p, b.rp.p, b.ci.p, b.v.p, base, oci, ov, nz);
  check_launch("spgemm_fill");
}
template <int T, int WPB>
static void launch_fill(int nrows, const int *rows, const Csr &a, const Csr &b, const int64_t *base, int *oci,
                        double *ov, int *nz, bool sorted, bool rw) {
  if (!nrows) return;
  if (sorted && rw) launch_fill_t<T, WPB, true, true>(nrows, rows, a, b, base, oci, ov, nz);
  else if (sorted) launch_fill_t<T, WPB, true, false>(nrows, rows, a, b, base, oci, ov, nz);
  else if (rw) launch_fill_t<T, WPB, false, true>(nrows, rows, a, b, base, oci, ov, nz);
  else launch_fill_t<T, WPB, false, false>(nrows, rows, a, b, base, oci, ov, nz);
}

static bool fill_sparse_tables() {  // MG_SPGEMM_SPARSE=0: load factor 1/2 in every bin (A/B)
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_SPGEMM_SPARSE");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

// MG_SPGEMM_ROWWISE=0 disables the one-B-row windows (A/B)
static bool rowwise_enabled() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_SPGEMM_ROWWISE");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

Csr spgemm(const Csr &a, const Csr &b, bool sorted, bool b_unique) {
  if (a.b != 1 || b.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "spgemm: scalar CSR only");
  if (a.nc != b.nr) throw MgError(MG_ERR_DIM_MISMATCH, "matmul: inner dimensions differ");
  int m = a.nr;
  Csr c;
  if (m == 0 || a.nnz == 0 || b.nnz == 0) {
    c.alloc(m, b.nc, 0);
    dzero(c.rp.p, sizeof(int) * ((size_t)m + 1));
    return c;
  }
  // one-B-row windows when B's rows are long enough to fill most of a window and
  // known to hold distinct columns (a product this library formed)
  const bool rw = b_unique && rowwise_enabled() && b.nr && (double)b.nnz / b.nr >= 20.0;
  DBuf<int> ub(m), cnt(m), nz(m);
  MG_ROWGROUP_LAUNCH(k_row_ub, m, a.nnz, m, a.rp.p, a.ci.p, b.rp.p, ub.p);
  check_launch("row_ub");
  {
    // count pass, tables sized by the product count (all keys could be distinct)
    RowBins bins;
    bins.build(ub.p, m, 1);
#define CB(k, T, W) launch_count<T, W>(bins.cnt[k], bins.rows.p + bins.off[k], a, b, cnt.p, rw)
    CB(0, 64, 8);
    CB(1, 128, 8);
    CB(2, 256, 8);
    CB(3, 512, 8);
    CB(4, 1024, 8);
    CB(5, 2048, 4);
    CB(6, 4096, 2);
#undef CB
    int ng = bins.cnt[NBIN];
    if (ng) {
      auto kern = rw ? k_spgemm_count_g<true> : k_spgemm_count_g<false>;
      kern<<<grid_for((int64_t)ng * 32, 128), 128, 0, stream()>>>(
          ng, bins.rows.p + bins.off[NBIN], bins.goff.p, bins.gsize.p, bins.pool.p, a.rp.p, a.ci.p, b.rp.p, b.ci.p,
          cnt.p);
      check_launch("spgemm_count_g");
    }
  }
  DBuf<int64_t> trp((size_t)m + 1);
  int64_t total = exclusive_scan_i32_to_i64(cnt.p, trp.p, m);
  DBuf<int> tci((size_t)total);
  DBuf<double> tv((size_t)total);
  {
    // fill pass, tables sized by the exact distinct count
    RowBins bins;
    bins.build(cnt.p, m, 2);
#define FB(k, T, W) \
  launch_fill<T, W>(bins.cnt[k], bins.rows.p + bins.off[k], a, b, trp.p, tci.p, tv.p, nz.p, sorted, rw)
    if (fill_sparse_tables()) {
      // load factor <= 1/4 for the two small bins (shorter probe runs: fill 9.7 ->
      // 8.8 ms and 11.1 -> 9.5 ms at 128^3); larger tables cost more in occupancy
      // than they save from bin 2 on
      FB(0, 128, 8);
      FB(1, 256, 8);
      FB(2, 256, 8);
    } else {
      FB(0, 64, 8);
      FB(1, 128, 8);
      FB(2, 256, 8);
    }
    FB(3, 512, 8);
    FB(4, 1024, 8);
    FB(5, 2048, 4);
    FB(6, 4096, 2);
#undef FB
    int ng = bins.cnt[NBIN];
    if (ng) {
      auto kern = sorted ? (rw ? k_spgemm_fill_g<true, true> : k_spgemm_fill_g<true, false>)
                         : (rw ? k_spgemm_fill_g<false, true> : k_spgemm_fill_g<false, false>);
      kern<<<grid_for((int64_t)ng * 32, 128), 128, 0, stream()>>>(
          ng, bins.rows.p + bins.off[NBIN], bins.goff.p, bins.gsize.p, bins.pool.p, a.rp.p, a.ci.p, a.v.p, b.rp.p,
          b.ci.p, b.v.p, trp.p, tci.p, tv.p, nz.p);
      check_launch("spgemm_fill_g");
    }
  }
  c.nr = m;
  c.nc = b.nc;
  c.b = 1;
  c.rp.alloc((size_t)m + 1);
  int64_t kept = exclusive_scan_i32_to_i32(nz.p, c.rp.p, m);
  c.nnz = kept;
  if (kept == total) {
    c.ci = std::move(tci);
    c.v = std::move(tv);
  } else {
    c.ci.alloc((size_t)kept);
    c.v.alloc((size_t)kept);
    MG_ROWGROUP_LAUNCH(k_compact, m, total, m, trp.p, tci.p, tv.p, c.rp.p, c.ci.p, c.v.p);
    check_launch("compact");
  }
  return c;
}

// ---- transpose (stable: rows of A^T have ascending columns) -----------------
template <int VS>
__global__ void k_row_ids(int m, const int *rp, int *rid) {
  for (RowGroup<VS> g; g.row < m; g.next()) {
    const int r = (int)g.row;
    for (int q = rp[r] + g.lane; q < rp[r + 1]; q += VS) rid[q] = r;
  }
}
__global__ void k_iota(int *a, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = (int)i;
}
__global__ void k_col_count(int64_t nnz, const int *ci, int *cnt) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&cnt[ci[i]], 1);
}
__global__ void k_permute_entries(int64_t nnz, const int *perm, const int *rid, const double *v, int *tci,
                                  double *tv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    int p = perm[i];
    tci[i] = rid[p];
    tv[i] = v[p];
  }
}

// ---- variable-major scalar CSR -> cell-major block CSR ------------------------
// SURVEY.md §8(b) mat_upload_csr_varmajor: the reference's BlockSystem matrix is
// scalar CSR over unknowns u = var * N + cell (assembly.py:95-120); the block
// kernels want block rows = cells, b x b row-major blocks, sorted block columns.
// Entry (r, c) goes to block (r % N, c % N) at (r / N, c / N); positions no entry
// fills are explicit zeros.  Keys (cell_r * N + cell_c) radix-sorted with the entry
// ids, run heads give the blocks.
__global__ void k_vm_keys(int64_t nnz, int N, const int *rid, const int *ci, int64_t *key, int *idx) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < nnz; q += (int64_t)gridDim.x * blockDim.x) {
    key[q] = (int64_t)(rid[q] % N) * N + (ci[q] % N);
    idx[q] = (int)q;
  }
}
__global__ void k_vm_heads(int64_t nnz, const int64_t *key, int *head) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x)
    head[p] = (p == 0 || key[p] != key[p - 1]) ? 1 : 0;
}
__global__ void k_vm_fill(int64_t nnz, int N, int b, const int64_t *key, const int *head, const int *seg,
                          const int *idx, const int *rid, const int *ci, const double *v, int *bcol, int *bcnt,
                          double *bv) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int blk = seg[p] + head[p] - 1;  // inclusive run index
    const int q = idx[p];
    if (head[p]) {
      bcol[blk] = (int)(key[p] % N);
      atomicAdd(&bcnt[key[p] / N], 1);
    }
    bv[(int64_t)blk * b * b + (rid[q] / N) * b + ci[q] / N] = v[q];
  }
}

Csr csr_varmajor_to_bsr(const Csr &a, int b) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "csr_varmajor_to_bsr: scalar CSR required");
  if (b < 1 || b > 3) throw MgError(MG_ERR_UNSUPPORTED, "block size must be 1, 2 or 3");
  if (a.nr != a.nc || a.nr % b) throw MgError(MG_ERR_DIM_MISMATCH, "variable-major matrix: n must be b * cells");
  const int N = a.nr / b;
  const int64_t nnz = a.nnz;
  Csr c;
  if (nnz == 0) {
    c.alloc(N, N, 0, b);
    dzero(c.rp.p, sizeof(int) * ((size_t)N + 1));
    return c;
  }
  DBuf<int> rid((size_t)nnz), idx((size_t)nnz), idx_s((size_t)nnz), head((size_t)nnz), seg((size_t)nnz + 1);
  DBuf<int64_t> key((size_t)nnz), key_s((size_t)nnz);
  MG_ROWGROUP_LAUNCH(k_row_ids, a.nr, a.nnz, a.nr, a.rp.p, rid.p);
  check_launch("row_ids");
  const int g = grid_for(nnz, 256, g_ctx->num_sms * 8);
  k_vm_keys<<<g, 256, 0, stream()>>>(nnz, N, rid.p, a.ci.p, key.p, idx.p);
  check_launch("vm_keys");
  int bits = 1;
  while (bits < 63 && ((int64_t)1 << bits) < (int64_t)N * N) ++bits;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, key.p, key_s.p, idx.p, idx_s.p, (int)nnz, 0, bits, stream());
  void *tmp = cub_scratch(tb);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, key.p, key_s.p, idx.p, idx_s.p, (int)nnz, 0, bits, stream()));
  count_launch(4);
  k_vm_heads<<<g, 256, 0, stream()>>>(nnz, key_s.p, head.p);
  check_launch("vm_heads");
  const int64_t nblk = exclusive_scan_i32_to_i32(head.p, seg.p, (int)nnz);
  c.alloc(N, N, nblk, b);
  DBuf<int> bcnt((size_t)N + 1);
  dzero(bcnt.p, sizeof(int) * ((size_t)N + 1));
  dzero(c.v.p, sizeof(double) * (size_t)nblk * b * b);
  k_vm_fill<<<g, 256, 0, stream()>>>(nnz, N, b, key_s.p, head.p, seg.p, idx_s.p, rid.p, a.ci.p, a.v.p, c.ci.p,
                                     bcnt.p, c.v.p);
  check_launch("vm_fill");
  exclusive_scan_i32_to_i32(bcnt.p, c.rp.p, N);
  return c;
}

Csr transpose(const Csr &a) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "transpose: scalar CSR only");
  Csr t;
  int64_t nnz = a.nnz;
  t.alloc(a.nc, a.nr, nnz);
  DBuf<int> cnt((size_t)a.nc + 1);
  dzero(cnt.p, sizeof(int) * ((size_t)a.nc + 1));
  if (nnz) {
    k_col_count<<<grid_for(nnz, 256, g_ctx->num_sms * 8), 256, 0, stream()>>>(nnz, a.ci.p, cnt.p);
    check_launch("col_count");
  }
  exclusive_scan_i32_to_i32(cnt.p, t.rp.p, a.nc);
  if (!nnz) return t;
  DBuf<int> rid((size_t)nnz), idx((size_t)nnz), keys_out((size_t)nnz), perm((size_t)nnz);
  MG_ROWGROUP_LAUNCH(k_row_ids, a.nr, a.nnz, a.nr, a.rp.p, rid.p);
  check_launch("row_ids");
  k_iota<<<grid_for(nnz, 256, g_ctx->num_sms * 8), 256, 0, stream()>>>(idx.p, nnz);
  check_launch("iota");
  int bits = 1;
  while ((1LL << bits) < (int64_t)a.nc) ++bits;
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, a.ci.p, keys_out.p, idx.p, perm.p, (int)nnz, 0, bits,
                                  stream());
  void *tmp = cub_scratch(bytes);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, bytes, a.ci.p, keys_out.p, idx.p, perm.p, (int)nnz, 0, bits,
                                          stream()));
  count_launch(4);
  k_permute_entries<<<grid_for(nnz, 256, g_ctx->num_sms * 8), 256, 0, stream()>>>(nnz, perm.p, rid.p,
                                                                                   a.v.p, t.ci.p, t.v.p);
  check_launch("permute_entries");
  return t;
}

// ---- extract A[rows][:, cols] (keeps stored zeros) ---------------------------
template <int VS>
__global__ void k_extract_count(int nr, const int *rows, const int *rp, const int *ci, const int *cmap,
                                int *cnt) {
  for (RowGroup<VS> g; g.row < nr; g.next()) {
    int r = rows[g.row];
    int c = 0;
    for (int q = rp[r] + g.lane; q < rp[r + 1]; q += VS) c += cmap[ci[q]] >= 0;
    c = g.sum(c);
    if (g.lane == 0) cnt[g.row] = c;
  }
}
template <int VS>
__global__ void k_extract_fill(int nr, const int *rows, const int *rp, const int *ci, const double *v,
                               const int *cmap, const int *orp, int *oci, double *ov) {
  for (RowGroup<VS> g; g.row < nr; g.next()) {
    int r = rows[g.row];
    int o = orp[g.row];
    const int e = rp[r + 1];
    for (int q0 = rp[r]; q0 < e; q0 += VS) {
      int q = q0 + g.lane;
      int m = q < e ? cmap[ci[q]] : -1;
      unsigned bal = g.ballot(m >= 0);
      if (m >= 0) {
        int p = o + g.rank(bal);
        oci[p] = m;
        ov[p] = v[q];
      }
      o += __popc(bal);
    }
  }
}

Csr extract(const Csr &a, const int *rows_dev, int nr, const int *cmap_dev, int nc) {
  Csr o;
  o.nr = nr;
  o.nc = nc;
  o.rp.alloc((size_t)nr + 1);
  DBuf<int> cnt((size_t)nr + 1);
  if (nr) {
    MG_ROWGROUP_LAUNCH(k_extract_count, nr, a.nr ? (int64_t)((double)a.nnz * nr / a.nr) : 0, nr, rows_dev, a.rp.p,
                       a.ci.p, cmap_dev, cnt.p);
    check_launch("extract_count");
  }
  o.nnz = exclusive_scan_i32_to_i32(cnt.p, o.rp.p, nr);
  o.ci.alloc((size_t)o.nnz);
  o.v.alloc((size_t)o.nnz);
  if (nr && o.nnz) {
    MG_ROWGROUP_LAUNCH(k_extract_fill, nr, a.nr ? (int64_t)((double)a.nnz * nr / a.nr) : 0, nr, rows_dev, a.rp.p,
                       a.ci.p, a.v.p, cmap_dev, o.rp.p, o.ci.p, o.v.p);
    check_launch("extract_fill");
  }
  return o;
}

void iota_i32(int *p, int64_t n) {
  if (n <= 0) return;
  k_iota<<<grid_for(n, 256, g_ctx->num_sms * 8), 256, 0, stream()>>>(p, n);
  check_launch("iota");
}

Csr copy_csr(const Csr &a) {
  Csr o;
  o.alloc(a.nr, a.nc, a.nnz, a.b);
  d2d(o.rp.p, a.rp.p, sizeof(int) * ((size_t)a.nr + 1));
  d2d(o.ci.p, a.ci.p, sizeof(int) * (size_t)a.nnz);
  d2d(o.v.p, a.v.p, sizeof(double) * (size_t)a.nnz * a.b * a.b);
  return o;
}

}  // namespace mg
