// Warp-level shared-memory hash tables, bitonic sort and row binning used by
// the SpGEMM and the extended+i interpolation kernels.
#pragma once
#include "common.cuh"

namespace mg {

// Fibonacci hashing: the HIGH bits of k * 2^32/phi.  (The low bits of a
// multiplicative hash depend only on the low bits of k, so stencil columns
// spaced by powers of two -- +-nx, +-nx*ny -- would all collide.)
__device__ __forceinline__ unsigned hash_k(int k, unsigned mask) {
  return ((unsigned)k * 2654435769u) >> __clz((int)mask);
}

// insert key; returns 1 if newly inserted (keys[] initialised to -1)
__device__ __forceinline__ int hash_insert(int *keys, unsigned mask, int k) {
  unsigned h = hash_k(k, mask);
#ifdef MG_BOUNDS_CHECK
  unsigned probes = 0;
#endif
  while (true) {
#ifdef MG_BOUNDS_CHECK
    MG_DCHECK(probes++ <= mask);  // table full: the sizing bound was wrong
#endif
    int cur = keys[h];
    if (cur == k) return 0;
    if (cur == -1) {
      int old = atomicCAS(&keys[h], -1, k);
      if (old == -1) return 1;
      if (old == k) return 0;
    }
    h = (h + 1) & mask;
  }
}

__device__ __forceinline__ unsigned hash_find(const int *keys, unsigned mask, int k) {
  unsigned h = hash_k(k, mask);
#ifdef MG_BOUNDS_CHECK
  unsigned probes = 0;
  while (keys[h] != k) {
    MG_DCHECK(keys[h] != -1 && probes++ <= mask);  // key absent
    h = (h + 1) & mask;
  }
#else
  while (keys[h] != k) h = (h + 1) & mask;
#endif
  return h;
}

// slot of k or -1 when absent
__device__ __forceinline__ int hash_find_opt(const int *keys, unsigned mask, int k) {
  unsigned h = hash_k(k, mask);
  while (true) {
    int cur = keys[h];
    if (cur == k) return (int)h;
    if (cur == -1) return -1;
    h = (h + 1) & mask;
  }
}

// warp-wide bitonic sort of L[0..P) ascending (P power of two >= 32)
__device__ __forceinline__ void warp_bitonic(int *L, int P, int lane) {
  for (int k = 2; k <= P; k <<= 1)
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = lane; i < P; i += 32) {
        int ixj = i ^ j;
        if (ixj > i) {
          int a = L[i], b = L[ixj];
          bool up = (i & k) == 0;
          if ((a > b) == up) { L[i] = b; L[ixj] = a; }
        }
      }
      __syncwarp();
    }
}

// Register bitonic sort of a warp's 32*E elements, blocked layout (lane owns
// elements lane*E .. lane*E+E-1), ascending; keys distinct except padding.
template <int E, bool VAL = true>
__device__ __forceinline__ void warp_sort_regs(int (&k)[E], int (&v)[E], int lane) {
#pragma unroll
  for (int size = 2; size <= 32 * E; size <<= 1) {
#pragma unroll
    for (int j = size >> 1; j > 0; j >>= 1) {
      if (j < E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if (e & j) continue;
          int m = lane * E + e;
          bool asc = (m & size) == 0;
          if ((k[e] > k[e ^ j]) == asc) {
            int tk = k[e]; k[e] = k[e ^ j]; k[e ^ j] = tk;
            if (VAL) { int tv = v[e]; v[e] = v[e ^ j]; v[e ^ j] = tv; }
          }
        }
      } else {
        const int lj = j / E;
        bool lower = (lane & lj) == 0;
#pragma unroll
        for (int e = 0; e < E; ++e) {
          int m = lane * E + e;
          bool asc = (m & size) == 0;
          int ok = __shfl_xor_sync(0xffffffffu, k[e], lj);
          int ov = VAL ? __shfl_xor_sync(0xffffffffu, v[e], lj) : 0;
          bool take = (lower == asc) ? (ok < k[e]) : (ok > k[e]);
          if (take) { k[e] = ok; if (VAL) v[e] = ov; }
        }
      }
    }
  }
}

struct WarpTables {
  int *keys;     // T
  int *pos;      // T
  int *list;     // T/2
  double *acc;   // T/2
  int *pcol;     // T/2  staged products / terms (column)
  double *pval;  // T/2  staged products / terms (value)
};

// per-warp table bytes for T slots:
// acc (T/2 f64) | [pval (T/2 f64)] | keys (T) | pos (T) | list (T/2) | [pcol (T/2)]
// the bracketed staging arrays exist only when `staged` (small / medium rows)
__host__ __device__ inline size_t table_bytes(int T, bool staged = true) {
  return (size_t)T * (staged ? 20 : 14);
}

__device__ __forceinline__ WarpTables carve(unsigned char *w, int T, bool staged = true) {
  WarpTables t;
  t.acc = (double *)w;
  t.pval = staged ? t.acc + T / 2 : nullptr;
  t.keys = (int *)(t.acc + (staged ? T : T / 2));
  t.pos = t.keys + T;
  t.list = t.pos + T;
  t.pcol = staged ? t.list + T / 2 : nullptr;
  return t;
}

// acc[pos(col[p])] += val[p] for p in [0, np) in index order (bit-exact sequential
// order per accumulator): 32 staged products per step, lanes that hit the same
// accumulator are serialised in lane order by their group leader.
__device__ __forceinline__ void ordered_accumulate(WarpTables t, unsigned mask, int np, int lane) {
  for (int c = 0; c < np; c += 32) {
    int p = c + lane;
    bool valid = p < np;
    int pos = valid ? t.pos[hash_find(t.keys, mask, t.pcol[p])] : -1 - lane;
    unsigned grp = __match_any_sync(0xffffffffu, pos);
    if (valid && lane == __ffs(grp) - 1) {
      double s = t.acc[pos];
      unsigned m = grp;
      while (m) {
        int l = __ffs(m) - 1;
        s = __dadd_rn(s, t.pval[c + l]);
        m &= m - 1;
      }
      t.acc[pos] = s;
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void table_clear(WarpTables t, int T, int lane) {
  for (int i = lane; i < T; i += 32) t.keys[i] = -1;
  __syncwarp();
}

template <int E>
__device__ __forceinline__ void table_sort_regs(WarpTables t, int T, int u, int lane) {
  // compact (key, slot) pairs: keys into list, slots into the (not yet used) acc area
  int *sl = (int *)t.acc;
  int filled = 0;
  MG_DCHECK(u <= 32 * E && u <= T / 2);
  for (int i0 = 0; i0 < T; i0 += 32) {
    int k = t.keys[i0 + lane];
    unsigned bal = __ballot_sync(0xffffffffu, k != -1);
    if (k != -1) {
      int p = filled + __popc(bal & ((1u << lane) - 1));
      MG_DCHECK(p < u);
      t.list[p] = k;
      sl[p] = i0 + lane;
    }
    filled += __popc(bal);
  }
  __syncwarp();
  int k[E], v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int m = lane * E + e;
    k[e] = m < u ? t.list[m] : 0x7fffffff;
    v[e] = m < u ? sl[m] : -1;
  }
  __syncwarp();
  warp_sort_regs<E>(k, v, lane);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    int m = lane * E + e;
    if (m < u) {
      t.list[m] = k[e];
      t.pos[v[e]] = m;
    }
  }
  __syncwarp();
}

// gather the u inserted keys into list[0..u) sorted ascending; pos[slot] = rank
__device__ __forceinline__ void table_sort(WarpTables t, int T, int u, int lane) {
  if (u <= 32) { table_sort_regs<1>(t, T, u, lane); return; }
  if (u <= 64) { table_sort_regs<2>(t, T, u, lane); return; }
  if (u <= 128) { table_sort_regs<4>(t, T, u, lane); return; }
  unsigned mask = (unsigned)T - 1;
  int P = 32;
  while (P < u) P <<= 1;
  MG_DCHECK(P <= T / 2);  // list holds T/2 keys
  int filled = 0;
  for (int i0 = 0; i0 < T; i0 += 32) {
    int k = t.keys[i0 + lane];
    unsigned bal = __ballot_sync(0xffffffffu, k != -1);
    if (k != -1) t.list[filled + __popc(bal & ((1u << lane) - 1))] = k;
    filled += __popc(bal);
  }
  MG_DCHECK(filled == u);
  for (int i = u + lane; i < P; i += 32) t.list[i] = 0x7fffffff;
  __syncwarp();
  warp_bitonic(t.list, P, lane);
  for (int q = lane; q < u; q += 32) t.pos[hash_find(t.keys, mask, t.list[q])] = q;
  __syncwarp();
}

// Row lists binned by an upper bound ub on the row's staged entries / keys:
// bin b < NBIN holds rows with ub <= 32 << b and uses T = 64 << b table slots;
// bin NBIN (the last) uses global-memory tables with T = pow2 >= 2 ub.
static const int NBIN = 7;   // smem bins up to ub <= 2048 (T = 4096)
struct RowBins {
  int cnt[NBIN + 1] = {};
  int off[NBIN + 1] = {};
  DBuf<int> rows;          // all rows grouped by bin
  DBuf<int> gsize;         // global bin: table slots per row
  DBuf<int64_t> goff;      // global bin: byte offsets into pool
  DBuf<unsigned char> pool;
  // layout of the global tables: 0 = WarpTables (14T), 1 = keys only (4T),
  // 2 = SpGEMM fill tables (14T + 256)
  void build(const int *ub_dev, int m, int layout = 0);
};

}  // namespace mg
