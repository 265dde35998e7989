// Warp-level shared-memory hash tables, bitonic sort and row binning used by
// the SpGEMM and the extended+i interpolation kernels.
#pragma once
#include "common.cuh"

namespace mg {

__device__ __forceinline__ unsigned hash_k(int k, unsigned mask) {
  return ((unsigned)k * 2654435761u) & mask;
}

// insert key; returns 1 if newly inserted (keys[] initialised to -1)
__device__ __forceinline__ int hash_insert(int *keys, unsigned mask, int k) {
  unsigned h = hash_k(k, mask);
  while (true) {
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
  while (keys[h] != k) h = (h + 1) & mask;
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

// gather the u inserted keys into list[0..u) sorted ascending; pos[slot] = rank
__device__ __forceinline__ void table_sort(WarpTables t, int T, int u, int lane) {
  unsigned mask = (unsigned)T - 1;
  int P = 32;
  while (P < u) P <<= 1;
  int filled = 0;
  for (int i0 = 0; i0 < T; i0 += 32) {
    int k = t.keys[i0 + lane];
    unsigned bal = __ballot_sync(0xffffffffu, k != -1);
    if (k != -1) t.list[filled + __popc(bal & ((1u << lane) - 1))] = k;
    filled += __popc(bal);
  }
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
