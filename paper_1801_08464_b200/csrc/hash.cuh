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
  int *keys;    // T
  int *pos;     // T
  int *list;    // T/2
  double *acc;  // T/2
};

// per-warp table bytes for T slots: acc (T/2 f64) | keys (T) | pos (T) | list (T/2)
__host__ __device__ inline size_t table_bytes(int T) { return (size_t)T * 14; }

__device__ __forceinline__ WarpTables carve(unsigned char *w, int T) {
  WarpTables t;
  t.acc = (double *)w;
  t.keys = (int *)(w + (size_t)T / 2 * 8);
  t.pos = t.keys + T;
  t.list = t.pos + T;
  return t;
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

// Row lists binned by an upper bound on the row's distinct keys:
// bin 0: ub <= 128 (T=256), 1: <= 512 (T=1024), 2: <= 2048 (T=4096),
// 3: global-memory tables with T = pow2 >= 2 ub.
struct RowBins {
  int cnt[4] = {0, 0, 0, 0};
  int off[4] = {0, 0, 0, 0};
  DBuf<int> rows;          // all rows grouped by bin
  DBuf<int> gsize;         // bin 3: table slots per row
  DBuf<int64_t> goff;      // bin 3: byte offsets into pool
  DBuf<unsigned char> pool;
  void build(const int *ub_dev, int m);
};

}  // namespace mg
