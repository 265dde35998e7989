// SpMV family: scalar CSR (sub-warp per row, fused epilogues) and block-CSR
// b = 2 / 3 (lane group per block row, vectorised block loads).
//
// Replaces scipy csr_matvec at every hot call site:
// the GMRES operator `a @ v` (linsolve.py:100), MGR residual / R / P products
// (mgr.py:347,355,357) and the AMG residual / restriction / prolongation
// (amg.py:347,361-364).  HBM-bound: algorithmic bytes per launch
// nnz*(8 b^2 + 4) + 4 (nr + 1) + 8 b (nc + nr).
#include "ops.cuh"

#include <cub/cub.cuh>

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
// y = [e_F; 0] + A x with the F values merged on the fly (MGR prolongation after
// an F-relaxation from zero: replaces fc_merge + y += A x, same sums)
struct EpiMergeAdd {
  const int *fmap;
  const double *ef;
  double *y;
  __device__ void operator()(int r, double s) const {
    const int f = fmap[r];
    y[r] = (f >= 0 ? ef[f] : 0.0) + s;
  }
};
// y = A x with the next level's first pre-sweep from zero folded in (same products
// as vmul: bs = sign * y, xo = d * bs)
struct EpiStoreScale {
  double *y;
  const double *sign;
  double *bs;
  const double *d;
  double *xo;
  __device__ void operator()(int r, double s) const {
    y[r] = s;
    if (sign) {
      s = sign[r] * s;
      bs[r] = s;
    }
    xo[r] = d[r] * s;
  }
};
// rows F of a residual, r_F = b[rows] - A[F, :] x, stored densely in F order, with the
// F-relaxation AMG's first pre-sweep from zero folded in as in EpiStoreScale (replaces
// residual on the whole of A + gather_scale: same differences, same products)
struct EpiResidRowsScale {
  const double *b;
  const int *rows;
  double *y;
  const double *sign;
  double *bs;
  const double *d;
  double *xo;
  __device__ void operator()(int i, double s) const {
    s = b[rows[i]] - s;
    y[i] = s;
    if (xo) {
      if (sign) {
        s = sign[i] * s;
        bs[i] = s;
      }
      xo[i] = d[i] * s;
    }
  }
};
struct EpiJacobi {
  const double *x, *b, *dinv;
  double *xo;
  __device__ void operator()(int i, double s) const { xo[i] = x[i] + dinv[i] * (b[i] - s); }
};

// x gather functor of the SpMV kernels
struct XPlain {
  const double *x;
  __device__ __forceinline__ double operator()(int c) const { return __ldg(x + c); }
};
// VS lanes cooperate on one row; each lane keeps U independent (value, column)
// loads in flight before the dependent x gathers, so a warp has VS*U*12 B of
// matrix traffic outstanding per round trip.  Groups stride over rows (grid
// sized to the resident capacity); every lane runs the shuffle (uniform loop).
template <int VS, int U, int IK, class Epi, class XG>
__global__ void __launch_bounds__(256) k_csr(int nr, const int *__restrict__ rows,
                                             const int *__restrict__ rp,
                                             const void *__restrict__ ci,
                                             const int *__restrict__ dict, unsigned long long mul,
                                             const double *__restrict__ v,
                                             XG x, Epi epi) {
  // IK: column encoding (SpmvPlan::ik) in CSR order: 0 int32, 1 u8 -> dict, 2 int16,
  // codes relative to anchor(row) = (row * mul) >> 32
  __shared__ int tbl[IK == 1 ? 256 : 1];
  PDL_ENTRY();
  if (IK == 1) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tbl[i] = __ldg(dict + i);
    __syncthreads();
  }
  const int lane = threadIdx.x % VS;
  const int g0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / VS);
  const int ng = (int)((int64_t)gridDim.x * blockDim.x / VS);
  const int warp_first = (int)(((int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31)) / VS);
  for (int idx = g0, wf = warp_first; wf < nr; idx += ng, wf += ng) {
    double sum = 0.0;
    int row = idx < nr ? (rows ? __ldg(rows + idx) : idx) : nr;
    if (idx < nr) {
      const int anc = IK ? (int)(((unsigned long long)row * mul) >> 32) : 0;
      int s = __ldg(rp + row), e = __ldg(rp + row + 1);
      for (int k0 = s; k0 < e; k0 += VS * U) {
        double vv[U];
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          int k = k0 + lane + u * VS;
          bool ok = k < e;
          vv[u] = ok ? __ldcs(v + k) : 0.0;
          if (IK == 0) cc[u] = ok ? __ldcs(static_cast<const int *>(ci) + k) : -1;
          else if (IK == 1) cc[u] = ok ? anc + tbl[__ldcs(static_cast<const unsigned char *>(ci) + k)] : -1;
          else cc[u] = ok ? anc + (int)__ldcs(static_cast<const short *>(ci) + k) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (cc[u] >= 0) sum += vv[u] * x(cc[u]);
      }
    }
#pragma unroll
    for (int off = VS / 2; off > 0; off >>= 1) sum += __shfl_down_sync(0xffffffffu, sum, off, VS);
    if (idx < nr && lane == 0) epi(row, sum);
  }
}

// ---- SELL-32: one thread per row, loads coalesced across the 32 rows of a slice ----
// IK selects the column encoding (SpmvPlan::ik): 0 int32, 1 u8 code -> dict, 2 int16
// code; codes are relative to anchor(row) = (row * mul) >> 32 and packed 4 / 2 per
// 32-bit word so that one word load per thread covers 4 / 2 entries (a coalesced
// 128 B warp access).  Slice lengths are multiples of 4 (build_sell).
__device__ __forceinline__ int sell_anchor(int row, unsigned long long mul) {
  return (int)(((unsigned long long)row * mul) >> 32);
}
template <int IK>
__device__ __forceinline__ void sell_cols4(const void *__restrict__ ci, int base, int wbase, int k, int anc,
                                           const int *tbl, int (&cc)[4]) {
  if (IK == 0) {
#pragma unroll
    for (int u = 0; u < 4; ++u) cc[u] = __ldcs(static_cast<const int *>(ci) + base + (k + u) * 32);
  } else if (IK == 1) {
    const unsigned w = __ldcs(static_cast<const unsigned *>(ci) + wbase + (k >> 2) * 32);
#pragma unroll
    for (int u = 0; u < 4; ++u) cc[u] = anc + tbl[(w >> (8 * u)) & 255u];
  } else {
    const unsigned *p = static_cast<const unsigned *>(ci) + wbase + (k >> 1) * 32;
    const unsigned w0 = __ldcs(p), w1 = __ldcs(p + 32);
    cc[0] = anc + (int)(short)(w0 & 0xffffu);
    cc[1] = anc + (int)(short)(w0 >> 16);
    cc[2] = anc + (int)(short)(w1 & 0xffffu);
    cc[3] = anc + (int)(short)(w1 >> 16);
  }
}
// perm (SELL-C-sigma, may be null): slice position -> row; rlen is by position
template <int UNR, int IK, bool PF, class Epi, class XG>
__global__ void __launch_bounds__(256) k_sell(int nr, const int *__restrict__ sptr, const int *__restrict__ rlen,
                                              const int *__restrict__ perm,
                                              const void *__restrict__ ci, const int *__restrict__ dict,
                                              unsigned long long mul, const double *__restrict__ v,
                                              XG x, Epi epi) {
  static_assert(UNR % 4 == 0, "SELL unroll is a multiple of the 4-entry code word");
  __shared__ int tbl[IK == 1 ? 256 : 1];
  PDL_ENTRY();
  if (IK == 1) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) tbl[i] = __ldg(dict + i);
    __syncthreads();
  }
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= nr) return;
  const int row = perm ? __ldg(perm + pos) : pos;
  const int sbase = __ldg(sptr + (pos >> 5));
  const int base = sbase + (pos & 31);
  const int wbase = (IK == 1 ? (sbase >> 2) : (sbase >> 1)) + (pos & 31);
  const int anc = IK ? sell_anchor(row, mul) : 0;
  const int len = __ldg(rlen + pos);
  double sum = 0.0;
  int k = 0;
  if (PF && len >= UNR) {
    // software pipelined: chunk i+1's values / codes are issued before chunk i's
    // products, so a thread keeps two chunks of matrix loads in flight
    double vv[UNR];
    int cc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) vv[u] = __ldcs(v + base + u * 32);
#pragma unroll
    for (int q = 0; q < UNR / 4; ++q) {
      int c4[4];
      sell_cols4<IK>(ci, base, wbase, 4 * q, anc, tbl, c4);
#pragma unroll
      for (int u = 0; u < 4; ++u) cc[4 * q + u] = c4[u];
    }
    for (;;) {
      double xg[UNR];
#pragma unroll
      for (int u = 0; u < UNR; ++u) xg[u] = x(cc[u]);
      k += UNR;
      const bool more = k + UNR <= len;
      double vn[UNR];
      if (more) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) vn[u] = __ldcs(v + base + (k + u) * 32);
#pragma unroll
        for (int q = 0; q < UNR / 4; ++q) {
          int c4[4];
          sell_cols4<IK>(ci, base, wbase, k + 4 * q, anc, tbl, c4);
#pragma unroll
          for (int u = 0; u < 4; ++u) cc[4 * q + u] = c4[u];
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) sum += vv[u] * xg[u];
      if (!more) break;
#pragma unroll
      for (int u = 0; u < UNR; ++u) vv[u] = vn[u];
    }
  }
  for (; k + UNR <= len; k += UNR) {
    double vv[UNR];
    int cc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) vv[u] = __ldcs(v + base + (k + u) * 32);
#pragma unroll
    for (int q = 0; q < UNR / 4; ++q) {
      int c4[4];
      sell_cols4<IK>(ci, base, wbase, k + 4 * q, anc, tbl, c4);
#pragma unroll
      for (int u = 0; u < 4; ++u) cc[4 * q + u] = c4[u];
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) sum += vv[u] * x(cc[u]);
  }
  for (; k < len; k += 4) {
    const int m = len - k;  // 1..UNR-1 entries left; the code word is padded
    double vv[4];
    int cc[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) vv[u] = u < m ? __ldcs(v + base + (k + u) * 32) : 0.0;
    if (IK == 0) {
#pragma unroll
      for (int u = 0; u < 4; ++u) cc[u] = u < m ? __ldcs(static_cast<const int *>(ci) + base + (k + u) * 32) : 0;
    } else {
      sell_cols4<IK>(ci, base, wbase, k, anc, tbl, cc);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < m) sum += vv[u] * x(cc[u]);
  }
  epi(row, sum);
}

// ---- SELL-32, u8 codes, the matrix streamed by bulk copies (TMA 1-D) ----------
// A CTA of 256 threads owns 8 consecutive slices (256 rows).  Stage t carries
// entries [4t, 4t+4) of all 8 slices: per slice one 1 KB copy of the values and
// one 128 B copy of the packed codes (cp.async.bulk into shared memory, completion
// counted on the stage's mbarrier).  D stages are in flight; thread 0 refills a
// stage after the CTA-wide barrier that ends its consumption.  Each thread sums its
// row in entry order from shared memory, so results equal k_sell's bit for bit.
// (The streamed loads no longer occupy registers or load slots: the x gathers issue
// as soon as a stage lands.)  MG_SELL_TMA=1 selects it for u8-coded, unpermuted
// SELL operators of <= 64 entries per row.
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t *b, unsigned parity) {
  unsigned ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(b)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Per-warp pipelines: warp w of the CTA streams its own slice; stage t = entries
// [E t, E t + E) (one E x 32-value copy and one E x 8-byte code copy); TMA_D stages
// in flight per warp; lane 0 refills a stage after a __syncwarp, so slices of
// different lengths never wait for each other.
template <class Epi, int TMA_D, int TMA_E, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_sell_tma(int nr, const int *__restrict__ sptr, const int *__restrict__ rlen,
                                                  const unsigned *__restrict__ codes, const int *__restrict__ dict,
                                                  unsigned long long mul, const double *__restrict__ v, XPlain x,
                                                  Epi epi) {
  __shared__ int tbl[256];
  __shared__ __align__(128) double sv[WPB][TMA_D][TMA_E * 32];
  __shared__ __align__(128) unsigned sc[WPB][TMA_D][TMA_E * 8];
  __shared__ __align__(8) uint64_t full[WPB][TMA_D];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int ns_total = (nr + 31) >> 5;
  const int s = blockIdx.x * WPB + w;
  if (lane == 0) {
    for (int d = 0; d < TMA_D; ++d) mbar_init(&full[w][d], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  PDL_ENTRY();
  for (int i = tid; i < 256; i += blockDim.x) tbl[i] = __ldg(dict + i);
  __syncthreads();
  const int sb = s < ns_total ? __ldg(sptr + s) : 0;
  const int sl = s < ns_total ? (__ldg(sptr + s + 1) - sb) >> 5 : 0;  // entries per row slot (multiple of 4)
  const int nst = (sl + TMA_E - 1) / TMA_E;
  auto issue = [&](int t) {
    const int b = t % TMA_D;
    const int e = min(TMA_E, sl - TMA_E * t);  // entries in this stage (a multiple of 4)
    mbar_expect_tx(&full[w][b], (unsigned)e * 32u * 9u);
    bulk_g2s(sv[w][b], v + sb + 32 * TMA_E * t, (unsigned)e * 256u, &full[w][b]);
    bulk_g2s(sc[w][b], codes + (sb >> 2) + 8 * TMA_E * t, (unsigned)e * 32u, &full[w][b]);
  };
  if (lane == 0)
    for (int t = 0; t < TMA_D && t < nst; ++t) issue(t);
  const int row = s * 32 + lane;
  const bool live = row < nr;
  const int len = live ? __ldg(rlen + row) : 0;
  const int anc = sell_anchor(row, mul);
  double sum = 0.0;
  for (int t = 0; t < nst; ++t) {
    const int b = t % TMA_D;
    const int k0 = TMA_E * t;
    if (k0 < len) {
      const unsigned par = (unsigned)((t / TMA_D) & 1);
      unsigned spins = 0;
      while (!mbar_try_wait(&full[w][b], par))
        if (++spins > (1u << 28)) __trap();  // a lost stage must fail loudly, never hang
#pragma unroll
      for (int q = 0; q < TMA_E / 4; ++q) {
        const int k = k0 + 4 * q;
        if (k < len) {
          const unsigned cw = sc[w][b][q * 32 + lane];
          const int m = len - k;
          double vv[4];
          int cc[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            vv[u] = sv[w][b][(4 * q + u) * 32 + lane];
            cc[u] = anc + tbl[(cw >> (8 * u)) & 255u];
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < m) sum += vv[u] * x(cc[u]);
        }
      }
    }
    __syncwarp();  // every lane is done with stage buffer b
    if (lane == 0 && t + TMA_D < nst) issue(t + TMA_D);
  }
  if (live) epi(row, sum);
}

static int sell_tma() {  // MG_SELL_TMA=1/2/3: (stages, entries) = (4, 4) / (3, 8) / (2, 16); 0 off
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_SELL_TMA");
    on = e ? atoi(e) : 0;
    return on;
  }();
  return on;
}

// per slice: max row length (warp per slice); Q rounds the slice length up to a
// multiple of Q entries (4 for the scalar SELL copy: whole code words)
__global__ void k_sell_len(int nr, int ns, const int *rp, const int *perm, int *rlen, int *slen, int q) {
  int s = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (s >= ns) return;
  int pos = s * 32 + lane;
  int row = pos < nr && perm ? perm[pos] : pos;
  int len = pos < nr ? rp[row + 1] - rp[row] : 0;
  if (pos < nr) rlen[pos] = len;
  int m = len;
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) slen[s] = (m + q - 1) / q * q * 32;
}
__global__ void k_sell_fill(int nr, const int *rp, const int *ci, const double *v, const int *sptr,
                            const int *perm, int *sci, double *sv) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= nr) return;
  const int row = perm ? perm[pos] : pos;
  int base = sptr[pos >> 5] + (pos & 31);
  int s = rp[row], e = rp[row + 1];
  for (int k = 0; k < e - s; ++k) {
    if (sci) sci[base + k * 32] = ci[s + k];
    sv[base + k * 32] = v[s + k];
  }
}

// ---- column compression (SpmvPlan::ik) ------------------------------------------
// code = col - anchor(row).  One pass over every stored column gives the code
// range [lo, hi] (min / max over all entries, so an unsorted row -- legal in
// scipy CSR -- still gets codes inside the range and never indexes the bitmap
// out of bounds).  When hi - lo < CWIN a second pass marks the distinct codes in
// a shared-memory bitmap per block (merged into a global one), and one block
// ranks them: <= 256 distinct -> u8 codes through a table.
constexpr int CWIN = 1 << 17;        // bitmap window (bits): 16 KB of shared memory
constexpr int CWORDS = CWIN / 32;
__global__ void __launch_bounds__(256) k_code_range(int nr, const int *__restrict__ rp,
                                                    const int *__restrict__ ci, unsigned long long mul, int *mm) {
  int lo = INT_MAX, hi = INT_MIN;
  const int lane = threadIdx.x & 7;
  const int g0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3);
  const int ng = (int)(((int64_t)gridDim.x * blockDim.x) >> 3);
  for (int row = g0; row < nr; row += ng) {
    const int anc = sell_anchor(row, mul);
    const int s = __ldg(rp + row), e = __ldg(rp + row + 1);
    for (int k = s + lane; k < e; k += 8) {
      const int t = __ldg(ci + k) - anc;
      lo = min(lo, t);
      hi = max(hi, t);
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mm, lo);
    atomicMax(mm + 1, hi);
  }
}
// distinct codes in [lo, lo + nw * 32): block bitmap in shared memory, nonzero
// words merged into the global bitmap
__global__ void __launch_bounds__(256) k_code_bitmap(int nr, const int *__restrict__ rp, const int *__restrict__ ci,
                                                     unsigned long long mul, int lo, int nw, unsigned *bm) {
  __shared__ unsigned sb[CWORDS];
  for (int w = threadIdx.x; w < nw; w += blockDim.x) sb[w] = 0u;
  __syncthreads();
  const int lane = threadIdx.x & 7;
  const int g0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3);
  const int ng = (int)(((int64_t)gridDim.x * blockDim.x) >> 3);
  for (int row = g0; row < nr; row += ng) {
    const int anc = sell_anchor(row, mul);
    const int s = __ldg(rp + row), e = __ldg(rp + row + 1);
    for (int k = s + lane; k < e; k += 8) {
      const unsigned t = (unsigned)(__ldg(ci + k) - anc - lo), bit = 1u << (t & 31);
      MG_DCHECK(t < (unsigned)nw * 32u);
      // a stencil operator has a few dozen codes: after their first sighting the
      // bits are only read (a shared atomic per entry on the same few words
      // serialises the block)
      if (!(sb[t >> 5] & bit)) atomicOr(sb + (t >> 5), bit);
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nw; w += blockDim.x)
    if (sb[w]) atomicOr(bm + w, sb[w]);
}
// per-word popcounts -> exclusive prefix (one block), the distinct count into
// mm[2] and the code table dict[rank] = code for the first 256 codes (ascending)
__global__ void __launch_bounds__(1024) k_code_dict(const unsigned *bm, int nw, int lo, int *wpre, int *mm,
                                                    int *dict) {
  __shared__ int part[1024];
  const int per = (nw + 1023) / 1024;
  const int t = threadIdx.x;
  int c = 0;
  for (int i = 0; i < per; ++i) {
    const int w = t * per + i;
    if (w < nw) c += __popc(bm[w]);
  }
  part[t] = c;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    int v = t >= o ? part[t - o] : 0;
    __syncthreads();
    part[t] += v;
    __syncthreads();
  }
  int run = part[t] - c;
  for (int i = 0; i < per; ++i) {
    const int w = t * per + i;
    if (w >= nw) break;
    unsigned bits = bm[w];
    wpre[w] = run;
    while (bits) {
      const int b = __ffs(bits) - 1;
      bits &= bits - 1;
      if (run < 256) dict[run] = lo + w * 32 + b;
      ++run;
    }
  }
  if (t == 1023) mm[2] = part[1023];
}
// codes of row `row` packed into its slice words (thread per row)
template <int IK>
__global__ void k_code_fill(int nr, const int *rp, const int *ci, const int *sptr, const int *perm,
                            unsigned long long mul, int lo, const unsigned *bm, const int *wpre, unsigned *code) {
  const int pos = blockIdx.x * blockDim.x + threadIdx.x;
  if (pos >= nr) return;
  const int row = perm ? perm[pos] : pos;
  constexpr int PW = IK == 1 ? 4 : 2;  // codes per word
  const int sbase = sptr[pos >> 5];
  unsigned *out = code + (sbase / PW) + (pos & 31);
  const int anc = sell_anchor(row, mul);
  const int s = rp[row], e = rp[row + 1];
  unsigned w = 0;
  for (int k = 0; k < e - s; ++k) {
    const int d = ci[s + k] - anc;
    unsigned c;
    if (IK == 1) {
      const unsigned t = (unsigned)(d - lo);
      c = (unsigned)(wpre[t >> 5] + __popc(bm[t >> 5] & ((1u << (t & 31)) - 1u)));
    } else {
      c = (unsigned)d & 0xffffu;
    }
    w |= c << ((k % PW) * (32 / PW));
    if (k % PW == PW - 1) {
      out[(k / PW) * 32] = w;
      w = 0;
    }
  }
  if ((e - s) % PW) out[((e - s) / PW) * 32] = w;
}

// codes in CSR order (8 lanes per row)
template <int IK>
__global__ void k_code_fill_csr(int nr, const int *__restrict__ rp, const int *__restrict__ ci,
                                unsigned long long mul, int lo, const unsigned *bm, const int *wpre, void *code) {
  const int lane = threadIdx.x & 7;
  const int g0 = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 3);
  const int ng = (int)(((int64_t)gridDim.x * blockDim.x) >> 3);
  for (int row = g0; row < nr; row += ng) {
    const int anc = sell_anchor(row, mul);
    const int s = rp[row], e = rp[row + 1];
    for (int k = s + lane; k < e; k += 8) {
      const int d = ci[k] - anc;
      if (IK == 1) {
        const unsigned t = (unsigned)(d - lo);
        static_cast<unsigned char *>(code)[k] =
            (unsigned char)(wpre[t >> 5] + __popc(bm[t >> 5] & ((1u << (t & 31)) - 1u)));
      } else {
        static_cast<short *>(code)[k] = (short)d;
      }
    }
  }
}

static int code_mode() {  // MG_SELL_CODES=0 keeps int32 columns
  static const int m = [] {
    int m = -1;
    const char *e = getenv("MG_SELL_CODES");
    m = e ? atoi(e) : 1;
    return m;
  }();
  return m;
}

// choose and build the column encoding of a SELL copy (padded >= 0) or of the
// CSR arrays (padded < 0); one or two host round trips
static void build_codes(const Csr &a, SpmvPlan &pl, int64_t padded) {
  pl.ik = 0;
  if (!code_mode() || a.nr == 0 || a.nnz == 0) return;
  pl.mul = (unsigned long long)(((unsigned __int128)(unsigned)a.nc << 32) / (unsigned)a.nr);
  DBuf<int> mm(3);
  dset_i32(mm.p, {INT_MAX, INT_MIN, 0});
  k_code_range<<<grid_for((int64_t)a.nr * 8, 256, g_ctx->num_sms * 8), 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p,
                                                                                           pl.mul, mm.p);
  check_launch("code_range");
  int st[3];
  d2h(st, mm.p, 2 * sizeof(int));
  const int lo = st[0], hi = st[1];
  const bool fits16 = lo >= -32768 && hi <= 32767;
  DBuf<unsigned> bm;
  DBuf<int> wpre;
  if ((int64_t)hi - lo < CWIN) {
    const int nw = (int)(((int64_t)hi - lo) / 32 + 1);
    bm.alloc(nw);
    wpre.alloc(nw);
    dzero(bm.p, sizeof(unsigned) * nw);
    pl.dict.alloc(256);
    dzero(pl.dict.p, 256 * sizeof(int));
    k_code_bitmap<<<grid_for((int64_t)a.nr * 8, 256, g_ctx->num_sms * 8), 256, 0, stream()>>>(
        a.nr, a.rp.p, a.ci.p, pl.mul, lo, nw, bm.p);
    check_launch("code_bitmap");
    k_code_dict<<<1, 1024, 0, stream()>>>(bm.p, nw, lo, wpre.p, mm.p, pl.dict.p);
    check_launch("code_dict");
    d2h(st + 2, mm.p + 2, sizeof(int));
    if (st[2] <= 256) pl.ik = 1;
  }
  if (!pl.ik && fits16) pl.ik = 2;
  if (pl.ik != 1) pl.dict.release();
  if (!pl.ik) return;
  if (padded < 0) {  // CSR order: 1 or 2 bytes per stored entry
    pl.scode.alloc((size_t)((a.nnz * pl.idx_bytes() + 3) / 4));
    const int g = grid_for((int64_t)a.nr * 8, 256, g_ctx->num_sms * 8);
    if (pl.ik == 1)
      k_code_fill_csr<1><<<g, 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, pl.mul, lo, bm.p, wpre.p, pl.scode.p);
    else
      k_code_fill_csr<2><<<g, 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, pl.mul, lo, bm.p, wpre.p, pl.scode.p);
    check_launch("code_fill_csr");
    return;
  }
  pl.scode.alloc((size_t)(padded / (pl.ik == 1 ? 4 : 2)));
  if (pl.ik == 1)
    k_code_fill<1><<<grid_for(a.nr, 256), 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, pl.sptr.p, pl.perm.p,
                                                              pl.mul, lo, bm.p, wpre.p, pl.scode.p);
  else
    k_code_fill<2><<<grid_for(a.nr, 256), 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, pl.sptr.p, pl.perm.p,
                                                              pl.mul, lo, bm.p, wpre.p, pl.scode.p);
  check_launch("code_fill");
}

static int sell_min_rows() {  // MG_SELL_MIN_ROWS: smallest operator given a SELL copy
  static const int v = [] {
    int v = -1;
    const char *e = getenv("MG_SELL_MIN_ROWS");
    v = e ? atoi(e) : 32768;
    return v;
  }();
  return v;
}

static double sell_min_avg() {
  static const double v = [] {
    double v = -1.0;
    const char *e = getenv("MG_SELL_MIN_AVG");
    v = e ? atof(e) : 3.0;
    return v;
  }();
  return v;
}

// SELL-C-sigma: rows sorted by length (descending, stable) inside windows of
// SIGMA rows, so the 32 rows of a slice have similar lengths (irregular coarse
// AMG levels).  perm[pos] = row.  One block per window.
constexpr int SIGMA = 1024;
__global__ void __launch_bounds__(256) k_sell_sort_window(int nr, const int *__restrict__ rp, int *perm) {
  using Sort = cub::BlockRadixSort<unsigned, 256, SIGMA / 256, int>;
  __shared__ typename Sort::TempStorage tmp;
  unsigned key[SIGMA / 256];
  int val[SIGMA / 256];
  const int base = blockIdx.x * SIGMA;
#pragma unroll
  for (int i = 0; i < SIGMA / 256; ++i) {
    const int pos = base + threadIdx.x * (SIGMA / 256) + i;
    key[i] = pos < nr ? ~(unsigned)(rp[pos + 1] - rp[pos]) : 0xffffffffu;
    val[i] = pos;
  }
  Sort(tmp).Sort(key, val);
#pragma unroll
  for (int i = 0; i < SIGMA / 256; ++i) {
    const int pos = base + threadIdx.x * (SIGMA / 256) + i;
    if (pos < nr) perm[pos] = val[i];
  }
}

// Sorted copies only for operators with rows for about one full wave of
// threads (one thread per row): measured at 128^3, coarse A_1 (518K rows)
// 115 -> 110 us and F-relax A_1 (733K) 50 -> 39 us, but A_2 (128K rows, 123
// per row) 34 -> 53 us, the long per-thread row loops left without enough
// warps to hide latency.  MG_SELL_SIGMA=<min rows>, 0 disables.
static int sell_sigma_min_rows() {
  static const int v = [] {
    int v = -1;
    const char *e = getenv("MG_SELL_SIGMA");
    v = e ? atoi(e) : 262144;
    return v;
  }();
  return v;
}

static void build_sell(const Csr &a, SpmvPlan &pl) {
  int ns = (a.nr + 31) / 32;
  DBuf<int> slen((size_t)ns + 1);
  pl.rlen.alloc(a.nr);
  k_sell_len<<<grid_for((int64_t)ns * 32, 256), 256, 0, stream()>>>(a.nr, ns, a.rp.p, nullptr, pl.rlen.p, slen.p,
                                                                      4);
  check_launch("sell_len");
  DBuf<int64_t> sp64((size_t)ns + 1);
  int64_t padded = exclusive_scan_i32_to_i64(slen.p, sp64.p, ns);
  // padded slots beyond a row's length are never loaded (predicated by rlen), so
  // padding costs footprint and idle lanes, not bandwidth: accept up to 2x for
  // short rows (where CSR lane groups are inefficient), 1.15x otherwise
  // (measured: irregular long-row coarse levels lose with SELL)
  double avg = (double)a.nnz / (a.nr ? a.nr : 1);
  static const double cap_long = [] {
    double cap_long = -1.0;
    const char *e = getenv("MG_SELL_CAP_LONG");
    cap_long = e ? atof(e) : 1.15;
    return cap_long;
  }();
  static const double cap_short = [] {
    double cap_short = -1.0;
    const char *e = getenv("MG_SELL_CAP_SHORT");
    cap_short = e ? atof(e) : 2.0;
    return cap_short;
  }();
  double cap = avg <= 16.0 ? cap_short : cap_long;
  // (+ the rounding of slice lengths to whole code words: at most 3 x 32 per slice)
  auto over = [&](int64_t pd) { return pd > (int64_t)(cap * (double)a.nnz) + 4096 + 96LL * ns || pd > 2000000000LL; };
  // Rows of very different lengths inside a slice (irregular AMG levels; the
  // MGR P = [W_p; I] with its 1-entry C rows next to ~6-entry F rows) leave
  // lanes idle for the slice's longest row: sort by length inside SIGMA windows
  // when that is needed to pass the cap, or when it cuts the padded slots by 20%
  const bool ragged = padded > (int64_t)(1.3 * (double)a.nnz) + 4096 + 96LL * ns;
  if ((over(padded) || ragged) && sell_sigma_min_rows() > 0 && a.nr >= sell_sigma_min_rows()) {
    DBuf<int> perm(a.nr), rl2(a.nr), sl2((size_t)ns + 1);
    k_sell_sort_window<<<(a.nr + SIGMA - 1) / SIGMA, 256, 0, stream()>>>(a.nr, a.rp.p, perm.p);
    check_launch("sell_sort_window");
    k_sell_len<<<grid_for((int64_t)ns * 32, 256), 256, 0, stream()>>>(a.nr, ns, a.rp.p, perm.p, rl2.p, sl2.p, 4);
    check_launch("sell_len_sorted");
    const int64_t p2 = exclusive_scan_i32_to_i64(sl2.p, sp64.p, ns);
    if (!over(p2) && (over(padded) || (double)p2 < 0.8 * (double)padded)) {
      pl.perm = std::move(perm);
      pl.rlen = std::move(rl2);
      slen = std::move(sl2);
      padded = p2;
    }
  }
  if (over(padded)) {
    pl.rlen.release();
    return;
  }
  pl.sptr.alloc((size_t)ns + 1);
  exclusive_scan_i32_to_i32(slen.p, pl.sptr.p, ns);
  build_codes(a, pl, padded);
  if (!pl.ik) pl.sci.alloc((size_t)padded);
  pl.sv.alloc((size_t)padded);
  k_sell_fill<<<grid_for(a.nr, 256), 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, a.v.p, pl.sptr.p, pl.perm.p,
                                                          pl.sci.p, pl.sv.p);
  check_launch("sell_fill");
  pl.sell = true;
}

// ---- block SELL-32 for the BCSR GMRES operator -------------------------------------
// slices of 32 block rows, block k of the slice's rows contiguous (32 b*b blocks),
// one thread per block row: every block load is a coalesced 1 KB (b = 2) warp access
template <int B>
__global__ void k_bsell_fill(int nr, const int *rp, const int *ci, const double *v, const int *sptr, int *sci,
                             double *sv) {
  int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nr) return;
  int base = sptr[row >> 5] + (row & 31);
  int s = rp[row], e = rp[row + 1];
  for (int k = 0; k < e - s; ++k) {
    sci[base + k * 32] = ci[s + k];
#pragma unroll
    for (int q = 0; q < B * B; ++q) sv[(int64_t)(base + k * 32) * B * B + q] = v[(int64_t)(s + k) * B * B + q];
  }
}

template <int B, int UNR>
__global__ void __launch_bounds__(256) k_bsell(int nr, const int *__restrict__ sptr, const int *__restrict__ rlen,
                                               const int *__restrict__ ci, const double *__restrict__ v,
                                               const double *__restrict__ x, double *__restrict__ y) {
  PDL_ENTRY();
  const int row = blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= nr) return;
  const int base = __ldg(sptr + (row >> 5)) + (row & 31);
  const int len = __ldg(rlen + row);
  double acc[B];
#pragma unroll
  for (int r = 0; r < B; ++r) acc[r] = 0.0;
  for (int k0 = 0; k0 < len; k0 += UNR) {
    double a[UNR][B * B], xc[UNR][B];
    int cc[UNR];
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int k = k0 + u;
      const int e = base + (k < len ? k : 0) * 32;
      cc[u] = k < len ? __ldcs(ci + e) : -1;
      if (B == 2) {
        const double2 *vb = reinterpret_cast<const double2 *>(v) + (int64_t)e * 2;
        double2 r0 = __ldcs(vb), r1 = __ldcs(vb + 1);
        a[u][0] = r0.x; a[u][1] = r0.y; a[u][2] = r1.x; a[u][3] = r1.y;
      } else {
#pragma unroll
        for (int q = 0; q < B * B; ++q) a[u][q] = __ldcs(v + (int64_t)e * B * B + q);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (cc[u] < 0) {
#pragma unroll
        for (int q = 0; q < B; ++q) xc[u][q] = 0.0;
        continue;
      }
      if (B == 2) {
        double2 t = __ldg(reinterpret_cast<const double2 *>(x) + cc[u]);
        xc[u][0] = t.x; xc[u][1] = t.y;
      } else {
#pragma unroll
        for (int q = 0; q < B; ++q) xc[u][q] = __ldg(x + (int64_t)cc[u] * B + q);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      if (cc[u] < 0) continue;
#pragma unroll
      for (int r = 0; r < B; ++r) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < B; ++q) t += a[u][r * B + q] * xc[u][q];
        acc[r] += t;
      }
    }
  }
  if (B == 2) {
    reinterpret_cast<double2 *>(y)[row] = make_double2(acc[0], acc[1]);
  } else {
#pragma unroll
    for (int r = 0; r < B; ++r) y[(int64_t)row * B + r] = acc[r];
  }
}

static void build_bsell(const Csr &a, SpmvPlan &pl) {
  const int B = a.b;
  int ns = (a.nr + 31) / 32;
  DBuf<int> slen((size_t)ns + 1);
  pl.rlen.alloc(a.nr);
  k_sell_len<<<grid_for((int64_t)ns * 32, 256), 256, 0, stream()>>>(a.nr, ns, a.rp.p, nullptr, pl.rlen.p, slen.p,
                                                                      1);
  check_launch("bsell_len");
  DBuf<int64_t> sp64((size_t)ns + 1);
  int64_t padded = exclusive_scan_i32_to_i64(slen.p, sp64.p, ns);
  if (padded > 2 * a.nnz + 4096 || padded * B * B > 2000000000LL) {
    pl.rlen.release();
    return;
  }
  pl.sptr.alloc((size_t)ns + 1);
  exclusive_scan_i32_to_i32(slen.p, pl.sptr.p, ns);
  pl.sci.alloc((size_t)padded);
  pl.sv.alloc((size_t)padded * B * B);
  if (B == 2)
    k_bsell_fill<2><<<grid_for(a.nr, 256), 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, a.v.p, pl.sptr.p, pl.sci.p,
                                                               pl.sv.p);
  else
    k_bsell_fill<3><<<grid_for(a.nr, 256), 256, 0, stream()>>>(a.nr, a.rp.p, a.ci.p, a.v.p, pl.sptr.p, pl.sci.p,
                                                               pl.sv.p);
  check_launch("bsell_fill");
  pl.sell = true;
}

void prepare_spmv(const Csr &a) {
  if (a.plan) return;
  if (a.b != 1) {  // block CSR (the GMRES operator): block SELL copy when large
    auto pl = std::make_unique<SpmvPlan>();
    if ((a.b == 2 || a.b == 3) && a.nr >= 32768) build_bsell(a, *pl);
    a.plan = std::move(pl);
    return;
  }
  auto pl = std::make_unique<SpmvPlan>();
  if (a.nr >= sell_min_rows() && (double)a.nnz >= sell_min_avg() * a.nr) build_sell(a, *pl);
  // large operators left in CSR (irregular long-row AMG levels): compressed
  // columns in CSR order when the codes fit
  if (!pl->sell && a.nnz >= (1 << 20) && a.nr > 0) build_codes(a, *pl, -1);
  a.plan = std::move(pl);
}

template <int B, int G, int U>
__global__ void __launch_bounds__(256) k_bsr(int nbr, const int *__restrict__ rp,
                                             const int *__restrict__ ci,
                                             const double *__restrict__ v,
                                             const double *__restrict__ x,
                                             double *__restrict__ y) {
  PDL_ENTRY();
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

// software-pipelined loop for the long-row (UNR = 8) variant: coarse A_1 (105
// per row) 77 -> 85% of HBM; the short-row variant loses with it (occupancy:
// 56 registers), A_hat 71 -> 61%.  MG_SELL_PF=0: plain unrolled loop (A/B).
static bool sell_pf() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_SELL_PF");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

// rows longer than this (average) take the UNR = 8 SELL kernel (software pipelined
// with MG_SELL_PF) instead of UNR = 4; MG_SELL_LONG_AVG overrides (A/B)
static double sell_long_avg() {
  static const double v = [] {
    double v = -1.0;
    const char *e = getenv("MG_SELL_LONG_AVG");
    v = e ? atof(e) : 64.0;
    return v;
  }();
  return v;
}

static int csr_mid_variant() {
  static const int v = [] {
    int v = -1;
    const char *e = getenv("MG_CSR_MID");
    v = e ? atoi(e) : 0;
    return v;
  }();
  return v;
}
static int csr_long_variant() {
  static const int v = [] {
    int v = -1;
    const char *e = getenv("MG_CSR_LONG");
    v = e ? atoi(e) : 0;
    return v;
  }();
  return v;
}

template <class Epi, class XG = XPlain>
static void launch_csr(const Csr &a, XG x, Epi epi) {
  if (a.nr == 0) return;
  double avg = a.nr ? (double)a.nnz / a.nr : 0.0;
  prepare_spmv(a);
  const SpmvPlan &pl = *a.plan;
#define LAUNCH_AVG(VS, U)                                                                                    \
  do {                                                                                                       \
    if (pl.ik == 1)                                                                                          \
      launch_pdl(k_csr<VS, U, 1, Epi, XG>, spmv_grid((int64_t)a.nr * VS), 256, 0, a.nr, nullptr, a.rp.p,      \
                 (const void *)pl.scode.p, pl.dict.p, pl.mul, a.v.p, x, epi);                                \
    else if (pl.ik == 2)                                                                                     \
      launch_pdl(k_csr<VS, U, 2, Epi, XG>, spmv_grid((int64_t)a.nr * VS), 256, 0, a.nr, nullptr, a.rp.p,      \
                 (const void *)pl.scode.p, pl.dict.p, pl.mul, a.v.p, x, epi);                                \
    else                                                                                                     \
      launch_pdl(k_csr<VS, U, 0, Epi, XG>, spmv_grid((int64_t)a.nr * VS), 256, 0, a.nr, nullptr, a.rp.p,      \
                 (const void *)a.ci.p, (const int *)nullptr, 0ull, a.v.p, x, epi);                          \
  } while (0)
  if (pl.sell) {
    const void *ci = pl.ik ? (const void *)pl.scode.p : (const void *)pl.sci.p;
#define LAUNCH_SELL(UNR, T, IK)                                                                                \
  do {                                                                                                         \
    if (UNR == 8 && sell_pf())                                                                                 \
      launch_pdl(k_sell<UNR, IK, true, Epi, XG>, grid_for(a.nr, T), T, 0, a.nr, pl.sptr.p, pl.rlen.p,          \
                 (const int *)pl.perm.p, ci, pl.dict.p, pl.mul, pl.sv.p, x, epi);                              \
    else                                                                                                       \
      launch_pdl(k_sell<UNR, IK, false, Epi, XG>, grid_for(a.nr, T), T, 0, a.nr, pl.sptr.p, pl.rlen.p,         \
                 (const int *)pl.perm.p, ci, pl.dict.p, pl.mul, pl.sv.p, x, epi);                              \
  } while (0)
    if (pl.ik == 1 && !pl.perm.p && avg >= 24 && avg <= sell_long_avg() && sell_tma()) {
      const int vtma = sell_tma();
      if (vtma == 1)
        launch_pdl(k_sell_tma<Epi, 4, 4, 8>, grid_for(a.nr, 256), 256, 0, a.nr, pl.sptr.p, pl.rlen.p,
                   (const unsigned *)pl.scode.p, pl.dict.p, pl.mul, pl.sv.p, x, epi);
      else if (vtma == 2)
        launch_pdl(k_sell_tma<Epi, 3, 8, 4>, grid_for(a.nr, 128), 128, 0, a.nr, pl.sptr.p, pl.rlen.p,
                   (const unsigned *)pl.scode.p, pl.dict.p, pl.mul, pl.sv.p, x, epi);
      else
        launch_pdl(k_sell_tma<Epi, 2, 16, 4>, grid_for(a.nr, 128), 128, 0, a.nr, pl.sptr.p, pl.rlen.p,
                   (const unsigned *)pl.scode.p, pl.dict.p, pl.mul, pl.sv.p, x, epi);
      check_launch("sell tma spmv");
      return;
    }
    if (avg > sell_long_avg()) {
      if (pl.ik == 1) LAUNCH_SELL(8, 128, 1);
      else if (pl.ik == 2) LAUNCH_SELL(8, 128, 2);
      else LAUNCH_SELL(8, 128, 0);
    } else {
      if (pl.ik == 1) LAUNCH_SELL(4, 256, 1);
      else if (pl.ik == 2) LAUNCH_SELL(4, 256, 2);
      else LAUNCH_SELL(4, 256, 0);
    }
#undef LAUNCH_SELL
    check_launch("sell spmv");
    return;
  }
  // lane-group size from the average row length (measured better than per-class
  // row binning: the row-list indirection adds a dependent load)
  if (avg <= 2.5) LAUNCH_AVG(2, 2);
  else if (avg <= 5) LAUNCH_AVG(4, 2);
  else if (avg <= 9) LAUNCH_AVG(4, 3);
  else if (avg <= 18) LAUNCH_AVG(8, 3);
  // measured on the config-3 hierarchies (tools/kbench.py): 8 lanes x 2 for
  // ~26/row (F-relax A_1, 58 -> 68% of HBM), 8 x 4 for ~40-60/row, 16 x 4
  // for the ~100-150/row coarse-AMG levels (76 -> 84%)
  else if (avg <= 36) LAUNCH_AVG(8, 2);
  else if (avg <= 72) {
    switch (csr_mid_variant()) {  // MG_CSR_MID (A/B of the lane split for 37-72 per row)
      case 1: LAUNCH_AVG(16, 2); break;
      case 2: LAUNCH_AVG(16, 4); break;
      case 3: LAUNCH_AVG(8, 2); break;
      case 4: LAUNCH_AVG(4, 4); break;
      default: LAUNCH_AVG(8, 4);
    }
  }
  else {
    switch (csr_long_variant()) {  // MG_CSR_LONG (A/B of the lane split for > 72 per row)
      case 1: LAUNCH_AVG(16, 8); break;
      case 2: LAUNCH_AVG(32, 4); break;
      case 3: LAUNCH_AVG(32, 2); break;
      case 4: LAUNCH_AVG(8, 8); break;
      default: LAUNCH_AVG(16, 4);
    }
  }
#undef LAUNCH_AVG
  check_launch("csr spmv");
}

static bool bsell_enabled() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_BSELL");
    on = !(e && *e == '0');
    return on;
  }();
  return on;
}

void spmv(const Csr &a, const double *x, double *y) {
  if (a.b == 1) {
    launch_csr(a, XPlain{x}, EpiStore{y});
    return;
  }
  if (a.nr == 0) return;
  const int T = 256;
  double avg = (double)a.nnz / a.nr;
  cudaStream_t s = stream();
  (void)T;
  prepare_spmv(a);
  if (a.plan->sell && bsell_enabled()) {
    const SpmvPlan &pl = *a.plan;
    if (a.b == 2) launch_pdl(k_bsell<2, 4>, grid_for(a.nr, 256), 256, 0, a.nr, pl.sptr.p, pl.rlen.p, pl.sci.p, pl.sv.p, x, y);
    else launch_pdl(k_bsell<3, 2>, grid_for(a.nr, 256), 256, 0, a.nr, pl.sptr.p, pl.rlen.p, pl.sci.p, pl.sv.p, x, y);
    check_launch("bsell spmv");
    return;
  }
  if (a.b == 2) {
    if (avg <= 4.5) launch_pdl(k_bsr<2, 2, 3>, spmv_grid((int64_t)a.nr * 2), 256, 0, a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
    else launch_pdl(k_bsr<2, 4, 2>, spmv_grid((int64_t)a.nr * 4), 256, 0, a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
  } else if (a.b == 3) {
    if (avg <= 4.5) launch_pdl(k_bsr<3, 2, 3>, spmv_grid((int64_t)a.nr * 2), 256, 0, a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
    else launch_pdl(k_bsr<3, 4, 2>, spmv_grid((int64_t)a.nr * 4), 256, 0, a.nr, a.rp.p, a.ci.p, a.v.p, x, y);
  } else {
    throw MgError(MG_ERR_UNSUPPORTED, "block size must be 1, 2 or 3");
  }
  check_launch("bsr spmv");
}

void residual(const Csr &a, const double *x, const double *b, double *r) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "residual: scalar CSR only");
  launch_csr(a, XPlain{x}, EpiResid{b, r});
}

void spmv_merge_add(const Csr &a, const double *x, const int *fmap, const double *ef, double *y) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "spmv_merge_add: scalar CSR only");
  launch_csr(a, XPlain{x}, EpiMergeAdd{fmap, ef, y});
}

void spmv_add(const Csr &a, const double *x, double *y) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "spmv_add: scalar CSR only");
  launch_csr(a, XPlain{x}, EpiAdd{y});
}

void spmv_store_scale(const Csr &a, const double *x, double *y, const double *sign, double *bs, const double *d,
                      double *xo) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "spmv_store_scale: scalar CSR only");
  launch_csr(a, XPlain{x}, EpiStoreScale{y, sign, bs, d, xo});
}

void residual_rows_scale(const Csr &a, const double *x, const double *b, const int *rows, double *y,
                         const double *sign, double *bs, const double *d, double *xo) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "residual_rows_scale: scalar CSR only");
  launch_csr(a, XPlain{x}, EpiResidRowsScale{b, rows, y, sign, bs, d, xo});
}

void jacobi_sweep(const Csr &a, const double *x, const double *b, const double *dinv, double *xo) {
  launch_csr(a, XPlain{x}, EpiJacobi{x, b, dinv, xo});
}

}  // namespace mg
