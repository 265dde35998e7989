// AMG setup kernels: row-sign normalisation, strength of connection, PMIS
// coarsening, extended+i interpolation (optional max_elmts truncation) and
// L1 row norms.
//
// Reference counterparts: strength_graph
// (amg.py:88-103, same definition), rs_splitting (amg.py:106-158, replaced by
// PMIS), classical_interpolation (amg.py:206-276, replaced by extended+i),
// Gauss-Seidel handles (amg.py:279-286, replaced by L1-Jacobi).  The
// operation order of every floating-point result is the one pinned in
// oracle/csrc/amg_oracle.c, so C/F splittings, P patterns and P values are
// bit-identical to the oracle (the file is compiled with --fmad=false and uses
// explicit __d*_rn intrinsics on the pinned sequences).
#include "ops.cuh"
#include "hash.cuh"
#include "amg_kernels.cuh"

namespace mg {

enum { UNDEC = 0, FPT = 1, CPT = 2 };

// ---- diagonal ----------------------------------------------------------------
template <int VS>
__global__ void k_row_diag(int n, const int *rp, const int *ci, const double *v, double *d) {
  for (RowGroup<VS> g; g.row < n; g.next()) {
    const int r = (int)g.row;
    int found = -1;
    for (int q = rp[r] + g.lane; q < rp[r + 1]; q += VS)
      if (ci[q] == r) found = q;
    unsigned bal = g.ballot(found >= 0);
    double val = 0.0;
    if (bal) {
      int q = g.bcast(found, __ffs(bal) - 1);
      val = __dadd_rn(0.0, v[q]);
    }
    if (g.lane == 0) d[r] = val;
  }
}

void row_diag(const Csr &a, double *d) {
  if (!a.nr) return;
  MG_ROWGROUP_LAUNCH(k_row_diag, a.nr, a.nnz, a.nr, a.rp.p, a.ci.p, a.v.p, d);
  check_launch("row_diag");
}

// ---- row-sign normalisation (amg.py:296-301; diags @ csr drops exact zeros) ----
__global__ void k_sign_count(int n, const int *rp, const double *v, const double *sgn, int *cnt) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  int c = 0;
  for (int q = rp[wid] + lane; q < rp[wid + 1]; q += 32) c += __dmul_rn(sgn[wid], v[q]) != 0.0;
  for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
  if (lane == 0) cnt[wid] = c;
}
__global__ void k_sign_fill(int n, const int *rp, const int *ci, const double *v, const double *sgn,
                            const int *orp, int *oci, double *ov) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= n) return;
  int o = orp[wid];
  for (int q0 = rp[wid]; q0 < rp[wid + 1]; q0 += 32) {
    int q = q0 + lane;
    double val = q < rp[wid + 1] ? __dmul_rn(sgn[wid], v[q]) : 0.0;
    bool keep = q < rp[wid + 1] && val != 0.0;
    unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      int p = o + __popc(bal & ((1u << lane) - 1));
      oci[p] = ci[q];
      ov[p] = val;
    }
    o += __popc(bal);
  }
}
__global__ void k_sign_of_diag(int n, const double *d, double *sgn, int *flags) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double di = d[i];
  if (di == 0.0) atomicMin(&flags[0], i);
  if (di < 0.0) atomicExch(&flags[1], 1);
  sgn[i] = di < 0.0 ? -1.0 : 1.0;
}

// returns false when no row needed flipping (out untouched)
bool sign_normalise(const Csr &a, Csr &out, DBuf<double> &sgn) {
  int n = a.nr;
  DBuf<double> d(n);
  row_diag(a, d.p);
  sgn.alloc(n);
  DBuf<int> flags(2);
  dset_i32(flags.p, {0x7fffffff, 0});
  if (n) {
    k_sign_of_diag<<<grid_for(n, 256), 256, 0, stream()>>>(n, d.p, sgn.p, flags.p);
    check_launch("sign_of_diag");
  }
  int hf[2];
  d2h(hf, flags.p, sizeof(hf));
  if (hf[0] != 0x7fffffff) throw MgError(MG_ERR_AMG_SETUP, "AMG expects a nonzero diagonal", hf[0]);
  if (!hf[1]) { sgn.release(); return false; }
  out.nr = n;
  out.nc = a.nc;
  out.b = 1;
  out.rp.alloc((size_t)n + 1);
  DBuf<int> cnt(n);
  k_sign_count<<<grid_for((int64_t)n * 32, 256), 256, 0, stream()>>>(n, a.rp.p, a.v.p, sgn.p, cnt.p);
  check_launch("sign_count");
  out.nnz = exclusive_scan_i32_to_i32(cnt.p, out.rp.p, n);
  out.ci.alloc((size_t)out.nnz);
  out.v.alloc((size_t)out.nnz);
  k_sign_fill<<<grid_for((int64_t)n * 32, 256), 256, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, sgn.p, out.rp.p,
                                                                     out.ci.p, out.v.p);
  check_launch("sign_fill");
  return true;
}

// ---- strength of connection (amg.py:88-103) ------------------------------------
template <int VS>
__global__ void k_strength(int n, const int *rp, const int *ci, const double *v, double theta, int8_t *s,
                           int *any) {
  for (RowGroup<VS> g; g.row < n; g.next()) {
    const int r = (int)g.row;
    int b = rp[r], e = rp[r + 1];
    if (e - b <= 2 * VS) {
      // rows of up to 2 VS entries: one load of the row into registers (the
      // three-pass loop below re-walks it with dependent loads); same results
      const int q0 = b + g.lane, q1 = q0 + VS;
      const bool in0 = q0 < e, in1 = q1 < e;
      const int c0 = in0 ? __ldg(ci + q0) : r, c1 = in1 ? __ldg(ci + q1) : r;
      const double a0 = in0 ? __ldg(v + q0) : 0.0, a1 = in1 ? __ldg(v + q1) : 0.0;
      const bool off0 = c0 != r, off1 = c1 != r;
      const bool has_neg = g.any((off0 && a0 < 0.0) || (off1 && a1 < 0.0));
      const double cand0 = (off0 && a0 < 0.0) ? -a0 : ((off0 && !has_neg) ? fabs(a0) : 0.0);
      const double cand1 = (off1 && a1 < 0.0) ? -a1 : ((off1 && !has_neg) ? fabs(a1) : 0.0);
      const double rmax = g.max(fmax(fmax(0.0, cand0), cand1));
      const double thr = __dmul_rn(theta, rmax);
      const int8_t st0 = (rmax > 0.0 && cand0 >= thr) ? 1 : 0, st1 = (rmax > 0.0 && cand1 >= thr) ? 1 : 0;
      if (in0) s[q0] = st0;
      if (in1) s[q1] = st1;
      const bool has = g.any((in0 && st0) || (in1 && st1));
      if (g.lane == 0 && has && *(volatile int *)any == 0) atomicExch(any, 1);
      continue;
    }
    bool neg = false;
    for (int q = b + g.lane; q < e; q += VS) neg |= (ci[q] != r) && (v[q] < 0.0);
    bool has_neg = g.any(neg);
    double rmax = 0.0;
    for (int q = b + g.lane; q < e; q += VS) {
      bool off = ci[q] != r;
      double a = v[q];
      double cand = (off && a < 0.0) ? -a : ((off && !has_neg) ? fabs(a) : 0.0);
      rmax = fmax(rmax, cand);
    }
    rmax = g.max(rmax);
    double thr = __dmul_rn(theta, rmax);
    int cnt = 0;
    for (int q = b + g.lane; q < e; q += VS) {
      bool off = ci[q] != r;
      double a = v[q];
      double cand = (off && a < 0.0) ? -a : ((off && !has_neg) ? fabs(a) : 0.0);
      int8_t st = (rmax > 0.0 && cand >= thr) ? 1 : 0;
      s[q] = st;
      cnt |= st;
    }
    // only "some strong edge exists" is consumed: one atomic the first time a
    // group sees an unset flag (a counter hit by every row serialised the kernel)
    bool has = g.any(cnt != 0);
    if (g.lane == 0 && has && *(volatile int *)any == 0) atomicExch(any, 1);
  }
}

int64_t strength(const Csr &a, double theta, DBuf<int8_t> &s) {
  s.alloc((size_t)(a.nnz ? a.nnz : 1));
  DBuf<int> any(1);
  dzero(any.p, sizeof(int));
  if (a.nr) {
    MG_ROWGROUP_LAUNCH(k_strength, a.nr, a.nnz, a.nr, a.rp.p, a.ci.p, a.v.p, theta, s.p, any.p);
    check_launch("strength");
  }
  int h = 0;
  d2h(&h, any.p, sizeof(int));
  return h;
}

// ---- PMIS ---------------------------------------------------------------------
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ULL;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  return z ^ (z >> 31);
}

template <int VS>
__global__ void k_st_count(int n, const int *rp, const int *ci, const int8_t *s, int *cnt) {
  for (RowGroup<VS> g; g.row < n; g.next()) {
    const int r = (int)g.row;
    for (int q = rp[r] + g.lane; q < rp[r + 1]; q += VS)
      if (s[q] && ci[q] != r) atomicAdd(&cnt[ci[q]], 1);
  }
}
__global__ void k_pmis_init(int n, const int *tcnt, uint64_t seed, int level, double *mu, int8_t *state,
                            int *undecided) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int st = tcnt[i];
  uint64_t x = seed ^ ((uint64_t)(uint32_t)level * 0x9E3779B97F4A7C15ULL) ^ (uint64_t)(int64_t)i;
  double u = __dmul_rn((double)(splitmix64(x) >> 11), 1.0 / 9007199254740992.0);
  mu[i] = __dadd_rn((double)st, u);
  state[i] = st == 0 ? FPT : UNDEC;
  if (st && *(volatile int *)undecided == 0) atomicExch(undecided, 1);  // only "any" is consumed
}
__device__ __forceinline__ bool beats(double mi, int i, double mj, int j) {
  return mi > mj || (mi == mj && i > j);
}
// One synchronous PMIS round without an explicit S^T.  The C test "mu_i beats
// every undecided j in S_i u S^T_i" is evaluated by pushing over S only: the row
// walk of i compares each undecided strong pair (i, j), j in S_i, and stamps the
// loser (mark[loser] = round).  Every pair of S u S^T is some row's S entry, so
// after the walk an undecided i is unstamped iff it beats all of them -- the same
// set the pull formulation (S_i and S^T_i walks) selects.  Stamps of equal value
// from several rows are benign writes; the round number makes a reset pass
// unnecessary.
template <int VS>
__global__ void k_pmis_mark(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                            const int8_t *__restrict__ s, const double *__restrict__ mu,
                            const int8_t *__restrict__ state, int *mark, int stamp) {
  for (RowGroup<VS> g; g.row < n; g.next()) {
    const int i = (int)g.row;
    if (state[i] != UNDEC) continue;
    const double mi = mu[i];
    bool lost = false;
    for (int q = rp[i] + g.lane; q < rp[i + 1]; q += VS) {
      const int j = ci[q];
      MG_DCHECK(j >= 0 && j < n);
      if (!s[q] || j == i || state[j] != UNDEC) continue;
      if (beats(mu[j], j, mi, i)) lost = true;
      else mark[j] = stamp;
    }
    if (g.any(lost) && g.lane == 0) mark[i] = stamp;
  }
}
// i (undecided): unstamped -> C; else F if some strong j in S_i is C (old, or new
// this round).  The new C set is read on the fly: k is new C iff it was undecided
// and unstamped; a k already rewritten by its own row this round reads CPT (new C)
// or FPT (new F, never new C), so every interleaving gives the same answer.
template <int VS>
__global__ void k_pmis_update2(int n, const int *__restrict__ rp, const int *__restrict__ ci,
                               const int8_t *__restrict__ s, const int *__restrict__ mark, int stamp,
                               int8_t *state, int *undecided) {
  for (RowGroup<VS> g; g.row < n; g.next()) {
    const int i = (int)g.row;
    if (state[i] != UNDEC) continue;
    if (mark[i] != stamp) {
      if (g.lane == 0) state[i] = CPT;
      continue;
    }
    bool f = false;
    for (int q = rp[i] + g.lane; q < rp[i + 1] && !f; q += VS) {
      const int k = ci[q];
      MG_DCHECK(k >= 0 && k < n);
      if (!s[q] || k == i) continue;
      const int8_t sk = ((volatile const int8_t *)state)[k];
      f = sk == CPT || (sk == UNDEC && mark[k] != stamp);
    }
    if (g.any(f)) {
      if (g.lane == 0) state[i] = FPT;
    } else if (g.lane == 0 && *(volatile int *)undecided == 0) {
      atomicExch(undecided, 1);
    }
  }
}

int pmis(const Csr &a, const int8_t *s, uint64_t seed, int level, DBuf<int8_t> &state) {
  int n = a.nr;
  state.alloc((size_t)(n ? n : 1));
  if (!n) return 0;
  // |S^T_i| (column counts of S) for the measure; no S^T itself
  DBuf<int> tcnt((size_t)n + 1);
  dzero(tcnt.p, sizeof(int) * ((size_t)n + 1));
  MG_ROWGROUP_LAUNCH(k_st_count, n, a.nnz, n, a.rp.p, a.ci.p, s, tcnt.p);
  check_launch("st_count");
  DBuf<double> mu(n);
  DBuf<int> mark(n), und(1);
  MG_CUDA(cudaMemsetAsync(mark.p, 0, sizeof(int) * (size_t)n, stream()));
  dzero(und.p, sizeof(int));
  k_pmis_init<<<grid_for(n, 256), 256, 0, stream()>>>(n, tcnt.p, seed, level, mu.p, state.p, und.p);
  check_launch("pmis_init");
  // rounds are checked for termination in pairs (a round with nothing
  // undecided is a no-op), halving the host round trips
  int hu = 1;
  int rounds = 0;
  while (hu > 0) {
    for (int pair = 0; pair < 2; ++pair) {
      ++rounds;
      MG_ROWGROUP_LAUNCH(k_pmis_mark, n, a.nnz, n, a.rp.p, a.ci.p, s, mu.p, state.p, mark.p, rounds);
      check_launch("pmis_mark");
      dzero(und.p, sizeof(int));
      MG_ROWGROUP_LAUNCH(k_pmis_update2, n, a.nnz, n, a.rp.p, a.ci.p, s, mark.p, rounds, state.p, und.p);
      check_launch("pmis_update");
    }
    d2h(&hu, und.p, sizeof(int));
    if (rounds > 100000) throw MgError(MG_ERR_AMG_SETUP, "PMIS did not terminate");
  }
  return rounds;
}

// ---- extended+i interpolation ----------------------------------------------------
// Pinned warp tree sum (oracle tree32): w = v; for off in 16,8,4,2,1: w[l] += w[l+off];
// result = w[0], broadcast to every lane.
__device__ __forceinline__ double warp_tree(double v) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v = __dadd_rn(v, __shfl_down_sync(0xffffffffu, v, off));
  return __shfl_sync(0xffffffffu, v, 0);
}

__device__ __forceinline__ bool opposite(double v, double dkk) {
  return (v < 0.0 && dkk > 0.0) || (v > 0.0 && dkk < 0.0);
}

// candidate bound per row: C rows 1; F rows: strong C + sum_{strong F k} |row k|
template <int VS>
__global__ void k_ext_ub(int n, const int *rp, const int *ci, const int8_t *s, const int8_t *state, int *ub) {
  for (RowGroup<VS> g; g.row < n; g.next()) {
    const int r = (int)g.row;
    int64_t c = 0;
    if (state[r] != CPT)
      for (int q = rp[r] + g.lane; q < rp[r + 1]; q += VS) {
        int j = ci[q];
        if (j == r || !s[q]) continue;
        c += state[j] == FPT ? (rp[j + 1] - rp[j]) : 1;
      }
    c = g.sum(c);
    if (g.lane == 0) ub[r] = c > 0x3fffffff ? 0x3fffffff : (int)c;
  }
}

struct ExtArgs {
  const int *rp, *ci;
  const double *v;
  const int8_t *s, *state;
  const int *cmap;
  int max_elmts;
  int mode;
  int *cnt;
  const int *prp;
  int *pci;
  double *pv;
  int *bad;
};

// insert Chat_i = C^s_i u (C^s_k for strong-F k) into keys (initialised to -1);
// returns |Chat_i| on every lane.  Lanes own consecutive entries of row i; the
// strong-F neighbours k of a 32-entry chunk are found with one ballot and the
// whole warp walks each row k (coalesced 32-entry chunks).
__device__ __forceinline__ int ext_candidates(int i, int *keys, unsigned mask, int lane, const ExtArgs &A) {
  const int *rp = A.rp, *ci = A.ci;
  const int8_t *s = A.s, *state = A.state;
  int b = rp[i], e = rp[i + 1];
  int mine = 0;
  for (int q0 = b; q0 < e; q0 += 32) {
    int q = q0 + lane;
    int kk = -1, kb_l = 0, ke_l = 0;
    if (q < e) {
      int j = ci[q];
      if (j != i && s[q]) {
        int sj = state[j];
        if (sj == CPT) {
          mine += hash_insert(keys, mask, j);
        } else if (sj == FPT) {
          kk = j;
          kb_l = rp[j];
          ke_l = rp[j + 1];
        }
      }
    }
    unsigned km = __ballot_sync(0xffffffffu, kk >= 0);
    while (km) {
      int src = __ffs(km) - 1;
      km &= km - 1;
      int k = __shfl_sync(0xffffffffu, kk, src);
      int kb = __shfl_sync(0xffffffffu, kb_l, src), ke = __shfl_sync(0xffffffffu, ke_l, src);
      for (int q2 = kb + lane; q2 < ke; q2 += 32) {
        int l = ci[q2];
        if (l != k && s[q2] && state[l] == CPT) mine += hash_insert(keys, mask, l);
      }
    }
  }
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  __syncwarp();
  return mine;
}

__device__ void ext_row(int i, int T, WarpTables t, int lane, const ExtArgs &A) {
  const int *rp = A.rp, *ci = A.ci;
  const double *v = A.v;
  const int8_t *s = A.s, *state = A.state;
  if (state[i] == CPT) {
    if (lane == 0) {
      if (A.mode == 0) A.cnt[i] = 1;
      else { A.pci[A.prp[i]] = A.cmap[i]; A.pv[A.prp[i]] = 1.0; }
    }
    return;
  }
  unsigned mask = (unsigned)T - 1;
  table_clear(t, T, lane);
  int b = rp[i], e = rp[i + 1];
  int u = ext_candidates(i, t.keys, mask, lane, A);
  int outlen = (A.max_elmts > 0 && u > A.max_elmts) ? A.max_elmts : u;
  if (A.mode == 0) {
    if (lane == 0) A.cnt[i] = outlen;
    return;
  }
  if (u == 0) return;
  table_sort(t, T, u, lane);
  double *num = t.acc;
  for (int q = lane; q < u; q += 32) num[q] = 0.0;
  __syncwarp();
  // direct numerators a_ij, j in Chat (distinct j: lane parallel)
  for (int q = b + lane; q < e; q += 32) {
    int j = ci[q];
    if (j == i) continue;
    int sl = hash_find_opt(t.keys, mask, j);
    if (sl >= 0) { int p = t.pos[sl]; num[p] = __dadd_rn(num[p], v[q]); }
  }
  __syncwarp();
  // dt = a_ii + TREE(weak lumps of row i): lanes classify, pinned warp tree
  double dt;
  {
    int found = -1;
    double lump = 0.0;
    for (int q0 = b; q0 < e; q0 += 32) {
      int q = q0 + lane;
      double term = 0.0;
      if (q < e) {
        int j = ci[q];
        if (j == i) found = q;
        else if (hash_find_opt(t.keys, mask, j) < 0 && !(s[q] && state[j] == FPT)) term = v[q];
      }
      lump = __dadd_rn(lump, warp_tree(term));
    }
    unsigned bal = __ballot_sync(0xffffffffu, found >= 0);
    double aii = bal ? __dadd_rn(0.0, v[__shfl_sync(0xffffffffu, found, __ffs(bal) - 1)]) : 0.0;
    dt = __dadd_rn(aii, lump);
  }
  // distribution through strong F neighbours k, in row-i order.  The strong-F
  // entries of a 32-entry chunk of row i are found with one ballot (their row
  // ranges prefetched by their own lanes); a row k of <= 64 entries is held in
  // registers (two entries per lane) for a_kk, beta_k, the numerators and the
  // a_ki term, so each k costs a single round trip to memory.
  for (int q0 = b; q0 < e; q0 += 32) {
    int qq = q0 + lane;
    int kk = -1, kb_l = 0, ke_l = 0;
    double aik_l = 0.0;
    if (qq < e) {
      int j = ci[qq];
      if (j != i && s[qq] && state[j] == FPT) {
        kk = j;
        aik_l = v[qq];
        kb_l = rp[j];
        ke_l = rp[j + 1];
      }
    }
    unsigned kmask = __ballot_sync(0xffffffffu, kk >= 0);
    while (kmask) {
      int src = __ffs(kmask) - 1;
      kmask &= kmask - 1;
      int k = __shfl_sync(0xffffffffu, kk, src);
      double aik = __shfl_sync(0xffffffffu, aik_l, src);
      int kb = __shfl_sync(0xffffffffu, kb_l, src), ke = __shfl_sync(0xffffffffu, ke_l, src);
      int len = ke - kb;
      if (len <= 64) {
        int l0 = -1, l1 = -1;
        double v0 = 0.0, v1 = 0.0;
        if (lane < len) { l0 = ci[kb + lane]; v0 = v[kb + lane]; }
        if (lane + 32 < len) { l1 = ci[kb + 32 + lane]; v1 = v[kb + 32 + lane]; }
        unsigned db = __ballot_sync(0xffffffffu, l0 == k || l1 == k);
        double dv = l0 == k ? v0 : v1;
        double akk = db ? __dadd_rn(0.0, __shfl_sync(0xffffffffu, dv, __ffs(db) - 1)) : 0.0;
        bool o0 = l0 >= 0 && l0 != k && opposite(v0, akk);
        bool o1 = l1 >= 0 && l1 != k && opposite(v1, akk);
        int s0 = o0 && l0 != i ? hash_find_opt(t.keys, mask, l0) : -1;
        int s1 = o1 && l1 != i ? hash_find_opt(t.keys, mask, l1) : -1;
        double beta = __dadd_rn(0.0, warp_tree(o0 && (l0 == i || s0 >= 0) ? v0 : 0.0));
        if (len > 32) beta = __dadd_rn(beta, warp_tree(o1 && (l1 == i || s1 >= 0) ? v1 : 0.0));
        if (beta == 0.0) {
          dt = __dadd_rn(dt, aik);
          continue;
        }
        double f = __ddiv_rn(aik, beta);
        if (s0 >= 0) { int p = t.pos[s0]; num[p] = __dadd_rn(num[p], __dmul_rn(f, v0)); }
        if (s1 >= 0) { int p = t.pos[s1]; num[p] = __dadd_rn(num[p], __dmul_rn(f, v1)); }
        unsigned bi = __ballot_sync(0xffffffffu, (o0 && l0 == i) || (o1 && l1 == i));
        if (bi) {
          double iv = (o0 && l0 == i) ? v0 : v1;
          dt = __dadd_rn(dt, __dmul_rn(f, __shfl_sync(0xffffffffu, iv, __ffs(bi) - 1)));
        }
        __syncwarp();
        continue;
      }
      // long rows: chunked reloads
      int found = -1;
      for (int q2 = kb + lane; q2 < ke; q2 += 32)
        if (ci[q2] == k) found = q2;
      unsigned bal = __ballot_sync(0xffffffffu, found >= 0);
      double akk = bal ? __dadd_rn(0.0, v[__shfl_sync(0xffffffffu, found, __ffs(bal) - 1)]) : 0.0;
    // beta = TREE over row k of abar_kl for l in Chat u {i}
    double beta = 0.0;
    int at_i = -1;
    for (int c0 = kb; c0 < ke; c0 += 32) {
      int q2 = c0 + lane;
      double term = 0.0;
      if (q2 < ke) {
        int l = ci[q2];
        double val = v[q2];
        if (l != k && opposite(val, akk)) {
          if (l == i) { term = val; at_i = q2; }
          else if (hash_find_opt(t.keys, mask, l) >= 0) term = val;
        }
      }
      beta = __dadd_rn(beta, warp_tree(term));
    }
    if (beta == 0.0) {
      dt = __dadd_rn(dt, aik);
      continue;
    }
    double f = __ddiv_rn(aik, beta);
    for (int q2 = kb + lane; q2 < ke; q2 += 32) {
      int l = ci[q2];
      if (l == k) continue;
      double val = v[q2];
      if (!opposite(val, akk)) continue;
      int sl = hash_find_opt(t.keys, mask, l);
      if (sl >= 0) { int p = t.pos[sl]; num[p] = __dadd_rn(num[p], __dmul_rn(f, val)); }
    }
    unsigned bi = __ballot_sync(0xffffffffu, at_i >= 0);
    if (bi) dt = __dadd_rn(dt, __dmul_rn(f, v[__shfl_sync(0xffffffffu, at_i, __ffs(bi) - 1)]));
    __syncwarp();
    }
  }
  if (dt == 0.0) {
    if (lane == 0) atomicMin(A.bad, i);
    return;
  }
  for (int q = lane; q < u; q += 32) num[q] = __ddiv_rn(-num[q], dt);
  __syncwarp();
  int o = A.prp[i];
  if (outlen == u) {
    for (int q = lane; q < u; q += 32) {
      A.pci[o + q] = A.cmap[t.list[q]];
      A.pv[o + q] = num[q];
    }
    return;
  }
  // truncation: keep the max_elmts largest |w| (ties: smaller column), rescale
  int *flag = t.pos;  // pos no longer needed
  for (int q = lane; q < u; q += 32) flag[q] = 0;
  __syncwarp();
  for (int r = 0; r < outlen; ++r) {
    double bw = -1.0;
    int bq = 0x7fffffff;
    for (int q = lane; q < u; q += 32) {
      if (flag[q]) continue;
      double aw = fabs(num[q]);
      if (aw > bw || (aw == bw && q < bq)) { bw = aw; bq = q; }
    }
    for (int o2 = 16; o2 > 0; o2 >>= 1) {
      double ow = __shfl_xor_sync(0xffffffffu, bw, o2);
      int oq = __shfl_xor_sync(0xffffffffu, bq, o2);
      if (ow > bw || (ow == bw && oq < bq)) { bw = ow; bq = oq; }
    }
    if (lane == 0 && bq < u) flag[bq] = 1;
    __syncwarp();
  }
  double s_all = 0.0, s_kept = 0.0;
  for (int q0 = 0; q0 < u; q0 += 32) {
    int q = q0 + lane;
    double w_q = q < u ? num[q] : 0.0;
    s_all = __dadd_rn(s_all, warp_tree(w_q));
    s_kept = __dadd_rn(s_kept, warp_tree(q < u && flag[q] ? w_q : 0.0));
  }
  if (lane == 0) {
    double scale = s_kept != 0.0 ? __ddiv_rn(s_all, s_kept) : 1.0;
    int w = 0;
    for (int q = 0; q < u; ++q)
      if (flag[q]) {
        A.pci[o + w] = A.cmap[t.list[q]];
        A.pv[o + w] = __dmul_rn(num[q], scale);
        ++w;
      }
  }
}

template <int T, int WPB>
__global__ void __launch_bounds__(WPB * 32, 2048 / (WPB * 32)) k_ext_smem(int nrows, const int *rows, ExtArgs A) {
  extern __shared__ __align__(16) unsigned char smem[];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  WarpTables t = carve(smem + table_bytes(T, false) * wid, T, false);
  for (int r = blockIdx.x * WPB + wid; r < nrows; r += gridDim.x * WPB) ext_row(rows[r], T, t, lane, A);
}
__global__ void k_ext_gmem(int nrows, const int *rows, const int64_t *goff, const int *gsize,
                           unsigned char *pool, ExtArgs A) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= nrows) return;
  int T = gsize[wid];
  ext_row(rows[wid], T, carve(pool + goff[wid], T, false), lane, A);
}

template <int T, int WPB>
static void launch_ext(int nrows, const int *rows, const ExtArgs &A) {
  if (!nrows) return;
  size_t sm = table_bytes(T, false) * WPB;
  MG_CUDA(cudaFuncSetAttribute(k_ext_smem<T, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  int grid = (nrows + WPB - 1) / WPB;
  int cap = g_ctx->num_sms * 16;
  if (grid > cap) grid = cap;
  k_ext_smem<T, WPB><<<grid, WPB * 32, sm, stream()>>>(nrows, rows, A);
  check_launch("ext_interp");
}

__global__ void k_cflags(int n, const int8_t *state, int *flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flag[i] = state[i] == CPT;
}
__global__ void k_cmap_from_scan(int n, const int8_t *state, const int *scan, int *cmap) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) cmap[i] = state[i] == CPT ? scan[i] : -1;
}

int coarse_map(const int8_t *state, int n, DBuf<int> &cmap) {
  DBuf<int> flag((size_t)(n ? n : 1)), scan((size_t)n + 1);
  cmap.alloc((size_t)(n ? n : 1));
  if (n) {
    k_cflags<<<grid_for(n, 256), 256, 0, stream()>>>(n, state, flag.p);
    check_launch("cflags");
  }
  int nc = (int)exclusive_scan_i32_to_i32(flag.p, scan.p, n);
  if (n) {
    k_cmap_from_scan<<<grid_for(n, 256), 256, 0, stream()>>>(n, state, scan.p, cmap.p);
    check_launch("cmap");
  }
  return nc;
}

// count pass: distinct interpolatory candidates u_i (keys-only tables, high
// occupancy); cnt = output row length (1 for C rows, min(u, max_elmts) else)
template <int T, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_ext_count(int nrows, const int *rows, ExtArgs A, int *ucnt) {
  __shared__ int skeys[WPB][T];
  int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int *keys = skeys[wid];
  for (int r = blockIdx.x * WPB + wid; r < nrows; r += gridDim.x * WPB) {
    int i = rows[r];
    if (A.state[i] == CPT) {
      if (lane == 0) { A.cnt[i] = 1; ucnt[i] = 0; }
      continue;
    }
    for (int q = lane; q < T; q += 32) keys[q] = -1;
    __syncwarp();
    int u = ext_candidates(i, keys, (unsigned)T - 1, lane, A);
    if (lane == 0) {
      ucnt[i] = u;
      A.cnt[i] = (A.max_elmts > 0 && u > A.max_elmts) ? A.max_elmts : u;
    }
    __syncwarp();
  }
}
__global__ void k_ext_count_g(int nrows, const int *rows, const int64_t *goff, const int *gsize,
                              unsigned char *pool, ExtArgs A, int *ucnt) {
  int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (wid >= nrows) return;
  int i = rows[wid];
  if (A.state[i] == CPT) {
    if (lane == 0) { A.cnt[i] = 1; ucnt[i] = 0; }
    return;
  }
  int T = gsize[wid];
  int *keys = (int *)(pool + goff[wid]);
  for (int q = lane; q < T; q += 32) keys[q] = -1;
  __syncwarp();
  int u = ext_candidates(i, keys, (unsigned)T - 1, lane, A);
  if (lane == 0) {
    ucnt[i] = u;
    A.cnt[i] = (A.max_elmts > 0 && u > A.max_elmts) ? A.max_elmts : u;
  }
}

template <int T, int WPB>
static void launch_ext_count(int nrows, const int *rows, const ExtArgs &A, int *ucnt) {
  if (!nrows) return;
  int grid = (nrows + WPB - 1) / WPB;
  int cap = g_ctx->num_sms * 32;
  if (grid > cap) grid = cap;
  k_ext_count<T, WPB><<<grid, WPB * 32, 0, stream()>>>(nrows, rows, A, ucnt);
  check_launch("ext_count");
}

Csr ext_interp(const Csr &a, const int8_t *s, const int8_t *state, const int *cmap, int nc, int max_elmts) {
  int n = a.nr;
  Csr p;
  p.nr = n;
  p.nc = nc;
  p.b = 1;
  p.rp.alloc((size_t)n + 1);
  DBuf<int> ub((size_t)(n ? n : 1)), cnt((size_t)(n ? n : 1)), ucnt((size_t)(n ? n : 1)), bad(1);
  const int big = 0x7fffffff;
  dset_i32(bad.p, {big});
  if (n) {
    MG_ROWGROUP_LAUNCH(k_ext_ub, n, a.nnz, n, a.rp.p, a.ci.p, s, state, ub.p);
    check_launch("ext_ub");
  }
  ExtArgs A{a.rp.p, a.ci.p, a.v.p, s, state, cmap, max_elmts, 0, cnt.p, nullptr, nullptr, nullptr, bad.p};
  {
    RowBins cb;
    cb.build(ub.p, n, 1);
    launch_ext_count<64, 8>(cb.cnt[0], cb.rows.p + cb.off[0], A, ucnt.p);
    launch_ext_count<128, 8>(cb.cnt[1], cb.rows.p + cb.off[1], A, ucnt.p);
    launch_ext_count<256, 8>(cb.cnt[2], cb.rows.p + cb.off[2], A, ucnt.p);
    launch_ext_count<512, 8>(cb.cnt[3], cb.rows.p + cb.off[3], A, ucnt.p);
    launch_ext_count<1024, 8>(cb.cnt[4], cb.rows.p + cb.off[4], A, ucnt.p);
    launch_ext_count<2048, 4>(cb.cnt[5], cb.rows.p + cb.off[5], A, ucnt.p);
    launch_ext_count<4096, 2>(cb.cnt[6], cb.rows.p + cb.off[6], A, ucnt.p);
    int ng = cb.cnt[NBIN];
    if (ng) {
      k_ext_count_g<<<grid_for((int64_t)ng * 32, 128), 128, 0, stream()>>>(ng, cb.rows.p + cb.off[NBIN], cb.goff.p,
                                                                            cb.gsize.p, cb.pool.p, A, ucnt.p);
      check_launch("ext_count_g");
    }
  }
  RowBins bins;
  bins.build(ucnt.p, n, 0);
  auto run = [&]() {
    launch_ext<64, 8>(bins.cnt[0], bins.rows.p + bins.off[0], A);
    launch_ext<128, 8>(bins.cnt[1], bins.rows.p + bins.off[1], A);
    launch_ext<256, 8>(bins.cnt[2], bins.rows.p + bins.off[2], A);
    launch_ext<512, 8>(bins.cnt[3], bins.rows.p + bins.off[3], A);
    launch_ext<1024, 8>(bins.cnt[4], bins.rows.p + bins.off[4], A);
    launch_ext<2048, 4>(bins.cnt[5], bins.rows.p + bins.off[5], A);
    launch_ext<4096, 2>(bins.cnt[6], bins.rows.p + bins.off[6], A);
    int ng = bins.cnt[NBIN];
    if (ng) {
      k_ext_gmem<<<grid_for((int64_t)ng * 32, 128), 128, 0, stream()>>>(ng, bins.rows.p + bins.off[NBIN],
                                                                         bins.goff.p, bins.gsize.p,
                                                                         bins.pool.p, A);
      check_launch("ext_gmem");
    }
  };
  p.nnz = exclusive_scan_i32_to_i32(cnt.p, p.rp.p, n);
  p.ci.alloc((size_t)p.nnz);
  p.v.alloc((size_t)p.nnz);
  A.mode = 1;
  A.prp = p.rp.p;
  A.pci = p.ci.p;
  A.pv = p.v.p;
  run();
  int hb = 0;
  d2h(&hb, bad.p, sizeof(int));
  if (hb != big)
    throw MgError(MG_ERR_AMG_SETUP, "extended interpolation hit a zero pivot at row " + std::to_string(hb), hb);
  return p;
}

// ---- L1 row norms: d_i = sum_j |a_ij| (sequential per row), dinv = 1/d --------
__global__ void k_l1inv(int n, const int *rp, const double *v, double *dinv) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (int q = rp[i]; q < rp[i + 1]; ++q) d = __dadd_rn(d, fabs(v[q]));
  dinv[i] = __ddiv_rn(1.0, d);
}
void l1_inverse(const Csr &a, double *dinv) {
  if (!a.nr) return;
  k_l1inv<<<grid_for(a.nr, 128), 128, 0, stream()>>>(a.nr, a.rp.p, a.v.p, dinv);
  check_launch("l1inv");
}

// ---- dense copy of a (small) CSR ----------------------------------------------
__global__ void k_to_dense(int n, int nc, const int *rp, const int *ci, const double *v, double *d) {
  int i = blockIdx.x;
  for (int q = rp[i] + threadIdx.x; q < rp[i + 1]; q += blockDim.x) d[(int64_t)i * nc + ci[q]] = v[q];
}
void to_dense(const Csr &a, double *d) {
  dzero(d, sizeof(double) * (size_t)a.nr * a.nc);
  if (!a.nr) return;
  k_to_dense<<<a.nr, 64, 0, stream()>>>(a.nr, a.nc, a.rp.p, a.ci.p, a.v.p, d);
  check_launch("to_dense");
}

}  // namespace mg
