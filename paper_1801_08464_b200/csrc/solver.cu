// Solver drivers: AMG hierarchy (amg.py:289-386 structure with PMIS /
// extended+i / L1-Jacobi), MGR hierarchy (mgr.py:265-377) and restarted
// right-preconditioned GMRES (krylov.py:44-144).  All vectors stay on the
// device; the host only runs the <= (m+1) x m Hessenberg / Givens recurrence.
#include <cmath>
#include <algorithm>
#include "ops.cuh"
#include "solver.cuh"
#include "sparse_util.cuh"
#include "amg_kernels.cuh"
#include "blockscale.cuh"
#include <cub/cub.cuh>

namespace mg {

static const int DENSE_LIMIT = 8192;

// ---- profiling of hot kernels ---------------------------------------------------
struct ProfRec { int kind; cudaEvent_t a, b; };
static thread_local std::vector<ProfRec> g_prof;

ProfScope::ProfScope(int k) : kind(k) {
  if (!g_ctx->profiling || k < 0) return;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, stream());
}
ProfScope::~ProfScope() {
  if (!a) return;
  cudaEventRecord(b, stream());
  g_prof.push_back({kind, a, b});
}
void prof_reset() {
  for (auto &r : g_prof) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
  g_prof.clear();
  g_ctx->timing.spmv_ms = g_ctx->timing.vcycle_ms = 0;
  g_ctx->timing.spmv_calls = g_ctx->timing.vcycle_calls = 0;
  for (double &p : g_ctx->timing.phase_ms) p = 0.0;
  g_ctx->timing.k0_ms = 0.0;
  g_ctx->timing.k0_calls = 0;
  g_ctx->timing.frelax_calls = 0;
  g_ctx->timing.frelax_bytes = 0.0;
}
static bool level_prof() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_PROF_LEVELS");
    on = e && *e == '1';
    return on;
  }();
  return on;
}

void prof_collect() {
  if (g_prof.empty()) return;
  cudaStreamSynchronize(stream());
  double lev[100] = {0};
  for (auto &r : g_prof) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.kind >= 100 && r.kind < 200) lev[r.kind - 100] += ms;
    if (r.kind >= 0 && r.kind < 8) g_ctx->timing.phase_ms[r.kind] += ms;
    if (r.kind == 8) { g_ctx->timing.k0_ms += ms; g_ctx->timing.k0_calls++; }
    if (r.kind == 0) { g_ctx->timing.spmv_ms += ms; g_ctx->timing.spmv_calls++; }
    else if (r.kind == 1) { g_ctx->timing.vcycle_ms += ms; g_ctx->timing.vcycle_calls++; }
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  if (level_prof()) {  // diagnostics: inclusive / exclusive V-cycle time per AMG level
    for (int hh = 0; hh < 2; ++hh)
      for (int l = 0; l < 50 && lev[hh * 50 + l] > 0; ++l)
        fprintf(stderr, "[mg] %s AMG level %d: inclusive %.3f ms, exclusive %.3f ms\n", hh ? "F-relax" : "coarse",
                l, lev[hh * 50 + l], lev[hh * 50 + l] - (l + 1 < 50 ? lev[hh * 50 + l + 1] : 0.0));
  }
}

// ================================ AMG ==============================================
double Amg::cycle_bytes() const {
  // Algorithmic bytes of one V(pre, post) cycle from x = 0, as executed
  // (SURVEY.md §8(d) with the zero-guess first sweep counted as what it is):
  //   first pre-sweep  x = D^-1 b            24 n
  //   each further sweep (SpMV_l + 16 n)     (reads b, D^-1; x gathered)
  //   residual          SpMV_l + 8 n          (skipped when pre == 0)
  //   restriction       SpMV(R_l);  prolongation SpMV(P_l) + 8 n (read-add)
  //   coarsest          8 n_c^2 + 16 n_c
  double tot = 0;
  for (size_t l = 0; l + 1 < L.size(); ++l) {
    const AmgLevel &v = L[l];
    double spmv = v.A.bytes_spmv(), n = v.n;
    double sweeps_spmv = (opts.pre > 0 ? opts.pre - 1 : 0) + opts.post;
    if (opts.pre > 0) tot += 24.0 * n + spmv + 8.0 * n;
    tot += sweeps_spmv * (spmv + 16.0 * n) + v.R.bytes_spmv() + v.P.bytes_spmv() + 8.0 * n;
  }
  tot += 8.0 * (double)cn * cn + 16.0 * cn;
  return tot;
}

std::unique_ptr<Amg> amg_setup(const Csr &a, const AmgOpts &o) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "amg_setup: scalar CSR required");
  if (a.nr != a.nc) throw MgError(MG_ERR_AMG_SETUP, "AMG expects a square operator");
  auto h = std::make_unique<Amg>();
  h->opts = o;
  // levels never move once built: the solve preparation of a finished level runs
  // on a worker stream while this thread coarsens the next one
  h->L.reserve((size_t)std::max(o.max_levels, 1) + 1);
  TaskGroup tasks;  // declared after h: joined before h can be destroyed
  auto prepare_level = [](AmgLevel &v) {
    v.l1inv.alloc((size_t)(v.n ? v.n : 1));
    l1_inverse(v.A, v.l1inv.p);
    prepare_spmv(v.A);
    prepare_spmv(v.P);
    prepare_spmv(v.R);
  };
  {
    AmgLevel l0;
    Csr flipped;
    DBuf<double> sgn;
    if (sign_normalise(a, flipped, sgn)) {
      l0.A = std::move(flipped);
      h->sign = std::move(sgn);
      h->has_sign = true;
    } else {
      l0.A = copy_csr(a);
    }
    l0.n = a.nr;
    h->L.push_back(std::move(l0));
  }
  while (h->L.back().n > o.cutoff && (int)h->L.size() < o.max_levels) {
    int li = (int)h->L.size() - 1;
    AmgLevel &cur = h->L[li];
    {
      char msg[96];
      snprintf(msg, sizeof msg, "amg level %d start n=%d nnz=%lld", li, cur.n, (long long)cur.A.nnz);
      trace(msg);
    }
    DBuf<int8_t> s;
    if (strength(cur.A, o.theta, s) == 0) break;  // no strong connection: no progress
    trace("  strength");
    DBuf<int8_t> state;
    pmis(cur.A, s.p, o.seed, li, state);
    trace("  pmis");
    DBuf<int> cmap;
    int nc = coarse_map(state.p, cur.n, cmap);
    if (nc == 0) throw MgError(MG_ERR_AMG_SETUP, "coarsening produced an empty C set");
    if (nc == cur.n) break;
    Csr p = ext_interp(cur.A, s.p, state.p, cmap.p, nc, o.max_elmts);
    trace("  ext_interp");
    Csr r = transpose(p);
    trace("  transpose");
    Csr ap = spgemm(cur.A, p, false);  // intermediate: R*(AP) sums do not depend on its order
    trace("  A*P");
    Csr ac = spgemm(r, ap, true, true);
    trace("  R*(AP)");
    cur.P = std::move(p);
    cur.R = std::move(r);
    cur.split = std::move(state);
    AmgLevel nxt;
    nxt.n = ac.nr;
    nxt.A = std::move(ac);
    h->L.push_back(std::move(nxt));
    // level li is final (A, P, R): its SELL copies / L1 norms are independent of
    // everything below; big levels prepare on a worker (the coarsening loop is
    // host-round-trip bound and leaves the GPU idle between its kernels)
    AmgLevel *lp = &h->L[li];
    if (lp->A.nnz >= (1 << 20)) tasks.run([lp, prepare_level]() { prepare_level(*lp); });
    else prepare_level(*lp);
  }
  tasks.join();
  for (size_t l = 0; l < h->L.size(); ++l) {
    AmgLevel &v = h->L[l];
    size_t n = (size_t)(v.n ? v.n : 1);
    v.x.alloc(n);
    v.b.alloc(n);
    v.r.alloc(n);
    v.t.alloc(n);
  }
  trace("  amg prepare joined");
  AmgLevel &last = h->L.back();
  if (last.n > std::max(o.cutoff, 200) && last.n > DENSE_LIMIT)
    throw MgError(MG_ERR_AMG_SETUP, "coarsening stalled at n=" + std::to_string(last.n) +
                                        " (dense coarsest solve limited to " + std::to_string(DENSE_LIMIT) + ")");
  h->cn = last.n;
  if (h->cn) {
    DBuf<double> dense((size_t)h->cn * h->cn);
    to_dense(last.A, dense.p);
    h->cinv.alloc((size_t)h->cn * h->cn);
    int bad = dense_inverse(dense.p, h->cinv.p, h->cn);
    if (bad >= 0) throw MgError(MG_ERR_SINGULAR, "coarsest AMG operator is singular", bad);
  }
  return h;
}

// The buffer level l's first pre-sweep from zero writes (x = D^-1 b): every sweep
// after it flips cur / oth, so it starts in the buffer that makes the last one land
// in x (no copy-back launch).  Producers of b (the restriction from level l-1, the
// MGR gather / restriction feeding the hierarchy) write x = D^-1 b there directly.
static double *first_buf(Amg &h, int l, double *x) {
  const int flips = (h.opts.pre > 0 ? h.opts.pre - 1 : 0) + h.opts.post;
  return (flips & 1) ? h.L[l].t.p : x;
}
static bool fused_pre(const Amg &h, int l) {  // level l has a pre-sweep that a producer can form
  return h.opts.pre > 0 && l + 1 < (int)h.L.size();
}

// pre_done: x_zero and the first pre-sweep's result is already in first_buf(l, x)
static void vcycle(Amg &h, int l, const double *b, double *x, bool x_zero, bool pre_done = false) {
  ProfScope plev(level_prof() && l < 50 ? 100 + (h.tag_k0 ? 0 : 50) + l : -1);
  AmgLevel &v = h.L[l];
  if (l + 1 == (int)h.L.size()) {
    dense_matvec(h.cinv.p, b, x, h.cn);
    return;
  }
  AmgLevel &nx = h.L[l + 1];
  double *cur = x, *oth = v.t.p;
  if (x_zero && first_buf(h, l, x) != x) std::swap(cur, oth);
  const int k0 = (h.tag_k0 && l == 0) ? 8 : -1;  // timed as the dominant kernel when profiling
  for (int s = 0; s < h.opts.pre; ++s) {
    if (x_zero) {
      if (!pre_done) vmul(cur, v.l1inv.p, b, v.n);
      x_zero = false;
    } else {
      ProfScope ps(k0);
      jacobi_sweep(v.A, cur, b, v.l1inv.p, oth);
      std::swap(cur, oth);
    }
  }
  const double *res = b;
  if (!x_zero) {
    residual(v.A, cur, b, v.r.p);
    res = v.r.p;
  }
  const bool fuse = fused_pre(h, l + 1);
  if (fuse) spmv_store_scale(v.R, res, nx.b.p, nullptr, nullptr, nx.l1inv.p, first_buf(h, l + 1, nx.x.p));
  else spmv(v.R, res, nx.b.p);
  vcycle(h, l + 1, nx.b.p, nx.x.p, true, fuse);
  if (x_zero) spmv(v.P, nx.x.p, cur);
  else spmv_add(v.P, nx.x.p, cur);
  for (int s = 0; s < h.opts.post; ++s) {
    ProfScope ps(k0);
    jacobi_sweep(v.A, cur, b, v.l1inv.p, oth);
    std::swap(cur, oth);
  }
  if (cur != x) vcopy(x, cur, v.n);
}

AmgPreTargets amg_pre_targets(Amg &h, double *x) {
  AmgPreTargets t;
  if (!fused_pre(h, 0)) return t;
  t.ok = true;
  t.sign = h.has_sign ? h.sign.p : nullptr;
  t.bs = h.has_sign ? h.L[0].b.p : nullptr;
  t.d = h.L[0].l1inv.p;
  t.xo = first_buf(h, 0, x);
  return t;
}

void amg_vcycle(Amg &h, const double *b, const double *x0, double *x, bool pre_done) {
  AmgLevel &l0 = h.L[0];
  const double *bb = b;
  if (h.has_sign) {
    if (!pre_done) vmul(l0.b.p, h.sign.p, b, l0.n);
    bb = l0.b.p;
  }
  if (x0) {
    if (x0 != x) vcopy(x, x0, l0.n);
    vcycle(h, 0, bb, x, false);
  } else {
    vcycle(h, 0, bb, x, true, pre_done);
  }
}

void amg_apply(Amg &h, const double *b, double *x, bool pre_done) {
  ProfScope ps(1);
  amg_vcycle(h, b, nullptr, x, pre_done);
  for (int c = 1; c < h.opts.cycles; ++c) amg_vcycle(h, b, x, x);
}

// ================================ MGR ==============================================
static void fsolver_setup(FSolver &fs, Csr &aff, const LevelSpec &sp, const AmgOpts &ao) {
  fs.kind = sp.frelax;
  fs.sweeps = sp.sweeps;
  fs.nf = aff.nr;
  size_t nf = (size_t)(aff.nr ? aff.nr : 1);
  fs.t1.alloc(nf);
  fs.t2.alloc(nf);
  if (sp.frelax == FR_JACOBI) {
    DBuf<double> d(nf);
    row_diag(aff, d.p);
    std::vector<double> hd(aff.nr);
    d2h(hd.data(), d.p, sizeof(double) * aff.nr);
    for (int i = 0; i < aff.nr; ++i)
      if (hd[i] == 0.0) throw MgError(MG_ERR_ZERO_F_DIAG, "zero diagonal in A_ff at fine row " + std::to_string(i), i);
    for (auto &v : hd) v = 1.0 / v;
    fs.invd.alloc(nf);
    h2d(fs.invd.p, hd.data(), sizeof(double) * aff.nr);
  } else if (sp.frelax == FR_AMG) {
    AmgOpts o = ao;
    o.max_levels = sp.max_levels ? sp.max_levels : ao.max_levels;
    o.pre = sp.pre;
    o.post = sp.post;
    o.cycles = 1;
    fs.amg = amg_setup(aff, o);
  } else if (sp.frelax == FR_EXACT) {
    if (aff.nr > DENSE_LIMIT)
      throw MgError(MG_ERR_UNSUPPORTED, "FRelax('exact') on the GPU is limited to n_f <= 8192");
    DBuf<double> dense((size_t)aff.nr * aff.nr);
    to_dense(aff, dense.p);
    fs.dinv.alloc((size_t)aff.nr * aff.nr);
    int bad = dense_inverse(dense.p, fs.dinv.p, aff.nr);
    if (bad >= 0) throw MgError(MG_ERR_SINGULAR, "A_ff is singular", bad);
  } else {
    tril_setup(aff, fs.tril);
    fs.ctrl.alloc(nf + 1);
  }
}

static void fsolve(FSolver &fs, const Csr &aff, const double *r, double *x, bool pre_done = false) {
  if (fs.kind == FR_JACOBI) {
    vmul(x, fs.invd.p, r, fs.nf);
    double *cur = x, *oth = fs.t1.p;
    for (int s = 1; s < fs.sweeps; ++s) {
      jacobi_sweep(aff, cur, r, fs.invd.p, oth);
      std::swap(cur, oth);
    }
    if (cur != x) vcopy(x, cur, fs.nf);
  } else if (fs.kind == FR_AMG) {
    amg_vcycle(*fs.amg, r, nullptr, x, pre_done);
  } else if (fs.kind == FR_GS) {
    // x = L^-1 r; x += L^-1 (r - A_ff x) per further sweep (mgr.py:185-188)
    trsv_lower(fs.tril, r, x, fs.ctrl.p);
    for (int s = 1; s < fs.sweeps; ++s) {
      residual(aff, x, r, fs.t1.p);
      trsv_lower(fs.tril, fs.t1.p, fs.t2.p, fs.ctrl.p);
      vadd(x, fs.t2.p, fs.nf);
    }
  } else {
    dense_matvec(fs.dinv.p, r, x, fs.nf);
  }
}

// per-cell block-diagonal relaxation: x[id] = inv_b r[id] per block
__global__ void k_bd_apply(int nblk, const int *ioff, const int64_t *moff, const int *idx, const double *inv,
                           const double *r, double *x) {
  PDL_ENTRY();
  int bi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= nblk) return;
  const int k = ioff[bi + 1] - ioff[bi];
  const int *id = idx + ioff[bi];
  const double *m = inv + moff[bi];
  for (int a = 0; a < k; ++a) {
    double s = 0.0;
    for (int c = 0; c < k; ++c) s += m[a * k + c] * r[id[c]];
    x[id[a]] = s;
  }
}
__global__ void k_bd_gather(int nblk, const int *ioff, const int64_t *moff, const int *idx, const int *rp,
                            const int *ci, const double *v, double *blk) {
  int bi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= nblk) return;
  const int k = ioff[bi + 1] - ioff[bi];
  const int *id = idx + ioff[bi];
  double *o = blk + moff[bi];
  for (int a = 0; a < k; ++a)
    for (int c = 0; c < k; ++c) {
      double val = 0.0;
      int row = id[a], col = id[c];
      for (int q = rp[row]; q < rp[row + 1]; ++q)
        if (ci[q] == col) { val = v[q]; break; }
      o[a * k + c] = val;
    }
}
// small dense inverses by Gauss-Jordan with partial pivoting, one thread per block
// (k <= 8).  K > 0: the same elimination with the block size fixed at compile time,
// so the augmented matrix lives in registers (identical operations, bitwise equal)
template <int K>
__device__ __forceinline__ bool bd_invert_fixed(const double *bk, double *o) {
  double a[K][2 * K];
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) a[i][j] = j < K ? bk[i * K + j] : (j - K == i ? 1.0 : 0.0);
#pragma unroll
  for (int c = 0; c < K; ++c) {
    int p = c;
#pragma unroll
    for (int i = c + 1; i < K; ++i)
      if (fabs(a[i][c]) > fabs(a[p][c])) p = i;
    // swap rows p and c with static indexing (p >= c)
    double pr[2 * K];
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) pr[j] = a[c][j];
#pragma unroll
    for (int i = c + 1; i < K; ++i)
      if (i == p) {
#pragma unroll
        for (int j = 0; j < 2 * K; ++j) { double t = a[i][j]; a[i][j] = pr[j]; pr[j] = t; }
      }
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) a[c][j] = pr[j];
    if (a[c][c] == 0.0) return false;
    const double pv = a[c][c];
#pragma unroll
    for (int j = 0; j < 2 * K; ++j) a[c][j] /= pv;
#pragma unroll
    for (int i = 0; i < K; ++i) {
      if (i == c) continue;
      const double f = a[i][c];
      if (f != 0.0) {
#pragma unroll
        for (int j = 0; j < 2 * K; ++j) a[i][j] -= f * a[c][j];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) o[i * K + j] = a[i][K + j];
  return true;
}
__global__ void k_bd_invert(int nblk, const int *ioff, const int64_t *moff, const double *blk, double *inv,
                            int *bad) {
  int bi = blockIdx.x * blockDim.x + threadIdx.x;
  if (bi >= nblk) return;
  const int k = ioff[bi + 1] - ioff[bi];
  const double *bk = blk + moff[bi];
  if (k == 2 || k == 3) {
    const bool ok = k == 2 ? bd_invert_fixed<2>(bk, inv + moff[bi]) : bd_invert_fixed<3>(bk, inv + moff[bi]);
    if (!ok) atomicMin(bad, bi);
    return;
  }
  double a[8][16];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < 2 * k; ++j) a[i][j] = j < k ? bk[i * k + j] : (j - k == i ? 1.0 : 0.0);
  for (int c = 0; c < k; ++c) {
    int p = c;
    for (int i = c + 1; i < k; ++i)
      if (fabs(a[i][c]) > fabs(a[p][c])) p = i;
    if (a[p][c] == 0.0) { atomicMin(bad, bi); return; }
    if (p != c)
      for (int j = 0; j < 2 * k; ++j) { double t = a[c][j]; a[c][j] = a[p][j]; a[p][j] = t; }
    double pv = a[c][c];
    for (int j = 0; j < 2 * k; ++j) a[c][j] /= pv;
    for (int i = 0; i < k; ++i) {
      if (i == c) continue;
      double f = a[i][c];
      if (f != 0.0)
        for (int j = 0; j < 2 * k; ++j) a[i][j] -= f * a[c][j];
    }
  }
  double *o = inv + moff[bi];
  for (int i = 0; i < k; ++i)
    for (int j = 0; j < k; ++j) o[i * k + j] = a[i][k + j];
}

// per-unknown owning cell: grouping on the device (mgr.py:219-224: unknowns grouped
// by cell, ascending inside a group, groups in ascending cell order)
__global__ void k_cells_unsorted(const int64_t *c, int n, int *flag) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i > 0 && i < n && c[i] < c[i - 1]) *flag = 1;
}
__global__ void k_cell_heads(const int64_t *c, int n, int *head) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || c[i] != c[i - 1]) ? 1 : 0;
}
__global__ void k_cell_starts(const int *head, const int *seg, int n, int nblk, int *ioff) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && head[i]) ioff[seg[i]] = i;
  if (i == 0) ioff[nblk] = n;
}
__global__ void k_block_sizes(const int *ioff, int nblk, int *ksq, int *kmax) {
  int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= nblk) return;
  const int k = ioff[b + 1] - ioff[b];
  ksq[b] = k <= 8 ? k * k : 0;
  atomicMax(kmax, k);
}
__global__ void k_gather_i64(int64_t *d, const int64_t *s, const int *idx, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) d[i] = s[idx[i]];
}

static std::unique_ptr<BlockDiag> blockdiag_setup(const Csr &a, const int64_t *cells) {
  // group unknowns by owning cell on the device: stable radix sort of (cell, index)
  // unless the cells are already non-decreasing (cell-major numbering), run heads,
  // block offsets; each group is one dense block (sizes may differ between cells)
  const int n = a.nr;
  auto bd = std::make_unique<BlockDiag>();
  bd->idx.alloc((size_t)(n ? n : 1));
  if (n == 0) {
    bd->ioff.alloc(1);
    dset_i32(bd->ioff.p, {0});
    bd->moff.alloc(1);
    dzero(bd->moff.p, sizeof(int64_t));
    return bd;
  }
  iota_i32(bd->idx.p, n);
  DBuf<int> st(2);
  dset_i32(st.p, {0, 0});
  k_cells_unsorted<<<grid_for(n, 256), 256, 0, stream()>>>(cells, n, st.p);
  check_launch("cells_unsorted");
  int unsorted = 0;
  d2h(&unsorted, st.p, sizeof(int));
  DBuf<int64_t> sorted_cells;
  const int64_t *keys = cells;
  if (unsorted) {
    sorted_cells.alloc(n);
    DBuf<int> order(n);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, cells, sorted_cells.p, bd->idx.p, order.p, n, 0, 64, stream());
    void *tmp = cub_scratch(tb);
    MG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, cells, sorted_cells.p, bd->idx.p, order.p, n, 0, 64,
                                            stream()));
    count_launch(8);
    std::swap(bd->idx, order);
    keys = sorted_cells.p;
  }
  DBuf<int> head(n), seg((size_t)n + 1);
  k_cell_heads<<<grid_for(n, 256), 256, 0, stream()>>>(keys, n, head.p);
  check_launch("cell_heads");
  const int nblk = (int)exclusive_scan_i32_to_i32(head.p, seg.p, n);
  bd->nblk = nblk;
  bd->ioff.alloc((size_t)nblk + 1);
  k_cell_starts<<<grid_for(n, 256), 256, 0, stream()>>>(head.p, seg.p, n, nblk, bd->ioff.p);
  check_launch("cell_starts");
  DBuf<int> ksq(nblk);
  k_block_sizes<<<grid_for(nblk, 256), 256, 0, stream()>>>(bd->ioff.p, nblk, ksq.p, st.p + 1);
  check_launch("block_sizes");
  bd->moff.alloc((size_t)nblk + 1);
  const int64_t tot = exclusive_scan_i32_to_i64(ksq.p, bd->moff.p, nblk);
  d2h(&bd->kmax, st.p + 1, sizeof(int));
  if (bd->kmax > 8) throw MgError(MG_ERR_UNSUPPORTED, "global_relax: per-cell blocks larger than 8");
  DBuf<double> blk((size_t)(tot ? tot : 1));
  bd->inv.alloc((size_t)(tot ? tot : 1));
  k_bd_gather<<<grid_for(nblk, 128), 128, 0, stream()>>>(nblk, bd->ioff.p, bd->moff.p, bd->idx.p, a.rp.p,
                                                         a.ci.p, a.v.p, blk.p);
  check_launch("bd_gather");
  DBuf<int> bad(1);
  const int big = 0x7fffffff;
  dset_i32(bad.p, {big});
  k_bd_invert<<<grid_for(nblk, 64), 64, 0, stream()>>>(nblk, bd->ioff.p, bd->moff.p, blk.p, bd->inv.p, bad.p);
  check_launch("bd_invert");
  int hb;
  d2h(&hb, bad.p, sizeof(int));
  if (hb != big) throw MgError(MG_ERR_SINGULAR, "singular per-cell block", hb);
  return bd;
}

std::unique_ptr<Mgr> mgr_setup(const Csr &a, const std::vector<LevelSpec> &plan, const AmgOpts &ao,
                               int coarse_kind, bool post_smoothing, const int64_t *cells_host) {
  if (a.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "mgr_setup: scalar CSR required");
  if (a.nr != a.nc) throw MgError(MG_ERR_DIM_MISMATCH, "mgr_setup: square matrix required");
  if (coarse_kind != 0 && coarse_kind != 1) throw MgError(MG_ERR_BAD_OPTION, "unknown coarse solver");
  timeline_reset();
  trace("mgr: enter");
  auto h = std::make_unique<Mgr>();
  h->n0 = a.nr;
  h->post_smoothing = post_smoothing;
  h->coarse_kind = coarse_kind;
  h->L.reserve(plan.size());
  TaskGroup tasks;  // declared after h: joined before h can be destroyed
  int parent_level = -1;       // MGR level this thread is building
  std::vector<int> task_level;  // MGR level of each worker task
  try {
    Csr cur = copy_csr(a);
    // per-unknown owning cell, tracked down the levels only when a level relaxes globally
    bool need_cells = false;
    for (const LevelSpec &sp : plan) need_cells |= sp.global_relax != 0;
    DBuf<int64_t> cells;  // device copy, gathered down the levels by the C lists
    if (need_cells) {
      cells.alloc((size_t)(a.nr ? a.nr : 1));
      if (cells_host) {
        h2d(cells.p, cells_host, sizeof(int64_t) * a.nr);
      } else {
        std::vector<int64_t> ident(a.nr);
        for (int i = 0; i < a.nr; ++i) ident[i] = i;
        h2d(cells.p, ident.data(), sizeof(int64_t) * a.nr);
      }
    }
    for (const LevelSpec &sp : plan) {
      int n = cur.nr;
      if ((int)sp.fmask.size() != n) throw MgError(MG_ERR_DIM_MISMATCH, "level plan mask length mismatch");
      int nf_h = 0;
      for (uint8_t m : sp.fmask) nf_h += m != 0;
      if (nf_h == 0 || nf_h == n) continue;
      h->L.emplace_back();
      MgrLevel &lv = h->L.back();  // stable: capacity reserved
      parent_level = (int)h->L.size() - 1;
      lv.n = n;
      lv.rp = sp.rp;
      DBuf<uint8_t> mask(n);
      h2d(mask.p, sp.fmask.data(), n);
      DBuf<int> cmap;
      DBuf<int> &fmap = lv.fmap;
      fc_split(mask.p, n, lv.flist, lv.clist, fmap, cmap, lv.nf, lv.nc);
      trace("mgr: fc_split");
      lv.Aff = extract(cur, lv.flist.p, lv.nf, fmap.p, lv.nf);
      trace("mgr: extract A_ff");
      // The F-relaxation setup (an AMG hierarchy on A_ff for FRelax('amg')) needs
      // only A_ff: it runs on a worker stream while this thread builds R, P, the
      // Galerkin product and everything below this level.
      {
        MgrLevel *lvp = &lv;
        const LevelSpec *spp = &sp;
        tasks.run([lvp, spp, ao]() {
          fsolver_setup(lvp->fs, lvp->Aff, *spp, ao);
          prepare_spmv(lvp->Aff);
          trace("mgr: F-solver setup");
        });
        task_level.push_back(parent_level);
      }
      build_rp(cur, fmap.p, cmap.p, lv.flist.p, lv.clist.p, lv.nf, lv.nc, sp.rp, lv.R, lv.P);
      trace("mgr: build_rp");
      Csr ap = spgemm(cur, lv.P, false);
      trace("mgr: A*P");
      Csr ac = spgemm(lv.R, ap, true, true);
      trace("mgr: R*(AP)");
      if (sp.global_relax) lv.bd = blockdiag_setup(cur, cells.p);
      if (need_cells) {
        DBuf<int64_t> nxt((size_t)(lv.nc ? lv.nc : 1));
        if (lv.nc) {
          k_gather_i64<<<grid_for(lv.nc, 256), 256, 0, stream()>>>(nxt.p, cells.p, lv.clist.p, lv.nc);
          check_launch("gather_cells");
        }
        std::swap(cells, nxt);
      }
      lv.A = std::move(cur);
      cur = std::move(ac);
      // the solve-phase preparation of this level (A[:, F], SELL copies, work
      // vectors) is independent of everything below: a second worker
      {
        MgrLevel *lvp = &lv;
        const bool want_af = !post_smoothing && !sp.global_relax;
        const bool want_afr = post_smoothing && !sp.global_relax;
        tasks.run([lvp, want_af, want_afr, n]() {
          if (want_afr) {
            // coarse correction first: the F-relaxation that follows needs the residual
            // r - A e on the F rows only (half of A), written densely in F order
            DBuf<int> allcols(n);
            iota_i32(allcols.p, n);
            lvp->AFr = extract(lvp->A, lvp->flist.p, lvp->nf, allcols.p, n);
            prepare_spmv(lvp->AFr);
          }
          if (want_af) {
            // after the F-relaxation from e = 0, e is zero on C: r - A e = r - A[:, F] e_F
            DBuf<int> allrows(n);
            iota_i32(allrows.p, n);
            lvp->AF = extract(lvp->A, allrows.p, n, lvp->fmap.p, lvp->nf);
            prepare_spmv(lvp->AF);
          }
          if (!want_afr) prepare_spmv(lvp->A);  // with A[F, :] the apply never multiplies by A itself
          prepare_spmv(lvp->R);
          prepare_spmv(lvp->P);
          lvp->res.alloc(n);
          lvp->rF.alloc(lvp->nf);
          lvp->eF.alloc(lvp->nf);
          lvp->rc.alloc(lvp->nc);
          lvp->ec.alloc(lvp->nc);
        });
        task_level.push_back(parent_level);
      }
    }
    parent_level = 1 << 30;  // below every level
    trace("mgr: levels done");
    if (coarse_kind == 0) {
      h->camg = amg_setup(cur, ao);
      h->camg->tag_k0 = true;
      trace("mgr: coarse AMG setup");
    } else {
      if (cur.nr > DENSE_LIMIT) throw MgError(MG_ERR_UNSUPPORTED, "coarse='exact' on the GPU is limited to n <= 8192");
      h->cn = cur.nr;
      DBuf<double> dense((size_t)cur.nr * cur.nr);
      to_dense(cur, dense.p);
      h->cinv.alloc((size_t)cur.nr * cur.nr);
      int bad = dense_inverse(dense.p, h->cinv.p, cur.nr);
      if (bad >= 0) throw MgError(MG_ERR_SINGULAR, "coarse operator is singular", bad);
    }
    h->coarse_A = std::move(cur);
  } catch (...) {
    // errors in the reference's order (mgr.py:280-300): per level build_rp,
    // RAP, then the F-solver; a failing F-solver of an earlier level wins over
    // this thread's error, this level's F-solver error loses to it
    std::exception_ptr pe = std::current_exception();
    std::vector<std::exception_ptr> we = tasks.join_errors();
    for (int k = 0; k < (int)we.size(); ++k)
      if (we[k] && task_level[k] < parent_level) std::rethrow_exception(we[k]);
    std::rethrow_exception(pe);
  }
  tasks.join();  // F-solver errors of any level
  trace("mgr: joined");
  timeline_dump();
  return h;
}

static void apply_level(Mgr &h, size_t k, const double *r, double *e, bool pre_done = false) {
  if (k == h.L.size()) {
    if (h.coarse_kind == 0) amg_apply(*h.camg, r, e, pre_done);
    else dense_matvec(h.cinv.p, r, e, h.cn);
    return;
  }
  MgrLevel &lv = h.L[k];
  bool zero = true;
  bool f_only = false;  // e = [e_F; 0] exactly (F-relaxation from zero)
  bool merged = true;   // false: e = [e_F; 0] not written yet (merged into the prolongation)
  if (lv.bd) {
    launch_pdl(k_bd_apply, grid_for(lv.bd->nblk, 128), 128, 0, lv.bd->nblk, lv.bd->ioff.p, lv.bd->moff.p,
                                                                 lv.bd->idx.p, lv.bd->inv.p, r, e);
    check_launch("bd_apply");
    zero = false;
  }
  auto resid = [&]() -> const double * {
    if (zero) return r;
    if (f_only && lv.AF.nr) residual(lv.AF, lv.eF.p, r, lv.res.p);  // skips the zero C columns
    else residual(lv.A, e, r, lv.res.p);
    return lv.res.p;
  };
  auto f_relax = [&]() {
    bool pre = false;
    {
      ProfScope ps(4);
      // the F-relaxation AMG's first pre-sweep (x = D^-1 r_F) is formed by the gather
      AmgPreTargets t;
      if (lv.fs.kind == FR_AMG) t = amg_pre_targets(*lv.fs.amg, lv.eF.p);
      if (!zero && lv.AFr.nr) {
        // r_F = r[F] - A[F, :] e in one pass over half of A (no full residual, no gather)
        residual_rows_scale(lv.AFr, e, r, lv.flist.p, lv.rF.p, t.sign, t.bs, t.d, t.ok ? t.xo : nullptr);
      } else {
        const double *rr = resid();
        if (t.ok) gather_scale(lv.rF.p, rr, lv.flist.p, lv.nf, t.sign, t.bs, t.d, t.xo);
        else gather(lv.rF.p, rr, lv.flist.p, lv.nf);
      }
      pre = t.ok;
    }
    {
      ProfScope ps(2);
      fsolve(lv.fs, lv.Aff, lv.rF.p, lv.eF.p, pre);
      if (g_ctx->profiling && lv.fs.amg) {
        g_ctx->timing.frelax_calls++;
        g_ctx->timing.frelax_bytes += lv.fs.amg->cycle_bytes();
      }
    }
    ProfScope ps(4);
    if (zero) {
      // e = [e_F; 0]: with A[:, F] the residual reads e_F directly and the merge
      // is folded into the prolongation's epilogue; otherwise one merge pass
      if (lv.AF.nr && !h.post_smoothing) merged = false;
      else fc_merge(e, lv.eF.p, lv.fmap.p, lv.n);
      f_only = true;
    } else {
      scatter_add(e, lv.eF.p, lv.flist.p, lv.nf);
      f_only = false;
    }
    zero = false;
  };
  auto coarse_correct = [&]() {
    bool pre = false;
    {
      ProfScope ps(4);
      const double *rr = resid();
      // restriction into the coarse AMG: its first pre-sweep is formed in the epilogue
      AmgPreTargets t;
      if (k + 1 == h.L.size() && h.coarse_kind == 0) t = amg_pre_targets(*h.camg, lv.ec.p);
      if (t.ok) spmv_store_scale(lv.R, rr, lv.rc.p, t.sign, t.bs, t.d, t.xo);
      else spmv(lv.R, rr, lv.rc.p);
      pre = t.ok;
    }
    apply_level(h, k + 1, lv.rc.p, lv.ec.p, pre);
    ProfScope ps(4);
    if (zero) spmv(lv.P, lv.ec.p, e);
    else if (!merged) spmv_merge_add(lv.P, lv.ec.p, lv.fmap.p, lv.eF.p, e);
    else spmv_add(lv.P, lv.ec.p, e);
    merged = true;
    zero = false;
    f_only = false;
  };
  if (h.post_smoothing) {
    coarse_correct();
    f_relax();
  } else {
    f_relax();
    coarse_correct();
  }
}

static void mgr_apply_direct(Mgr &h, const double *r, double *e, const double *const *rslot = nullptr) {
  const double *rr = r;
  if (h.has_prescale) {
    ProfScope ps(5);
    if (rslot) block_apply_indirect(h.prescale, rslot, h.pre_buf.p);
    else block_apply(h.prescale, r, h.pre_buf.p);
    rr = h.pre_buf.p;
  }
  apply_level(h, 0, rr, e);
}

void Mgr::drop_graph() {
  if (!gexec) return;
  // park it in its context for the next hierarchy's update (one slot)
  if (gctx && !gctx->parked_exec) gctx->parked_exec = gexec;
  else cudaGraphExecDestroy(gexec);
  gexec = nullptr;
}
Mgr::~Mgr() { drop_graph(); }

static bool graphs_enabled() {
  static const int on = [] {
    int on = -1;
    const char *e = getenv("MG_GRAPHS");
    on = !(e && *e == '0');
    return on;
  }();
  return on != 0;
}

// Capture one apply (gin -> gout) as a CUDA graph: the ~100 dependent kernel
// launches of an MGR + 2 AMG cycles replay with minimal inter-kernel gaps.
static bool capture_apply(Mgr &h) {
  if (!h.gout.p) {
    if (h.has_prescale) h.in_slot.alloc(1);
    else h.gin.alloc((size_t)h.n0);
    h.gout.alloc((size_t)h.n0);
  }
  cudaGraph_t graph = nullptr;
  int64_t l0 = g_ctx->launches;
  if (cudaStreamBeginCapture(stream(), cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  bool ok = true;
  try {
    if (h.has_prescale) mgr_apply_direct(h, nullptr, h.gout.p, h.in_slot.p);
    else mgr_apply_direct(h, h.gin.p, h.gout.p);
  } catch (...) {
    ok = false;
  }
  cudaError_t e = cudaStreamEndCapture(stream(), &graph);
  if (!ok || e != cudaSuccess || !graph) {
    cudaGetLastError();
    if (graph) cudaGraphDestroy(graph);
    g_ctx->launches = l0;
    return false;
  }
  // a parked executable of a previous hierarchy with the same topology is updated
  // in place (kernel parameters only), else a new one is instantiated
  e = cudaErrorUnknown;
  if (g_ctx->parked_exec) {
    cudaGraphExecUpdateResultInfo info{};
    if (cudaGraphExecUpdate(g_ctx->parked_exec, graph, &info) == cudaSuccess) {
      h.gexec = g_ctx->parked_exec;
      e = cudaSuccess;
    } else {
      cudaGetLastError();
      cudaGraphExecDestroy(g_ctx->parked_exec);
    }
    g_ctx->parked_exec = nullptr;
  }
  const bool updated = e == cudaSuccess;
  if (e != cudaSuccess) e = cudaGraphInstantiate(&h.gexec, graph, 0);
  cudaGraphDestroy(graph);
  static const bool gtrace = getenv("MG_GRAPH_TRACE") != nullptr;
  if (gtrace) fprintf(stderr, "[mg] MGR apply graph %s\n", updated ? "updated in place" : "instantiated");
  if (e != cudaSuccess) {
    cudaGetLastError();
    h.gexec = nullptr;
    g_ctx->launches = l0;
    return false;
  }
  h.graph_kernels = g_ctx->launches - l0;
  h.gctx = g_ctx;
  g_ctx->launches = l0;
  return true;
}

const double *mgr_apply_result(Mgr &h, const double *r, double *e) {
  if (g_ctx->profiling || !graphs_enabled() || h.graph_failed) {
    mgr_apply_direct(h, r, e);
    return e;
  }
  if (!h.gexec && !capture_apply(h)) {
    h.graph_failed = true;
    mgr_apply_direct(h, r, e);
    return e;
  }
  if (h.has_prescale) set_device_ptr(h.in_slot.p, r);
  else if (r != h.gin.p) vcopy(h.gin.p, r, h.n0);
  MG_CUDA(cudaGraphLaunch(h.gexec, stream()));
  g_ctx->launches += h.graph_kernels;
  return h.gout.p;
}

void mgr_apply(Mgr &h, const double *r, double *e) {
  const double *out = mgr_apply_result(h, r, e);
  if (out != e) vcopy(e, out, h.n0);
}

// ================================ GMRES ============================================
static void op_apply(const Csr &a, const double *x, double *y) {
  ProfScope ps(0);
  spmv(a, x, y);
}

GmresOut gmres(const Csr &a, Mgr *m, const double *b, double *x, const GmresOpts &o, double a_norm, Ilu *ilu) {
  int64_t n = (int64_t)a.nr * a.b;
  if ((int64_t)a.nc * a.b != n) throw MgError(MG_ERR_DIM_MISMATCH, "gmres: square operator required");
  if (m && m->n0 != n) throw MgError(MG_ERR_DIM_MISMATCH, "gmres: preconditioner dimension mismatch");
  if (o.rel_tol <= 0.0) throw MgError(MG_ERR_BAD_OPTION, "rel_tol must be positive");
  if (o.restart < 1 || o.max_iter < 1) throw MgError(MG_ERR_BAD_OPTION, "restart and max_iter must be at least 1");
  GmresOut out;
  bool use_anorm = a_norm >= 0.0;
  double b_norm = nrm2(b, n);
  out.rhs_norm = b_norm;
  if (b_norm == 0.0) {
    vfill(x, 0.0, n);
    out.converged = 1;
    return out;
  }
  double tol = o.rel_tol * b_norm;
  auto accepted = [&](double res, double xn) {
    if (res <= tol) return true;
    return use_anorm && res <= o.rel_tol * (a_norm * xn + b_norm);
  };
  int mmax = std::min(o.restart, o.max_iter);
  // reorth 1: DCGS2 (default, restart <= 31); 2: classic CGS2, the reference's two
  // full projection passes in krylov.py:101-107 order; 0: one CGS pass
  const bool dcgs2 = o.reorth == 1 && mmax <= 31;
  static const bool trace = [] {  // MG_GMRES_TRACE=1: per-step |g| and cycle-top residuals on stderr
    const char *e = getenv("MG_GMRES_TRACE");
    return e && *e == '1';
  }();
  // basis row stride padded off a power of two (K streams 32 MB apart otherwise collide)
  const int64_t ldv = ((n + 1) & ~(int64_t)1) + 1024;
  DBuf<double> V((size_t)(mmax + 1) * ldv), w(n), z(n), r(n), xt(n), u(n), t(n), proj((size_t)2 * (mmax + 1) + 8),
      coefd(2 * 32 + 3);
  double *c_dev = proj.p, *c2_dev = proj.p + (mmax + 1), *nrm_dev = proj.p + 2 * (mmax + 1);
  std::vector<double> hbuf(2 * (mmax + 1) + 1);
  vfill(x, 0.0, n);
  int total = 0;
  if (ilu && ilu->n != n) throw MgError(MG_ERR_DIM_MISMATCH, "gmres: preconditioner dimension mismatch");
  auto precond = [&](const double *v, double *out_) -> const double * {
    if (ilu) {
      ilu_apply(*ilu, v, out_);
      return out_;
    }
    if (!m) return v;
    return mgr_apply_result(*m, v, out_);
  };
  while (true) {
    double res;
    if (total) {
      op_apply(a, x, t.p);
      vsub(r.p, b, t.p, n);
      res = nrm2(r.p, n);
    } else {
      vcopy(r.p, b, n);
      res = b_norm;
    }
    if (trace) fprintf(stderr, "[gmres] cycle top: total %d res %.17g relres %.6e\n", total, res, res / b_norm);
    if (!std::isfinite(res)) {
      // a NaN / Inf residual (non-finite matrix, rhs or preconditioner output)
      // cannot recover: report non-convergence now (the reference keeps
      // iterating on NaNs until max_iter and returns converged=False too)
      out.iterations = total;
      out.converged = 0;
      out.residual_norm = res;
      return out;
    }
    double xn = use_anorm ? nrm2(x, n) : 0.0;
    if (accepted(res, xn)) {
      out.iterations = total;
      out.converged = 1;
      out.residual_norm = res;
      return out;
    }
    if (total >= o.max_iter) {
      out.iterations = total;
      out.converged = 0;
      out.residual_norm = res;
      return out;
    }
    int mm = std::min(o.restart, o.max_iter - total);
    std::vector<double> H((size_t)(mm + 1) * mm, 0.0), cs(mm, 0.0), sn(mm, 0.0), g(mm + 1, 0.0);
    auto h_at = [&](int i, int j) -> double & { return H[(size_t)i * mm + j]; };
    vdiv_scalar(V.p, r.p, res, n);
    g[0] = res;
    auto assemble = [&](int k, double *xout) {
      std::vector<double> y(k, 0.0);
      for (int i = k - 1; i >= 0; --i) {
        double s = g[i];
        for (int j = i + 1; j < k; ++j) s -= h_at(i, j) * y[j];
        y[i] = s / h_at(i, i);
      }
      if (k) {
        h2d(c_dev, y.data(), sizeof(double) * k);
        combine(V.p, ldv, k, c_dev, u.p, n);
      } else {
        vfill(u.p, 0.0, n);
      }
      const double *mz = precond(u.p, z.p);
      if (xout != x) vcopy(xout, x, n);
      vadd(xout, mz, n);
    };
    int k = 0;
    bool early = false;
    double early_res = 0.0;
    if (dcgs2) {
      // One-reduction CGS2 with delayed reorthogonalisation (DCGS2): V[j] holds
      // the once-orthogonalised u_j (unnormalised); one dot pass gives
      // [Q^T u, Q^T w, u.u, u.w], the update pass finalises q_j (the second
      // CGS pass of u_j) and forms u_{j+1} from w in the same read of Q.  The
      // provisional column j-1 of H is corrected with the reorthogonalisation
      // coefficients (h += beta s, h_{j,j-1} = beta alpha), and the first
      // projection of w is reconstructed from Q^T w through the Arnoldi
      // relation of the corrected columns.  Two basis passes per step instead
      // of CGS2's four; GMRES's decisions use the same Givens / |g| tests.
      std::vector<double> Hr((size_t)(mm + 1) * mm, 0.0), coef(2 * 32 + 3), sv(mm), tv(mm), cvec(mm + 1);
      auto hr = [&](int i, int jj) -> double & { return Hr[(size_t)i * mm + jj]; };
      auto givens = [&](int kc) {  // H, g <- QR of the first kc raw columns
        for (size_t q = 0; q < H.size(); ++q) H[q] = Hr[q];
        std::fill(g.begin(), g.end(), 0.0);
        g[0] = res;
        for (int jj = 0; jj < kc; ++jj) {
          for (int i = 0; i < jj; ++i) {
            double t0 = cs[i] * h_at(i, jj) + sn[i] * h_at(i + 1, jj);
            h_at(i + 1, jj) = -sn[i] * h_at(i, jj) + cs[i] * h_at(i + 1, jj);
            h_at(i, jj) = t0;
          }
          double den = std::hypot(h_at(jj, jj), h_at(jj + 1, jj));
          if (den == 0.0) return jj;
          cs[jj] = h_at(jj, jj) / den;
          sn[jj] = h_at(jj + 1, jj) / den;
          h_at(jj, jj) = den;
          h_at(jj + 1, jj) = 0.0;
          g[jj + 1] = -sn[jj] * g[jj];
          g[jj] = cs[jj] * g[jj];
        }
        return kc;
      };
      for (int j = 0; j < mm; ++j) {
        double *vj = V.p + (int64_t)j * ldv;
        const double *mz = precond(vj, z.p);
        op_apply(a, mz, w.p);
        {
          ProfScope ps(3);
          mdot2x(V.p, ldv, j + 1, vj, w.p, n, proj.p);
        }
        {
          ProfScope ps(6);
          d2h(hbuf.data(), proj.p, sizeof(double) * (2 * (j + 1)));
        }
        const int K = j + 1;
        const double uu_raw = hbuf[j], uw_raw = hbuf[K + j];
        const double bt = std::sqrt(uu_raw), sigma = 1.0 / bt;
        double ss = 0.0, st = 0.0;
        for (int i = 0; i < j; ++i) {
          sv[i] = sigma * hbuf[i];
          tv[i] = sigma * hbuf[K + i];
          ss += sv[i] * sv[i];
          st += sv[i] * tv[i];
        }
        const double a2 = sigma * sigma * uu_raw - ss;
        if (!(a2 > 0.0) || !(bt > 0.0)) {  // u_j in span(Q): breakdown
          // the step counts like the reference's (total is incremented before
          // its den == 0 test, krylov.py:110-119), so max_iter always ends the
          // loop even when the breakdown repeats at j = 0
          ++total;
          k = j;
          break;
        }
        const double alpha = std::sqrt(a2);
        if (j >= 1) {  // delayed correction of column j-1 (provisional h_{j,j-1} = bt)
          for (int i = 0; i < j; ++i) hr(i, j - 1) += bt * sv[i];
          hr(j, j - 1) = bt * alpha;
        }
        for (int i = 0; i <= j; ++i) {
          double c = 0.0;
          for (int q = 0; q < j; ++q) c += hr(i, q) * sv[q];
          cvec[i] = c;
        }
        const double qw = (sigma * sigma * uw_raw - st) / alpha;
        for (int i = 0; i < j; ++i) hr(i, j) = (tv[i] - cvec[i]) / alpha;
        hr(j, j) = (qw - cvec[j]) / alpha;
        const double gam = qw / alpha;
        for (int i = 0; i < j; ++i) {
          coef[i] = sv[i];
          coef[j + i] = tv[i] - gam * sv[i];
        }
        coef[2 * j] = sigma;
        coef[2 * j + 1] = 1.0 / alpha;
        coef[2 * j + 2] = gam;
        MG_CUDA(cudaMemcpyAsync(coefd.p, coef.data(), sizeof(double) * (2 * j + 3), cudaMemcpyHostToDevice,
                                stream()));
        {
          ProfScope ps(3);
          dcgs2_update(V.p, ldv, j, coefd.p, w.p, n, nrm_dev);
        }
        double nrm2v = 0.0;
        {
          ProfScope ps(6);
          d2h(&nrm2v, nrm_dev, sizeof(double));
        }
        const double hn = std::sqrt(nrm2v);
        hr(j + 1, j) = hn;  // provisional until the next step's reorthogonalisation
        ++total;
        k = j + 1;
        int kq = givens(k);
        if (kq < k) {
          k = kq;
          break;
        }
        bool happy = hn <= 1e-14 * std::max(res, 1.0);
        if (trace) fprintf(stderr, "[gmres] it %d |g| %.17g hn %.17g\n", total, std::fabs(g[j + 1]), hn);
        if (std::fabs(g[j + 1]) <= tol || happy || total >= o.max_iter) break;
        if (use_anorm && o.check_every && k % o.check_every == 0) {
          assemble(k, xt.p);
          op_apply(a, xt.p, t.p);
          vsub(r.p, b, t.p, n);
          double rt = nrm2(r.p, n);
          if (accepted(rt, nrm2(xt.p, n))) {
            early = true;
            early_res = rt;
            break;
          }
        }
      }
    } else
    for (int j = 0; j < mm; ++j) {
      double *vj = V.p + (int64_t)j * ldv;
      const double *mz = precond(vj, z.p);
      op_apply(a, mz, w.p);
      int K = j + 1;
      {
        ProfScope ps(3);
        mdot(V.p, ldv, K, w.p, n, c_dev);
        if (o.reorth) {
          update_mdot(V.p, ldv, K, c_dev, w.p, n, c2_dev);
          update_norm2(V.p, ldv, K, c2_dev, w.p, n, nrm_dev);
        } else {
          update_norm2(V.p, ldv, K, c_dev, w.p, n, nrm_dev);
        }
      }
      {
        ProfScope ps(6);
        d2h(hbuf.data(), proj.p, sizeof(double) * (2 * (mmax + 1) + 1));
      }
      for (int i = 0; i < K; ++i) h_at(i, j) = o.reorth ? hbuf[i] + hbuf[(mmax + 1) + i] : hbuf[i];
      double hn = std::sqrt(hbuf[2 * (mmax + 1)]);
      h_at(j + 1, j) = hn;
      ++total;
      k = j + 1;
      for (int i = 0; i < j; ++i) {
        double t = cs[i] * h_at(i, j) + sn[i] * h_at(i + 1, j);
        h_at(i + 1, j) = -sn[i] * h_at(i, j) + cs[i] * h_at(i + 1, j);
        h_at(i, j) = t;
      }
      double den = std::hypot(h_at(j, j), h_at(j + 1, j));
      if (den == 0.0) {
        k = j;
        break;
      }
      cs[j] = h_at(j, j) / den;
      sn[j] = h_at(j + 1, j) / den;
      h_at(j, j) = den;
      h_at(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      bool happy = hn <= 1e-14 * std::max(res, 1.0);
      if (trace) fprintf(stderr, "[gmres] it %d |g| %.17g hn %.17g\n", total, std::fabs(g[j + 1]), hn);
      if (std::fabs(g[j + 1]) <= tol || happy || total >= o.max_iter) break;
      if (use_anorm && o.check_every && k % o.check_every == 0) {
        assemble(k, xt.p);
        op_apply(a, xt.p, t.p);
        vsub(r.p, b, t.p, n);
        double rt = nrm2(r.p, n);
        if (accepted(rt, nrm2(xt.p, n))) {
          early = true;
          early_res = rt;
          break;
        }
      }
      vdiv_scalar(V.p + (int64_t)(j + 1) * ldv, w.p, hn, n);
    }
    ++out.cycles;
    if (out.first_cycle < 0) out.first_cycle = total;
    if (early) {
      vcopy(x, xt.p, n);
      out.iterations = total;
      out.converged = 1;
      out.residual_norm = early_res;
      return out;
    }
    assemble(k, x);
  }
}

}  // namespace mg
