// extern "C" boundary of libmgrgpu (declared in include/mgrgpu.h).
// Every entry point catches internal errors and maps them to a status code;
// nothing falls back to the CPU.
#include <memory>
#include "ops.cuh"
#include "solver.cuh"
#include "sparse_util.cuh"
#include "blockscale.cuh"
#include "amg_kernels.cuh"

using namespace mg;

struct mg_ctx { Ctx c; };
// `ready` is set while an asynchronous upload (mg_mat_upload_bsr_async) may
// still be in flight on the context's copy stream: the first use of the
// matrix orders the context stream after it (C() below).
struct mg_mat {
  Csr m;
  cudaEvent_t ready = nullptr;
  ~mg_mat() {
    if (ready) {  // never used: the copies land before the buffers (and the host arrays) are released
      cudaEventSynchronize(ready);
      cudaEventDestroy(ready);
    }
  }
};
struct mg_amg {
  Amg *h = nullptr;
  bool owned = true;
  ~mg_amg() { if (owned) delete h; }
};
struct mg_mgr { std::unique_ptr<Mgr> h; };
struct mg_ilu { std::unique_ptr<Ilu> f; };
namespace mg {
struct AsmGeo;
AsmGeo *asm_create(const mg_asm_desc &d);
void asm_destroy(AsmGeo *g);
void asm_assemble(AsmGeo &g, const double *p, const double *s, const double *r, const double *p_old,
                  const double *s_old, const double *r_old, double dt, double *res, int *active, Csr *jac);
}  // namespace mg
struct mg_asm {
  mg::AsmGeo *g = nullptr;
  int n = 0;
  ~mg_asm() { if (g) mg::asm_destroy(g); }
};

namespace {
struct Enter {
  Ctx *prev;
  explicit Enter(mg_ctx *ctx) : prev(g_ctx) {
    g_ctx = &ctx->c;
    cudaSetDevice(ctx->c.device);
  }
  ~Enter() { g_ctx = prev; }
};

template <class F>
int guard(mg_ctx *ctx, F &&f) {
  if (!ctx) return MG_ERR_BAD_OPTION;
  Enter e(ctx);
  ctx->c.err.clear();
  ctx->c.err_row = -1;
  try {
    f();
    return MG_OK;
  } catch (const MgError &err) {
    ctx->c.err = err.msg;
    ctx->c.err_row = err.row;
    return err.code;
  } catch (const std::exception &ex) {
    ctx->c.err = ex.what();
    return MG_ERR_CUDA;
  }
}

// input matrix of an API call: waits for a pending asynchronous upload
Csr &C(const mg_mat *x) {
  auto *m = const_cast<mg_mat *>(x);
  if (m->ready) {
    MG_CUDA(cudaStreamWaitEvent(stream(), m->ready, 0));
    cudaEventDestroy(m->ready);
    m->ready = nullptr;
  }
  return m->m;
}

Csr upload_csr(int nrows, int ncols, int b, const int32_t *indptr, const int32_t *indices, const double *vals) {
  if (nrows < 0 || ncols < 0) throw MgError(MG_ERR_BAD_OPTION, "negative dimension");
  int64_t nnz = indptr[nrows] - indptr[0];
  if (indptr[0] != 0) throw MgError(MG_ERR_BAD_OPTION, "indptr must start at 0");
  Csr m;
  m.alloc(nrows, ncols, nnz, b);
  h2d(m.rp.p, indptr, sizeof(int) * ((size_t)nrows + 1));
  h2d(m.ci.p, indices, sizeof(int) * (size_t)nnz);
  h2d(m.v.p, vals, sizeof(double) * (size_t)nnz * b * b);
  return m;
}

AmgOpts conv(const mg_amg_opts *o) {
  AmgOpts a;
  if (!o) return a;
  a.theta = o->strength_theta;
  a.max_levels = o->max_levels;
  a.cutoff = o->coarse_size_cutoff;
  a.pre = o->pre_sweeps;
  a.post = o->post_sweeps;
  a.cycles = o->cycles;
  a.max_elmts = o->max_elmts;
  a.seed = o->seed;
  if (!(a.theta > 0.0 && a.theta < 1.0)) throw MgError(MG_ERR_BAD_OPTION, "strength_theta must lie in (0, 1)");
  if (a.pre < 0 || a.post < 0) throw MgError(MG_ERR_BAD_OPTION, "sweep counts must be nonnegative");
  if (a.max_levels < 1 || a.cutoff < 1 || a.cycles < 1)
    throw MgError(MG_ERR_BAD_OPTION, "max_levels, coarse_size_cutoff and cycles must be >= 1");
  if (a.max_elmts < 0) throw MgError(MG_ERR_BAD_OPTION, "max_elmts must be >= 0");
  return a;
}

int64_t vec_len(const Csr &m) { return (int64_t)m.nr * m.b; }

struct DevVec {
  DBuf<double> b;
  DevVec(const double *host, int64_t n) : b((size_t)(n ? n : 1)) {
    if (host) h2d(b.p, host, sizeof(double) * n);
  }
};
}  // namespace

extern "C" {

int mg_ctx_create(int device, mg_ctx **out) {
  if (!out) return MG_ERR_BAD_OPTION;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return MG_ERR_CUDA;
  }
  if (device < 0 || device >= ndev) return MG_ERR_BAD_OPTION;
  auto *ctx = new mg_ctx();
  ctx->c.device = device;
  if (cudaSetDevice(device) != cudaSuccess) { delete ctx; return MG_ERR_CUDA; }
  if (cudaStreamCreateWithFlags(&ctx->c.stream, cudaStreamNonBlocking) != cudaSuccess) { delete ctx; return MG_ERR_CUDA; }
  cudaDeviceGetAttribute(&ctx->c.num_sms, cudaDevAttrMultiProcessorCount, device);
  // keep freed pool memory cached (stream-ordered allocator)
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  *out = ctx;
  return MG_OK;
}

int mg_ctx_destroy(mg_ctx *ctx) {
  if (!ctx) return MG_OK;
  {
    Enter e(ctx);
    cudaStreamSynchronize(ctx->c.stream);
    if (ctx->c.hbuf) cudaFreeHost(ctx->c.hbuf);
    if (ctx->c.copy_stream) {
      cudaStreamSynchronize(ctx->c.copy_stream);
      cudaStreamDestroy(ctx->c.copy_stream);
    }
    alloc_release_cache(&ctx->c);
    for (auto &kv : ctx->c.block_size)  // blocks still owned by live handles
      if (!alloc_in_slab(&ctx->c, kv.first)) cudaFree(kv.first);
    ctx->c.block_size.clear();
    alloc_release_slabs(&ctx->c);
    if (ctx->c.ev0) { cudaEventDestroy(ctx->c.ev0); cudaEventDestroy(ctx->c.ev1); }
    cudaStreamDestroy(ctx->c.stream);
  }
  delete ctx;
  return MG_OK;
}

const char *mg_last_error(mg_ctx *ctx) { return ctx ? ctx->c.err.c_str() : "null context"; }
int64_t mg_last_error_row(mg_ctx *ctx) { return ctx ? ctx->c.err_row : -1; }
int mg_ctx_sync(mg_ctx *ctx) { return guard(ctx, [&] { sync(); }); }
int64_t mg_ctx_launches(mg_ctx *ctx) { return ctx ? ctx->c.launches : 0; }
int64_t mg_ctx_device_bytes(mg_ctx *ctx) { return ctx ? ctx->c.dev_bytes : 0; }

int mg_mat_upload_csr(mg_ctx *ctx, int nrows, int ncols, const int32_t *indptr, const int32_t *indices,
                      const double *vals, mg_mat **out) {
  return guard(ctx, [&] {
    auto *m = new mg_mat();
    try { m->m = upload_csr(nrows, ncols, 1, indptr, indices, vals); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_mat_upload_bsr(mg_ctx *ctx, int nbrows, int nbcols, int b, const int32_t *rowptr, const int32_t *colind,
                      const double *vals, mg_mat **out) {
  return guard(ctx, [&] {
    if (b < 1 || b > 3) throw MgError(MG_ERR_UNSUPPORTED, "block size must be 1, 2 or 3");
    auto *m = new mg_mat();
    try { m->m = upload_csr(nbrows, nbcols, b, rowptr, colind, vals); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_mat_upload_csr_varmajor(mg_ctx *ctx, int n, int b, const int32_t *indptr, const int32_t *indices,
                               const double *vals, mg_mat **out) {
  return guard(ctx, [&] {
    if (b < 1 || b > 3) throw MgError(MG_ERR_UNSUPPORTED, "block size must be 1, 2 or 3");
    if (n < 0 || n % b) throw MgError(MG_ERR_DIM_MISMATCH, "variable-major matrix: n must be b * cells");
    Csr scalar = upload_csr(n, n, 1, indptr, indices, vals);
    auto *m = new mg_mat();
    try { m->m = csr_varmajor_to_bsr(scalar, b); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_mat_upload_bsr_async(mg_ctx *ctx, int nbrows, int nbcols, int b, const int32_t *rowptr,
                            const int32_t *colind, const double *vals, mg_mat **out) {
  return guard(ctx, [&] {
    if (b < 1 || b > 3) throw MgError(MG_ERR_UNSUPPORTED, "block size must be 1, 2 or 3");
    if (nbrows < 0 || nbcols < 0) throw MgError(MG_ERR_BAD_OPTION, "negative dimension");
    if (rowptr[0] != 0) throw MgError(MG_ERR_BAD_OPTION, "indptr must start at 0");
    int64_t nnz = rowptr[nbrows];
    Ctx &c = *g_ctx;
    if (!c.copy_stream) MG_CUDA(cudaStreamCreateWithFlags(&c.copy_stream, cudaStreamNonBlocking));
    auto *m = new mg_mat();
    try {
      m->m.alloc(nbrows, nbcols, nnz, b);
      // pool blocks may have been freed by work still queued on the context stream
      cudaEvent_t fork;
      MG_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
      MG_CUDA(cudaEventRecord(fork, c.stream));
      MG_CUDA(cudaStreamWaitEvent(c.copy_stream, fork, 0));
      cudaEventDestroy(fork);
      MG_CUDA(cudaMemcpyAsync(m->m.rp.p, rowptr, sizeof(int) * ((size_t)nbrows + 1), cudaMemcpyHostToDevice,
                              c.copy_stream));
      MG_CUDA(cudaMemcpyAsync(m->m.ci.p, colind, sizeof(int) * (size_t)nnz, cudaMemcpyHostToDevice, c.copy_stream));
      MG_CUDA(cudaMemcpyAsync(m->m.v.p, vals, sizeof(double) * (size_t)nnz * b * b, cudaMemcpyHostToDevice,
                              c.copy_stream));
      MG_CUDA(cudaEventCreateWithFlags(&m->ready, cudaEventDisableTiming));
      MG_CUDA(cudaEventRecord(m->ready, c.copy_stream));
    } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_mat_info(mg_ctx *ctx, const mg_mat *m, int *nrows, int *ncols, int64_t *nnz, int *b) {
  return guard(ctx, [&] {
    if (nrows) *nrows = C(m).nr;
    if (ncols) *ncols = C(m).nc;
    if (nnz) *nnz = C(m).nnz;
    if (b) *b = C(m).b;
  });
}

int mg_mat_download(mg_ctx *ctx, const mg_mat *m, int32_t *indptr, int32_t *indices, double *vals) {
  return guard(ctx, [&] {
    const Csr &c = C(m);
    if (indptr) d2h(indptr, c.rp.p, sizeof(int) * ((size_t)c.nr + 1));
    if (indices) d2h(indices, c.ci.p, sizeof(int) * (size_t)c.nnz);
    if (vals) d2h(vals, c.v.p, sizeof(double) * (size_t)c.nnz * c.b * c.b);
  });
}

int mg_mat_free(mg_ctx *ctx, mg_mat *m) {
  return guard(ctx, [&] { delete m; });
}

int mg_spmv(mg_ctx *ctx, const mg_mat *a, const double *x, double *y) {
  return guard(ctx, [&] {
    const Csr &c = C(a);
    DevVec dx(x, (int64_t)c.nc * c.b), dy(nullptr, vec_len(c));
    spmv(c, dx.b.p, dy.b.p);
    d2h(y, dy.b.p, sizeof(double) * vec_len(c));
  });
}

int mg_spmv_dev(mg_ctx *ctx, const mg_mat *a, const double *x_dev, double *y_dev) {
  return guard(ctx, [&] { spmv(C(a), x_dev, y_dev); });
}

int mg_spmv_layout(mg_ctx *ctx, const mg_mat *a, int *sell, int *index_bytes, int *sorted) {
  return guard(ctx, [&] {
    const Csr &c = C(a);
    prepare_spmv(c);
    if (sell) *sell = c.plan->sell ? 1 : 0;
    if (index_bytes) *index_bytes = c.plan->idx_bytes();
    if (sorted) *sorted = c.plan->perm.p ? 1 : 0;
  });
}

int mg_matmul(mg_ctx *ctx, const mg_mat *a, const mg_mat *b, mg_mat **out) {
  return guard(ctx, [&] {
    auto *m = new mg_mat();
    try { m->m = spgemm(C(a), C(b)); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_triple_product(mg_ctx *ctx, const mg_mat *r, const mg_mat *a, const mg_mat *p, mg_mat **out) {
  return guard(ctx, [&] {
    if (C(r).nc != C(a).nr || C(a).nc != C(p).nr)
      throw MgError(MG_ERR_DIM_MISMATCH, "triple_product: inner dimensions differ");
    Csr ap = spgemm(C(a), C(p), false);
    auto *m = new mg_mat();
    try { m->m = spgemm(C(r), ap, true, true); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_transpose(mg_ctx *ctx, const mg_mat *a, mg_mat **out) {
  return guard(ctx, [&] {
    auto *m = new mg_mat();
    try { m->m = transpose(C(a)); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_extract(mg_ctx *ctx, const mg_mat *a, const int64_t *rows, int nr, const int64_t *cols, int nc,
               mg_mat **out) {
  return guard(ctx, [&] {
    const Csr &c = C(a);
    if (c.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "extract: scalar CSR only");
    std::vector<int> hr(nr), cmap(c.nc, -1);
    for (int i = 0; i < nr; ++i) {
      if (rows[i] < 0 || rows[i] >= c.nr) throw MgError(MG_ERR_BAD_OPTION, "row index out of range");
      if (i && rows[i] <= rows[i - 1]) throw MgError(MG_ERR_BAD_OPTION, "row indices must be sorted and duplicate-free");
      hr[i] = (int)rows[i];
    }
    for (int j = 0; j < nc; ++j) {
      if (cols[j] < 0 || cols[j] >= c.nc) throw MgError(MG_ERR_BAD_OPTION, "column index out of range");
      if (j && cols[j] <= cols[j - 1]) throw MgError(MG_ERR_BAD_OPTION, "column indices must be sorted and duplicate-free");
      cmap[cols[j]] = j;
    }
    DBuf<int> dr((size_t)(nr ? nr : 1)), dm((size_t)(c.nc ? c.nc : 1));
    if (nr) h2d(dr.p, hr.data(), sizeof(int) * nr);
    if (c.nc) h2d(dm.p, cmap.data(), sizeof(int) * c.nc);
    auto *m = new mg_mat();
    try { m->m = extract(c, dr.p, nr, dm.p, nc); } catch (...) { delete m; throw; }
    *out = m;
  });
}

int mg_block_scale(mg_ctx *ctx, const mg_mat *a_bsr, int equilibrate, mg_mat **dinv_out, mg_mat **ahat_out) {
  return guard(ctx, [&] {
    auto d = std::make_unique<mg_mat>();
    auto ah = std::make_unique<mg_mat>();
    block_scale(C(a_bsr), d->m, ah->m, equilibrate != 0);
    *dinv_out = d.release();
    *ahat_out = ah.release();
  });
}

int mg_equilibrate(mg_ctx *ctx, const mg_mat *a, mg_mat **scaled_out, double *row_out, double *col_scale_out) {
  return guard(ctx, [&] {
    if (C(a).b != 1) throw MgError(MG_ERR_UNSUPPORTED, "equilibrate: scalar CSR required");
    int n = C(a).nr;
    DBuf<double> row((size_t)(n ? n : 1)), cs((size_t)(n ? n : 1));
    auto o = std::make_unique<mg_mat>();
    equilibrate(C(a), o->m, row.p, cs.p);
    if (row_out) d2h(row_out, row.p, sizeof(double) * n);
    if (col_scale_out) d2h(col_scale_out, cs.p, sizeof(double) * n);
    *scaled_out = o.release();
  });
}

int mg_abs_row_sum_max(mg_ctx *ctx, const mg_mat *a, double *out) {
  return guard(ctx, [&] { *out = abs_row_sum_max(C(a)); });
}

int mg_block_apply(mg_ctx *ctx, const mg_mat *dinv, const double *v, double *z) {
  return guard(ctx, [&] {
    int64_t n = vec_len(C(dinv));
    DevVec dv(v, n), dz(nullptr, n);
    block_apply(C(dinv), dv.b.p, dz.b.p);
    d2h(z, dz.b.p, sizeof(double) * n);
  });
}

int mg_build_rp(mg_ctx *ctx, const mg_mat *a, const uint8_t *f_mask, int kind, mg_mat **r_out, mg_mat **p_out) {
  return guard(ctx, [&] {
    const Csr &c = C(a);
    if (c.b != 1 || c.nr != c.nc) throw MgError(MG_ERR_DIM_MISMATCH, "build_rp: square scalar CSR required");
    if (kind < 0 || kind > 3) throw MgError(MG_ERR_BAD_OPTION, "unknown RpKind");
    int n = c.nr;
    DBuf<uint8_t> mask((size_t)(n ? n : 1));
    h2d(mask.p, f_mask, n);
    DBuf<int> flist, clist, fmap, cmap;
    int nf = 0, nc = 0;
    fc_split(mask.p, n, flist, clist, fmap, cmap, nf, nc);
    auto r = std::make_unique<mg_mat>();
    auto p = std::make_unique<mg_mat>();
    build_rp(c, fmap.p, cmap.p, flist.p, clist.p, nf, nc, kind, r->m, p->m);
    *r_out = r.release();
    *p_out = p.release();
  });
}

int mg_strength(mg_ctx *ctx, const mg_mat *a, double theta, int8_t *mask, int64_t *n_strong) {
  return guard(ctx, [&] {
    const Csr &m = C(a);
    if (m.b != 1) throw MgError(MG_ERR_UNSUPPORTED, "strength_graph: scalar CSR required");
    if (!(theta > 0.0 && theta < 1.0)) throw MgError(MG_ERR_BAD_OPTION, "strength_theta must lie in (0, 1)");
    DBuf<int8_t> s;
    const int64_t ns = strength(m, theta, s);
    if (m.nnz) d2h(mask, s.p, (size_t)m.nnz);
    if (n_strong) *n_strong = ns;
  });
}

int mg_amg_setup(mg_ctx *ctx, const mg_mat *a, const mg_amg_opts *opts, mg_amg **out) {
  return guard(ctx, [&] {
    auto h = std::make_unique<mg_amg>();
    h->h = amg_setup(C(a), conv(opts)).release();
    *out = h.release();
  });
}

int mg_amg_vcycle(mg_ctx *ctx, mg_amg *h, const double *b, const double *x0, double *x) {
  return guard(ctx, [&] {
    int64_t n = h->h->L[0].n;
    DevVec db(b, n), dx(x0, n);
    amg_vcycle(*h->h, db.b.p, x0 ? dx.b.p : nullptr, dx.b.p);
    d2h(x, dx.b.p, sizeof(double) * n);
  });
}

int mg_amg_apply(mg_ctx *ctx, mg_amg *h, const double *b, double *x) {
  return guard(ctx, [&] {
    int64_t n = h->h->L[0].n;
    DevVec db(b, n), dx(nullptr, n);
    amg_apply(*h->h, db.b.p, dx.b.p);
    d2h(x, dx.b.p, sizeof(double) * n);
  });
}

int mg_amg_nlevels(mg_ctx *ctx, const mg_amg *h, int *nlevels, int *has_row_sign) {
  return guard(ctx, [&] {
    if (nlevels) *nlevels = (int)h->h->L.size();
    if (has_row_sign) *has_row_sign = h->h->has_sign;
  });
}

int mg_amg_level_mat(mg_ctx *ctx, const mg_amg *h, int level, int what, mg_mat **out) {
  return guard(ctx, [&] {
    if (level < 0 || level >= (int)h->h->L.size()) throw MgError(MG_ERR_BAD_OPTION, "level out of range");
    const AmgLevel &l = h->h->L[level];
    const Csr *src = what == 0 ? &l.A : what == 1 ? &l.P : what == 3 ? &l.R : nullptr;
    if (!src) throw MgError(MG_ERR_BAD_OPTION, "unknown matrix selector");
    if (what != 0 && level + 1 == (int)h->h->L.size()) throw MgError(MG_ERR_BAD_OPTION, "coarsest level has no P");
    auto m = std::make_unique<mg_mat>();
    m->m = copy_csr(*src);
    *out = m.release();
  });
}

int mg_amg_splitting(mg_ctx *ctx, const mg_amg *h, int level, int8_t *state) {
  return guard(ctx, [&] {
    if (level < 0 || level + 1 >= (int)h->h->L.size()) throw MgError(MG_ERR_BAD_OPTION, "level has no splitting");
    const AmgLevel &l = h->h->L[level];
    d2h(state, l.split.p, (size_t)l.n);
  });
}

int mg_amg_row_sign(mg_ctx *ctx, const mg_amg *h, double *sign) {
  return guard(ctx, [&] {
    int n = h->h->L[0].n;
    if (h->h->has_sign) d2h(sign, h->h->sign.p, sizeof(double) * n);
    else for (int i = 0; i < n; ++i) sign[i] = 1.0;
  });
}

int mg_amg_free(mg_ctx *ctx, mg_amg *h) {
  return guard(ctx, [&] { delete h; });
}

int mg_mgr_setup(mg_ctx *ctx, const mg_mat *a, const mg_level_spec *plan, int nlevels, const mg_amg_opts *amg_opts,
                 int coarse_kind, int post_smoothing, const int64_t *cells, mg_mgr **out) {
  return guard(ctx, [&] {
    const Csr &c = C(a);
    std::vector<LevelSpec> specs;
    int n = c.nr;
    for (int k = 0; k < nlevels; ++k) {
      const mg_level_spec &s = plan[k];
      LevelSpec ls;
      ls.fmask.assign(s.f_mask, s.f_mask + n);
      ls.rp = s.rp_kind;
      ls.frelax = s.frelax_kind;
      ls.sweeps = s.frelax_sweeps;
      ls.pre = s.frelax_pre;
      ls.post = s.frelax_post;
      ls.max_levels = s.frelax_max_levels;
      ls.global_relax = s.global_relax;
      if (ls.rp < 0 || ls.rp > 3) throw MgError(MG_ERR_BAD_OPTION, "unknown RpKind");
      if (ls.frelax < 0 || ls.frelax > 3) throw MgError(MG_ERR_BAD_OPTION, "unknown F-relaxation");
      if (ls.sweeps < 1) throw MgError(MG_ERR_BAD_OPTION, "sweeps must be >= 1");
      int nf = 0;
      for (uint8_t m : ls.fmask) nf += m != 0;
      if (nf > 0 && nf < n) n -= nf;  // next level size
      specs.push_back(std::move(ls));
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, stream());
    auto h = std::make_unique<mg_mgr>();
    h->h = mgr_setup(c, specs, conv(amg_opts), coarse_kind, post_smoothing != 0, cells);
    cudaEventRecord(e1, stream());
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    g_ctx->timing.setup_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *out = h.release();
  });
}

int mg_mgr_set_prescale(mg_ctx *ctx, mg_mgr *h, const mg_mat *dinv) {
  return guard(ctx, [&] {
    if (vec_len(C(dinv)) != h->h->n0) throw MgError(MG_ERR_DIM_MISMATCH, "prescale dimension mismatch");
    h->h->prescale = copy_csr(C(dinv));
    h->h->has_prescale = true;
    h->h->drop_graph();
    h->h->pre_buf.alloc((size_t)h->h->n0);
  });
}

int mg_mgr_apply(mg_ctx *ctx, mg_mgr *h, const double *r, double *e) {
  return guard(ctx, [&] {
    int64_t n = h->h->n0;
    DevVec dr(r, n), de(nullptr, n);
    mgr_apply(*h->h, dr.b.p, de.b.p);
    d2h(e, de.b.p, sizeof(double) * n);
  });
}

int mg_mgr_apply_dev(mg_ctx *ctx, mg_mgr *h, const double *r_dev, double *e_dev) {
  return guard(ctx, [&] { mgr_apply(*h->h, r_dev, e_dev); });
}

int mg_mgr_nlevels(mg_ctx *ctx, const mg_mgr *h, int *nlevels) {
  return guard(ctx, [&] { *nlevels = (int)h->h->L.size(); });
}

int mg_mgr_level_mat(mg_ctx *ctx, const mg_mgr *h, int level, int what, mg_mat **out) {
  return guard(ctx, [&] {
    const Mgr &g = *h->h;
    if (level < 0 || level >= (int)g.L.size()) throw MgError(MG_ERR_BAD_OPTION, "level out of range");
    const MgrLevel &l = g.L[level];
    const Csr *src = nullptr;
    switch (what) {
      case 0: src = &l.A; break;
      case 1: src = &l.R; break;
      case 2: src = &l.P; break;
      case 3: src = level + 1 < (int)g.L.size() ? &g.L[level + 1].A : &g.coarse_A; break;
      case 4: src = &l.Aff; break;
      default: throw MgError(MG_ERR_BAD_OPTION, "unknown matrix selector");
    }
    auto m = std::make_unique<mg_mat>();
    m->m = copy_csr(*src);
    *out = m.release();
  });
}

int mg_mgr_level_amg(mg_ctx *ctx, const mg_mgr *h, int level, const mg_amg **out) {
  return guard(ctx, [&] {
    // borrowed view of the hierarchy's AMG; release it with mg_amg_free
    const Mgr &g = *h->h;
    Amg *p = nullptr;
    if (level < 0) p = g.camg.get();
    else if (level < (int)g.L.size()) p = g.L[level].fs.amg.get();
    if (!p) throw MgError(MG_ERR_BAD_OPTION, "no AMG hierarchy at that level");
    auto v = new mg_amg();
    v->h = p;
    v->owned = false;
    *out = v;
  });
}

int mg_mgr_free(mg_ctx *ctx, mg_mgr *h) {
  return guard(ctx, [&] { delete h; });
}

static int gmres_common(mg_ctx *ctx, const mg_mat *a, mg_mgr *m, const double *b_dev, double *x_dev,
                        const mg_gmres_opts *opts, double a_norm, mg_gmres_result *res, Ilu *ilu = nullptr) {
  GmresOpts o;
  if (opts) {
    o.rel_tol = opts->rel_tol;
    o.max_iter = opts->max_iter;
    o.restart = opts->restart;
    o.reorth = opts->reorthogonalize;
    o.check_every = opts->check_every;
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  prof_reset();
  cudaEventRecord(e0, stream());
  GmresOut out = gmres(C(a), m ? m->h.get() : nullptr, b_dev, x_dev, o, a_norm, ilu);
  cudaEventRecord(e1, stream());
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  prof_collect();
  g_ctx->timing.solve_ms = ms;
  g_ctx->timing.spmv_bytes = C(a).bytes_spmv();
  g_ctx->timing.vcycle_bytes = (m && m->h->camg) ? m->h->camg->cycle_bytes() : 0.0;
  g_ctx->timing.k0_bytes = (m && m->h->camg) ? m->h->camg->k0_bytes() : 0.0;
  res->iterations = out.iterations;
  res->converged = out.converged;
  res->residual_norm = out.residual_norm;
  res->rhs_norm = out.rhs_norm;
  res->cycles = out.cycles;
  res->first_cycle_iterations = out.first_cycle;
  return MG_OK;
}

int mg_gmres(mg_ctx *ctx, const mg_mat *a, mg_mgr *m, const double *b, double *x, const mg_gmres_opts *opts,
             double a_norm, mg_gmres_result *res) {
  return guard(ctx, [&] {
    int64_t n = vec_len(C(a));
    DevVec db(b, n), dx(nullptr, n);
    gmres_common(ctx, a, m, db.b.p, dx.b.p, opts, a_norm, res);
    d2h(x, dx.b.p, sizeof(double) * n);
  });
}

int mg_gmres_dev(mg_ctx *ctx, const mg_mat *a, mg_mgr *m, const double *b_dev, double *x_dev,
                 const mg_gmres_opts *opts, double a_norm, mg_gmres_result *res) {
  return guard(ctx, [&] { gmres_common(ctx, a, m, b_dev, x_dev, opts, a_norm, res); });
}

int mg_gmres_ilu(mg_ctx *ctx, const mg_mat *a, mg_ilu *f, const double *b, double *x, const mg_gmres_opts *opts,
                 double a_norm, mg_gmres_result *out) {
  return guard(ctx, [&] {
    int64_t n = vec_len(C(a));
    DevVec db(b, n), dx(nullptr, n);
    gmres_common(ctx, a, nullptr, db.b.p, dx.b.p, opts, a_norm, out, f ? f->f.get() : nullptr);
    d2h(x, dx.b.p, sizeof(double) * n);
  });
}

int mg_ilu_factor(mg_ctx *ctx, const mg_mat *a, int level, mg_ilu **out) {
  return guard(ctx, [&] {
    auto h = std::make_unique<mg_ilu>();
    h->f = ilu_factor(C(a), level);
    *out = h.release();
  });
}

int mg_ilu_matrix(mg_ctx *ctx, const mg_ilu *f, mg_mat **out) {
  return guard(ctx, [&] {
    auto m = std::make_unique<mg_mat>();
    m->m = copy_csr(f->f->LU);
    *out = m.release();
  });
}

int mg_ilu_apply(mg_ctx *ctx, mg_ilu *f, const double *r, double *x) {
  return guard(ctx, [&] {
    int64_t n = f->f->n;
    DevVec dr(r, n), dx(nullptr, n);
    ilu_apply(*f->f, dr.b.p, dx.b.p);
    d2h(x, dx.b.p, sizeof(double) * n);
  });
}

int mg_ilu_free(mg_ctx *ctx, mg_ilu *f) {
  return guard(ctx, [&] { delete f; });
}

int mg_asm_create(mg_ctx *ctx, const mg_asm_desc *d, mg_asm **out) {
  return guard(ctx, [&] {
    if (!d || d->n_cells <= 0) throw MgError(MG_ERR_BAD_OPTION, "assembly: empty problem");
    auto h = std::make_unique<mg_asm>();
    h->g = asm_create(*d);
    h->n = d->n_cells;
    *out = h.release();
  });
}

int mg_asm_assemble(mg_ctx *ctx, mg_asm *a, const double *p, const double *s, const double *rho,
                    const double *p_old, const double *s_old, const double *rho_old, double dt, double *res,
                    int *active, mg_mat **jac_out) {
  return guard(ctx, [&] {
    const int n = a->n;
    DevVec dp(p, n), ds(s, n), dr(rho, n), dpo(p_old, n), dso(s_old, n), dro(rho_old, n), dres(nullptr, 3 * (int64_t)n);
    DBuf<int> dact(n);
    std::unique_ptr<mg_mat> m;
    if (jac_out) m = std::make_unique<mg_mat>();
    asm_assemble(*a->g, dp.b.p, ds.b.p, dr.b.p, dpo.b.p, dso.b.p, dro.b.p, dt, dres.b.p, dact.p,
                 m ? &m->m : nullptr);
    if (res) d2h(res, dres.b.p, sizeof(double) * 3 * (size_t)n);
    if (active) d2h(active, dact.p, sizeof(int) * (size_t)n);
    if (jac_out) *jac_out = m.release();
  });
}

int mg_asm_free(mg_ctx *ctx, mg_asm *a) {
  return guard(ctx, [&] { delete a; });
}

int mg_dev_alloc(mg_ctx *ctx, int64_t bytes, void **out) {
  return guard(ctx, [&] {
    void *p = nullptr;
    MG_CUDA(cudaMalloc(&p, (size_t)bytes));
    *out = p;
  });
}
int mg_dev_free(mg_ctx *ctx, void *p) {
  return guard(ctx, [&] { MG_CUDA(cudaFree(p)); });
}
int mg_memcpy_h2d(mg_ctx *ctx, void *dst, const void *src, int64_t bytes) {
  return guard(ctx, [&] { h2d(dst, src, (size_t)bytes); });
}
int mg_memcpy_d2h(mg_ctx *ctx, void *dst, const void *src, int64_t bytes) {
  return guard(ctx, [&] { d2h(dst, src, (size_t)bytes); });
}

int mg_timer_start(mg_ctx *ctx) {
  return guard(ctx, [&] {
    if (!ctx->c.ev0) {
      MG_CUDA(cudaEventCreate(&ctx->c.ev0));
      MG_CUDA(cudaEventCreate(&ctx->c.ev1));
    }
    MG_CUDA(cudaEventRecord(ctx->c.ev0, stream()));
  });
}

int mg_timer_stop(mg_ctx *ctx, double *ms) {
  return guard(ctx, [&] {
    if (!ctx->c.ev0) throw MgError(MG_ERR_BAD_OPTION, "mg_timer_start was not called");
    MG_CUDA(cudaEventRecord(ctx->c.ev1, stream()));
    MG_CUDA(cudaEventSynchronize(ctx->c.ev1));
    float f = 0.f;
    MG_CUDA(cudaEventElapsedTime(&f, ctx->c.ev0, ctx->c.ev1));
    *ms = f;
  });
}

int mg_get_timing(mg_ctx *ctx, mg_timing *t) {
  if (!ctx || !t) return MG_ERR_BAD_OPTION;
  *t = ctx->c.timing;
  return MG_OK;
}
int mg_set_profiling(mg_ctx *ctx, int on) {
  if (!ctx) return MG_ERR_BAD_OPTION;
  ctx->c.profiling = on;
  return MG_OK;
}

}  // extern "C"
