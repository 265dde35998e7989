// MGR transfer operators: F/C split maps and build_rp (mgr.py:117-156).
//
//   P = [W_p; I] (n x nc),  R = [W_r, I] (nc x n), original indexing,
//   W_p = -((1/d_f) * A_fc)  (dia @ csr: product then negation, zeros dropped)
//   W_r = -(A_cf * (1/d_f))  (csr @ dia), only for NONINJECTIVE
//   INJECTION: W_p = W_r = 0;  IDEAL: W_p = -A_ff^-1 A_fc, W_r = -A_cf A_ff^-1
// The D_ff zero check runs for every non-IDEAL kind, INJECTION included, and
// reports the original row, as the reference does (mgr.py:132-135).
#include "ops.cuh"
#include "solver.cuh"
#include "sparse_util.cuh"
#include "amg_kernels.cuh"

namespace mg {

__global__ void k_fc_flags(int n, const uint8_t *m, int *ff, int *cf) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) { ff[i] = m[i] != 0; cf[i] = m[i] == 0; }
}
__global__ void k_fc_maps(int n, const uint8_t *m, const int *fs, const int *cs, int *fmap, int *cmap,
                          int *flist, int *clist) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (m[i]) { fmap[i] = fs[i]; cmap[i] = -1; flist[fs[i]] = i; }
  else { cmap[i] = cs[i]; fmap[i] = -1; clist[cs[i]] = i; }
}

void fc_split(const uint8_t *fmask_dev, int n, DBuf<int> &flist, DBuf<int> &clist, DBuf<int> &fmap,
              DBuf<int> &cmap, int &nf, int &nc) {
  DBuf<int> ff(n), cf(n), fs((size_t)n + 1), cs((size_t)n + 1);
  k_fc_flags<<<grid_for(n, 256), 256, 0, stream()>>>(n, fmask_dev, ff.p, cf.p);
  check_launch("fc_flags");
  nf = (int)exclusive_scan_i32_to_i32(ff.p, fs.p, n);
  nc = (int)exclusive_scan_i32_to_i32(cf.p, cs.p, n);
  flist.alloc((size_t)(nf ? nf : 1));
  clist.alloc((size_t)(nc ? nc : 1));
  fmap.alloc(n);
  cmap.alloc(n);
  k_fc_maps<<<grid_for(n, 256), 256, 0, stream()>>>(n, fmask_dev, fs.p, cs.p, fmap.p, cmap.p, flist.p, clist.p);
  check_launch("fc_maps");
}

__global__ void k_fdiag_check(int nf, const int *flist, const double *d, int *bad) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nf && d[flist[i]] == 0.0) atomicMin(bad, flist[i]);
}

// P rows (thread per row).  mode 0 count / 1 fill
__global__ void k_p_rows(int n, const int *rp, const int *ci, const double *v, const double *d,
                         const int *cmap, int kind, int mode, int *cnt, const int *orp, int *oci, double *ov) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int c = 0;
  int o = mode ? orp[i] : 0;
  if (cmap[i] >= 0) {
    if (mode) { oci[o] = cmap[i]; ov[o] = 1.0; }
    c = 1;
  } else if (kind != RP_INJECTION) {
    double inv = __ddiv_rn(1.0, d[i]);
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      int cj = cmap[ci[q]];
      if (cj < 0) continue;
      double val = __dmul_rn(inv, v[q]);
      if (val == 0.0) continue;
      if (mode) { oci[o + c] = cj; ov[o + c] = -val; }
      ++c;
    }
  }
  if (!mode) cnt[i] = c;
}

// R rows (thread per coarse row); F columns kept in original indexing
__global__ void k_r_rows(int nc, const int *clist, const int *rp, const int *ci, const double *v,
                         const double *d, const int *fmap, int kind, int mode, int *cnt, const int *orp,
                         int *oci, double *ov) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= nc) return;
  int i = clist[c];
  int o = mode ? orp[c] : 0;
  int k = 0;
  bool ident = false;
  if (kind == RP_NONINJECTIVE) {
    for (int q = rp[i]; q < rp[i + 1]; ++q) {
      int j = ci[q];
      if (!ident && j > i) {
        if (mode) { oci[o + k] = i; ov[o + k] = 1.0; }
        ++k;
        ident = true;
      }
      if (fmap[j] < 0) continue;
      double val = __dmul_rn(v[q], __ddiv_rn(1.0, d[j]));
      if (val == 0.0) continue;
      if (mode) { oci[o + k] = j; ov[o + k] = -val; }
      ++k;
    }
  }
  if (!ident) {
    if (mode) { oci[o + k] = i; ov[o + k] = 1.0; }
    ++k;
  }
  if (!mode) cnt[c] = k;
}

// ---- dense helpers for RpKind.IDEAL (test sizes) -------------------------------
__global__ void k_dense_mm(int m, int k, int n, const double *a, const double *b, double *c, double alpha) {
  int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (int64_t)m * n) return;
  int i = (int)(t / n), j = (int)(t % n);
  double s = 0.0;
  for (int q = 0; q < k; ++q) s += a[(int64_t)i * k + q] * b[(int64_t)q * n + j];
  c[t] = alpha * s;
}
// sparse rows from dense W (row r of the output gets the nonzeros of W row wr, columns mapped by colmap)
__global__ void k_dense_rows(int nrows, int wcols, const double *w, const int *colmap, const int *is_w_row,
                             const int *wrow, const int *ident_col, int mode, int *cnt, const int *orp,
                             int *oci, double *ov) {
  int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nrows) return;
  int k = 0, o = mode ? orp[r] : 0;
  if (is_w_row[r]) {
    const double *wr = w + (int64_t)wrow[r] * wcols;
    // columns colmap[j] ascending in j; identity column (if any) merged in order
    int ic = ident_col[r];
    bool done = ic < 0;
    for (int j = 0; j < wcols; ++j) {
      int col = colmap[j];
      if (!done && ic < col) { if (mode) { oci[o + k] = ic; ov[o + k] = 1.0; } ++k; done = true; }
      if (wr[j] != 0.0) { if (mode) { oci[o + k] = col; ov[o + k] = wr[j]; } ++k; }
    }
    if (!done) { if (mode) { oci[o + k] = ic; ov[o + k] = 1.0; } ++k; }
  } else {
    if (mode) { oci[o] = ident_col[r]; ov[o] = 1.0; }
    k = 1;
  }
  if (!mode) cnt[r] = k;
}

static Csr rows_from_dense(int nrows, int ncols, int wcols, const double *w, const int *colmap,
                           const int *is_w_row, const int *wrow, const int *ident_col) {
  Csr out;
  out.nr = nrows;
  out.nc = ncols;
  out.rp.alloc((size_t)nrows + 1);
  DBuf<int> cnt((size_t)(nrows ? nrows : 1));
  k_dense_rows<<<grid_for(nrows, 128), 128, 0, stream()>>>(nrows, wcols, w, colmap, is_w_row, wrow, ident_col, 0,
                                                           cnt.p, nullptr, nullptr, nullptr);
  check_launch("dense_rows");
  out.nnz = exclusive_scan_i32_to_i32(cnt.p, out.rp.p, nrows);
  out.ci.alloc((size_t)out.nnz);
  out.v.alloc((size_t)out.nnz);
  k_dense_rows<<<grid_for(nrows, 128), 128, 0, stream()>>>(nrows, wcols, w, colmap, is_w_row, wrow, ident_col, 1,
                                                           nullptr, out.rp.p, out.ci.p, out.v.p);
  check_launch("dense_rows");
  return out;
}

__global__ void k_ideal_maps(int n, const int *fmap, const int *cmap, int *p_isw, int *p_wrow, int *p_ident) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  p_isw[i] = fmap[i] >= 0;
  p_wrow[i] = fmap[i] >= 0 ? fmap[i] : 0;
  p_ident[i] = fmap[i] >= 0 ? -1 : cmap[i];
}
__global__ void k_iota_i(int *a, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = i;
}
__global__ void k_ones_i(int *a, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) a[i] = 1;
}

static void build_rp_ideal(const Csr &a, const int *fmap, const int *cmap, const int *flist, const int *clist,
                           int nf, int nc, Csr &r, Csr &p) {
  const int LIM = 8192;
  if (nf > LIM || nc > 4 * LIM)
    throw MgError(MG_ERR_UNSUPPORTED, "RpKind.IDEAL on the GPU is limited to nf <= 8192 (dense A_ff^-1)");
  int n = a.nr;
  Csr aff = extract(a, flist, nf, fmap, nf);
  Csr afc = extract(a, flist, nf, cmap, nc);
  Csr acf = extract(a, clist, nc, fmap, nf);
  DBuf<double> dff((size_t)nf * nf), inv((size_t)nf * nf), dfc((size_t)nf * nc), dcf((size_t)nc * nf);
  DBuf<double> wp((size_t)nf * nc), wr((size_t)nc * nf);
  to_dense(aff, dff.p);
  to_dense(afc, dfc.p);
  to_dense(acf, dcf.p);
  int bad = dense_inverse(dff.p, inv.p, nf);
  if (bad >= 0) throw MgError(MG_ERR_SINGULAR, "A_ff is singular (IDEAL reduction)", bad);
  k_dense_mm<<<grid_for((int64_t)nf * nc, 128), 128, 0, stream()>>>(nf, nf, nc, inv.p, dfc.p, wp.p, -1.0);
  check_launch("dense_mm");
  k_dense_mm<<<grid_for((int64_t)nc * nf, 128), 128, 0, stream()>>>(nc, nf, nf, dcf.p, inv.p, wr.p, -1.0);
  check_launch("dense_mm");
  // P: n rows; F rows from W_p (columns 0..nc-1), C rows identity at cmap
  DBuf<int> isw(n), wrow(n), ident(n), pcols((size_t)nc + 1);
  k_ideal_maps<<<grid_for(n, 256), 256, 0, stream()>>>(n, fmap, cmap, isw.p, wrow.p, ident.p);
  check_launch("ideal_maps");
  k_iota_i<<<grid_for(nc, 256), 256, 0, stream()>>>(pcols.p, nc);
  check_launch("iota");
  p = rows_from_dense(n, nc, nc, wp.p, pcols.p, isw.p, wrow.p, ident.p);
  // R: nc rows; W_r row c over F columns (flist) + identity at clist[c]
  DBuf<int> risw((size_t)nc + 1), rwrow((size_t)nc + 1);
  k_ones_i<<<grid_for(nc, 256), 256, 0, stream()>>>(risw.p, nc);
  k_iota_i<<<grid_for(nc, 256), 256, 0, stream()>>>(rwrow.p, nc);
  check_launch("ideal_r_maps");
  r = rows_from_dense(nc, n, nf, wr.p, flist, risw.p, rwrow.p, clist);
}

void build_rp(const Csr &a, const int *fmap, const int *cmap, const int *flist, const int *clist, int nf, int nc,
              int kind, Csr &r, Csr &p) {
  int n = a.nr;
  if (nf == 0 || nc == 0) throw MgError(MG_ERR_BAD_OPTION, "both F and C sets must be nonempty");
  if (kind == RP_IDEAL) {
    build_rp_ideal(a, fmap, cmap, flist, clist, nf, nc, r, p);
    return;
  }
  DBuf<double> d(n);
  row_diag(a, d.p);
  DBuf<int> bad(1);
  const int big = 0x7fffffff;
  dset_i32(bad.p, {big});
  k_fdiag_check<<<grid_for(nf, 256), 256, 0, stream()>>>(nf, flist, d.p, bad.p);
  check_launch("fdiag_check");
  int hb = 0;
  d2h(&hb, bad.p, sizeof(int));
  if (hb != big) throw MgError(MG_ERR_ZERO_F_DIAG, "zero diagonal in A_ff at fine row " + std::to_string(hb), hb);
  // P
  p.nr = n;
  p.nc = nc;
  p.b = 1;
  p.rp.alloc((size_t)n + 1);
  DBuf<int> cnt((size_t)n + 1);
  k_p_rows<<<grid_for(n, 128), 128, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, d.p, cmap, kind, 0, cnt.p, nullptr,
                                                   nullptr, nullptr);
  check_launch("p_rows");
  p.nnz = exclusive_scan_i32_to_i32(cnt.p, p.rp.p, n);
  p.ci.alloc((size_t)p.nnz);
  p.v.alloc((size_t)p.nnz);
  k_p_rows<<<grid_for(n, 128), 128, 0, stream()>>>(n, a.rp.p, a.ci.p, a.v.p, d.p, cmap, kind, 1, nullptr, p.rp.p,
                                                   p.ci.p, p.v.p);
  check_launch("p_rows");
  // R
  r.nr = nc;
  r.nc = n;
  r.b = 1;
  r.rp.alloc((size_t)nc + 1);
  k_r_rows<<<grid_for(nc, 128), 128, 0, stream()>>>(nc, clist, a.rp.p, a.ci.p, a.v.p, d.p, fmap, kind, 0, cnt.p,
                                                    nullptr, nullptr, nullptr);
  check_launch("r_rows");
  r.nnz = exclusive_scan_i32_to_i32(cnt.p, r.rp.p, nc);
  r.ci.alloc((size_t)r.nnz);
  r.v.alloc((size_t)r.nnz);
  k_r_rows<<<grid_for(nc, 128), 128, 0, stream()>>>(nc, clist, a.rp.p, a.ci.p, a.v.p, d.p, fmap, kind, 1, nullptr,
                                                    r.rp.p, r.ci.p, r.v.p);
  check_launch("r_rows");
}

}  // namespace mg
