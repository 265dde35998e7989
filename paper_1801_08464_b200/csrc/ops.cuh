// Host-side launchers shared across translation units.
#pragma once
#include "common.cuh"

namespace mg {

// ---- SpMV family (spmv.cu) --------------------------------------------------
// bin rows by length class once (syncs); done at setup for solve-phase matrices
void prepare_spmv(const Csr &a);
// y = A x
void spmv(const Csr &a, const double *x, double *y);
// r = b - A x
void residual(const Csr &a, const double *x, const double *b, double *r);
// y = y + A x
void spmv_add(const Csr &a, const double *x, double *y);
// y = [ef scattered by fmap (fmap[i] < 0: 0)] + A x
void spmv_merge_add(const Csr &a, const double *x, const int *fmap, const double *ef, double *y);
// y = A x; bs = sign .* y (when sign); xo = d .* (bs or y): a restriction fused with
// the coarser AMG level's first pre-sweep from zero (x = D^-1 b)
void spmv_store_scale(const Csr &a, const double *x, double *y, const double *sign, double *bs, const double *d,
                      double *xo);
// xo = x + dinv .* (b - A x)   (L1-Jacobi sweep)
void jacobi_sweep(const Csr &a, const double *x, const double *b, const double *dinv, double *xo);

// ---- vectors (blas.cu) ------------------------------------------------------
void vfill(double *x, double val, int64_t n);
void vcopy(double *dst, const double *src, int64_t n);
void vmul(double *y, const double *a, const double *x, int64_t n);          // y = a .* x
void vaxpy(double *y, double a, const double *x, int64_t n);                // y += a x
void vadd(double *y, const double *x, int64_t n);                           // y += x
void vdiv_scalar(double *y, const double *x, double d, int64_t n);          // y = x / d
void vsub(double *r, const double *b, const double *ax, int64_t n);         // r = b - ax
void gather(double *dst, const double *src, const int *idx, int64_t n);     // dst[i] = src[idx[i]]
void scatter_add(double *dst, const double *src, const int *idx, int64_t n);// dst[idx[i]] += src[i]
// dst = src[idx]; bs = sign .* dst (when sign); xo = d .* (bs or dst)
// y = b[rows] - A x for a row-extracted operator A (rows = the source rows), plus the
// EpiStoreScale outputs when xo is given (xo = d .* (sign .* y))
void residual_rows_scale(const Csr &a, const double *x, const double *b, const int *rows, double *y,
                         const double *sign, double *bs, const double *d, double *xo);
void gather_scale(double *dst, const double *src, const int *idx, int64_t n, const double *sign, double *bs,
                  const double *d, double *xo);
void scatter_set(double *dst, const double *src, const int *idx, int64_t n);// dst[idx[i]] = src[i]
// e[i] = fmap[i] >= 0 ? ef[fmap[i]] : 0   (F values into a zeroed full vector, one pass)
void fc_merge(double *e, const double *ef, const int *fmap, int64_t n);
// deterministic reductions; result left in device memory `out` (and returned when host=true)
double dot(const double *x, const double *y, int64_t n);
double nrm2(const double *x, int64_t n);
// CGS2 pieces on the basis V (row stride ldv), k0..k0+K-1 vectors
void mdot(const double *V, int64_t ldv, int K, const double *w, int64_t n, double *out_dev);
// w -= sum_k c[k] V_k ; out = V^T w (fused second projection)
void update_mdot(const double *V, int64_t ldv, int K, const double *c_dev, double *w, int64_t n,
                 double *out_dev);
// w -= sum_k c[k] V_k ; out[0] = ||w||^2
void update_norm2(const double *V, int64_t ldv, int K, const double *c_dev, double *w, int64_t n,
                  double *out_dev);
// DCGS2 (one reduction per Arnoldi step, delayed reorthogonalisation):
// out = [V^T u (K), V^T w (K)], K <= 32
void mdot2x(const double *V, int64_t ldv, int K, const double *u, const double *w, int64_t n, double *out_dev);
// V[j] = (sigma V[j] - Q s)/alpha; V[j+1] = (sigma w - Q e - gamma sigma V[j])/alpha; norm2 = ||V[j+1]||^2
// coef = [s (j), e (j), sigma, 1/alpha, gamma], j <= 32
void dcgs2_update(double *V, int64_t ldv, int j, const double *coef_dev, const double *w, int64_t n,
                  double *norm2_dev);
// u = sum_k y[k] V_k
void combine(const double *V, int64_t ldv, int K, const double *y_dev, double *u, int64_t n);

// ---- dense (dense.cu) -------------------------------------------------------
// explicit inverse of an n x n row-major matrix (Gauss-Jordan, partial pivot);
// returns -1 on success else the elimination step with a zero pivot
int dense_inverse(const double *a_dev, double *inv_dev, int n);
// y = Ainv b  (dense n x n)
void dense_matvec(const double *m_dev, const double *x, double *y, int n);

}  // namespace mg
