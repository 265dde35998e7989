/*
 * mgrgpu.h — C-ABI of the B200-native MGR-GMRES library (libmgrgpu.so).
 *
 * Plain C types only (no torch / CUDA types in the signatures).  Every call
 * returns an int status (MG_OK = 0); on error the message is available from
 * mg_last_error(ctx) and, for MG_ERR_ZERO_F_DIAG, the offending row from
 * mg_last_error_row(ctx).  Host pointers are caller-owned and copied; the
 * library owns all device memory behind the opaque handles.  One context per
 * host thread; calls are stream-ordered on the context's stream and
 * synchronous at the ABI unless they take device pointers (suffix _dev).
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/ncpflow/...); the Python host side
 * (paper_1801_08464_b200/) binds them with ctypes behind the reference's own
 * function names, so ncpflow callers switch by import.
 */
#ifndef MGRGPU_H
#define MGRGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes; the Python side maps them to the reference's exception types */
enum {
  MG_OK = 0,
  MG_ERR_ZERO_F_DIAG = 1,   /* ncpflow.mgr.ZeroFDiagonal(row)   mgr.py:41-44,132-135   */
  MG_ERR_AMG_SETUP = 2,     /* ncpflow.amg.AmgSetupError        amg.py:27-28           */
  MG_ERR_DIM_MISMATCH = 3,  /* ncpflow.sparse.DimensionMismatch sparse.py:18-19        */
  MG_ERR_BAD_OPTION = 4,    /* ValueError (bad options / empty F or C sets) mgr.py:121  */
  MG_ERR_CUDA = 5,          /* CUDA runtime failure (no silent fallback)               */
  MG_ERR_SINGULAR = 6,      /* ncpflow.sparse.SingularMatrixError sparse.py:22-28      */
  MG_ERR_UNSUPPORTED = 7,   /* feature not available on the GPU path                    */
  MG_ERR_ZERO_PIVOT = 8     /* ncpflow.ilu.ZeroPivot(row)        ilu.py:24-27,131-140   */
};

typedef struct mg_ctx mg_ctx;
typedef struct mg_mat mg_mat;   /* CSR (b == 1) or block-CSR (b = 2, 3) matrix */
typedef struct mg_amg mg_amg;   /* AMG hierarchy  (ncpflow.amg.AmgHierarchy)   */
typedef struct mg_mgr mg_mgr;   /* MGR hierarchy  (ncpflow.mgr.MgrHierarchy)   */

/* ---- context ------------------------------------------------------------ */
int mg_ctx_create(int device, mg_ctx **out);
int mg_ctx_destroy(mg_ctx *ctx);
const char *mg_last_error(mg_ctx *ctx);
int64_t mg_last_error_row(mg_ctx *ctx);
int mg_ctx_sync(mg_ctx *ctx);
/* count of this library's kernel launches since creation (bench gpu_launches) */
int64_t mg_ctx_launches(mg_ctx *ctx);
/* device memory currently held by the library (bytes) */
int64_t mg_ctx_device_bytes(mg_ctx *ctx);

/* ---- matrices (ncpflow.sparse.CsrMatrix, sparse.py:35-143) ---------------- */
/* scalar CSR, sorted column indices, int32 indices, f64 values */
int mg_mat_upload_csr(mg_ctx *ctx, int nrows, int ncols, const int32_t *indptr,
                      const int32_t *indices, const double *vals, mg_mat **out);
/* block CSR: nbrows block rows, b x b row-major blocks, sorted block columns */
int mg_mat_upload_bsr(mg_ctx *ctx, int nbrows, int nbcols, int b, const int32_t *rowptr,
                      const int32_t *colind, const double *vals, mg_mat **out);
/* the reference's BlockSystem matrix (assembly.py:95-120: scalar CSR over the
   variable-major unknowns u = var * N + cell, N = n / b) converted on the device
   into the cell-major b x b block CSR the block kernels use (SURVEY.md §8(b)
   mat_upload_csr_varmajor); block positions no entry fills are explicit zeros.
   Vectors for it are cell-major: x_cell[cell * b + var] = x_var[var * N + cell]. */
int mg_mat_upload_csr_varmajor(mg_ctx *ctx, int n, int b, const int32_t *indptr, const int32_t *indices,
                               const double *vals, mg_mat **out);
/* mg_mat_upload_bsr without the host wait: the copies run on the context's
   copy stream and overlap whatever the context is computing; the first call
   that uses the matrix (or mg_mat_free) orders the context stream after them.
   The host arrays must stay valid and unmodified until the context has
   synchronised after that first use (any call returning a host result, or
   mg_ctx_sync) or mg_mat_free has returned, and must be
   pinned for the copies to be asynchronous (pageable memory still works, the
   driver then stages it synchronously).  Lets a caller upload time step k+1's
   Jacobian while step k is being solved. */
int mg_mat_upload_bsr_async(mg_ctx *ctx, int nbrows, int nbcols, int b, const int32_t *rowptr,
                            const int32_t *colind, const double *vals, mg_mat **out);
/* nrows/ncols are scalar dims for CSR and block dims for BSR */
int mg_mat_info(mg_ctx *ctx, const mg_mat *m, int *nrows, int *ncols, int64_t *nnz, int *b);
int mg_mat_download(mg_ctx *ctx, const mg_mat *m, int32_t *indptr, int32_t *indices,
                    double *vals);
int mg_mat_free(mg_ctx *ctx, mg_mat *m);

/* ---- sparse kernels ------------------------------------------------------- */
/* y = A x (sparse.py:174-178 spmv; the GMRES operator `a @ v`, linsolve.py:100) */
int mg_spmv(mg_ctx *ctx, const mg_mat *a, const double *x, double *y);
int mg_spmv_dev(mg_ctx *ctx, const mg_mat *a, const double *x_dev, double *y_dev);
/* Solve-phase layout the SpMV kernels use for `a` (built on first use; no
   reference counterpart, the layout is an implementation detail exposed for
   tests and profiling): *sell = 1 for a SELL-32 copy, 0 for plain CSR/BSR;
   *index_bytes = stored bytes per column index (4 int32; 2 / 1 for the
   lossless int16 / u8-dictionary column codes of large stencil-like operators);
   *sorted = 1 when the SELL rows are length-sorted inside windows (SELL-C-sigma) */
int mg_spmv_layout(mg_ctx *ctx, const mg_mat *a, int *sell, int *index_bytes, int *sorted);
/* C = A B with scipy csr_matmat semantics (sparse.py:193-196): exact zeros dropped */
int mg_matmul(mg_ctx *ctx, const mg_mat *a, const mg_mat *b, mg_mat **out);
/* R (A P) (sparse.py:199-203) */
int mg_triple_product(mg_ctx *ctx, const mg_mat *r, const mg_mat *a, const mg_mat *p,
                      mg_mat **out);
int mg_transpose(mg_ctx *ctx, const mg_mat *a, mg_mat **out);
/* A[rows][:, cols] keeping stored zeros (sparse.py:181-190); index sets sorted */
int mg_extract(mg_ctx *ctx, const mg_mat *a, const int64_t *rows, int nr, const int64_t *cols,
               int nc, mg_mat **out);

/* ---- per-cell block scaling (cf. mgr.py:212-242) ------- */
/* from a BSR A: the per-cell prescale blocks G_i = Lambda_i D_i^-1 (D_i the
 * diagonal block; Lambda the equilibration lambda_r = |D_i[0][r]| or the
 * column max when zero; Lambda = I when equilibrate == 0) as a block-diagonal
 * BSR, and Ahat = G A as scalar CSR in cell-major unknown order with
 * diagonal blocks exactly diag(Lambda_i) and zero entries of the scaled
 * off-diagonal blocks dropped.  Returns the first singular cell via
 * mg_last_error_row on MG_ERR_SINGULAR. */
int mg_block_scale(mg_ctx *ctx, const mg_mat *a_bsr, int equilibrate, mg_mat **dinv_out,
                   mg_mat **ahat_out);
/* z = G v (per-cell b x b matvec) */
int mg_block_apply(mg_ctx *ctx, const mg_mat *dinv, const double *v, double *z);

/* ---- GmresSolver system scaling (linsolve.py:94-122) ------------------------ */
/* Symmetric infinity-norm equilibration (replaces GmresSolver._equilibrated,
 * linsolve.py:107-122): *scaled_out = (diag(1/row) A) diag(col_scale), two
 * rounded products per value with exact zeros dropped (scipy csr_matmat);
 * row_out[n] = max_j |a_ij| (0 -> 1): divide the rhs by it; col_scale_out[n]
 * = 1 / max_i |a_ij| / row_i (0 -> 1): multiply the solution by it.  Host
 * output arrays. */
int mg_equilibrate(mg_ctx *ctx, const mg_mat *a, mg_mat **scaled_out, double *row_out, double *col_scale_out);
/* max_i sum_j |a_ij| of a scalar CSR matrix (the a_norm of linsolve.py:97-98) */
int mg_abs_row_sum_max(mg_ctx *ctx, const mg_mat *a, double *out);

/* ---- ILU(k) comparator (ilu.py:53-174) ------------- */
typedef struct mg_ilu mg_ilu;
/* level-k incomplete LU of a square scalar CSR matrix (symbolic level-of-fill
 * closure on the host for k >= 1, numeric IKJ elimination on the device, no
 * pivoting).  MG_ERR_ZERO_PIVOT with the reference's row via
 * mg_last_error_row. */
int mg_ilu_factor(mg_ctx *ctx, const mg_mat *a, int level, mg_ilu **out);
/* combined L\U factor (unit lower diagonal implicit), as IluFactorization.matrix */
int mg_ilu_matrix(mg_ctx *ctx, const mg_ilu *f, mg_mat **out);
/* x = U^-1 L^-1 r (host vectors) */
int mg_ilu_apply(mg_ctx *ctx, mg_ilu *f, const double *r, double *x);
int mg_ilu_free(mg_ctx *ctx, mg_ilu *f);

/* ---- Newton system assembly (assembly.py:247-346) -- */
/* Problem description: the reference Problem's precomputed geometry (interior
 * faces a -> b with T, T_geo, g.dx; Dirichlet faces with their rule; per-cell
 * incidence lists in the reference's np.add.at order), constitutive models and
 * fluid constants.  Host arrays, copied at mg_asm_create. */
typedef struct {
  int n_cells, n_faces, n_dirichlet, n_neumann, n_rules;
  double cell_volume;
  /* fluid (physics.FluidParams; c_h, c_v precomputed) */
  double phi, diff_lh, mu_l, mu_g, rho_w_std, c_h, c_v;
  /* relperm / capillary models (van_genuchten flag, parameters, m = 1 - 1/n) */
  int rp_van_genuchten;
  double s_lr, s_gr, rp_m, rp_eps;
  int cp_van_genuchten;
  double p_entry, cp_n, cp_m, cp_eps;
  const int *face_a, *face_b;                      /* n_faces */
  const double *trans, *tgeo, *gdx;                /* n_faces */
  const int *dir_cell, *dir_rule;                  /* n_dirichlet */
  const double *dir_trans, *dir_tgeo, *dir_gdx;    /* n_dirichlet */
  /* Dirichlet rule ghost states: p_l, s_l, rho_lh, P_c, dP_c, lambda_l, lambda_g */
  const double *rule_p, *rule_s, *rule_rho, *rule_pc, *rule_dpc, *rule_lam_l, *rule_lam_g;
  /* per-cell incidence (n_cells + 1 offsets): entries f (a-side interior face),
   * f + 2^30 (b-side interior face), n_faces + q (Dirichlet face q), -1 - k
   * (Neumann contribution k); in the reference's accumulation order */
  const int *inc_rp, *inc_ent;
  const double *neu_w, *neu_h;                     /* n_neumann: -w*area, -h*area */
} mg_asm_desc;
typedef struct mg_asm mg_asm;
int mg_asm_create(mg_ctx *ctx, const mg_asm_desc *d, mg_asm **out);
/* Residual (host res[3 n]), active set (host active[n], 1 = gas present) and,
 * when jac_out != NULL, the Jacobian as a 3n x 3n scalar CSR device matrix
 * (variable-major, duplicates merged, explicit zeros kept).  States are host
 * arrays of n: p_l, s_l, rho_lh and the previous step's. */
int mg_asm_assemble(mg_ctx *ctx, mg_asm *a, const double *p, const double *s, const double *rho,
                    const double *p_old, const double *s_old, const double *rho_old, double dt, double *res,
                    int *active, mg_mat **jac_out);
int mg_asm_free(mg_ctx *ctx, mg_asm *a);

/* ---- MGR build_rp (mgr.py:117-156) ------------------------------------------ */
enum { MG_RP_INJECTIVE = 0, MG_RP_NONINJECTIVE = 1, MG_RP_INJECTION = 2, MG_RP_IDEAL = 3 };
int mg_build_rp(mg_ctx *ctx, const mg_mat *a, const uint8_t *f_mask, int kind, mg_mat **r_out,
                mg_mat **p_out);

/* ---- AMG (amg.py:31-49 options; PMIS / extended+i / L1-Jacobi on the GPU) -- */
typedef struct {
  double strength_theta;   /* 0.25 */
  int max_levels;          /* 25 */
  int coarse_size_cutoff;  /* 50 */
  int pre_sweeps;          /* 1 */
  int post_sweeps;         /* 1 */
  int cycles;              /* 1 */
  int max_elmts;           /* interpolation truncation, 0 = none */
  uint64_t seed;           /* PMIS measure seed */
} mg_amg_opts;

/* strength_graph (amg.py:88-103): int8 mask over every stored entry of A (1 = strong:
   cand >= theta * rowmax and rowmax > 0, cand = -a_ij for negative off-diagonals,
   |a_ij| in rows without one; the diagonal is never strong); n_strong may be NULL */
int mg_strength(mg_ctx *ctx, const mg_mat *a, double theta, int8_t *mask, int64_t *n_strong);
int mg_amg_setup(mg_ctx *ctx, const mg_mat *a, const mg_amg_opts *opts, mg_amg **out);
/* one V(pre,post) cycle from x0 (NULL = zero), amg.py:370-378 */
int mg_amg_vcycle(mg_ctx *ctx, mg_amg *h, const double *b, const double *x0, double *x);
/* `cycles` V-cycles from zero, amg.py:381-386 */
int mg_amg_apply(mg_ctx *ctx, mg_amg *h, const double *b, double *x);
int mg_amg_nlevels(mg_ctx *ctx, const mg_amg *h, int *nlevels, int *has_row_sign);
/* level matrices / interpolation / splitting for bit-exact comparisons.
 * what: 0 = A_l, 1 = P_l, 2 = splitting (int8 into vals buffer as bytes) */
int mg_amg_level_mat(mg_ctx *ctx, const mg_amg *h, int level, int what, mg_mat **out);
int mg_amg_splitting(mg_ctx *ctx, const mg_amg *h, int level, int8_t *state);
/* row signs applied at level 0 (amg.py:296-301); returns all +1 when none */
int mg_amg_row_sign(mg_ctx *ctx, const mg_amg *h, double *sign);
int mg_amg_free(mg_ctx *ctx, mg_amg *h);

/* ---- MGR (mgr.py:54-78 specs, 265-310 setup, 336-377 apply) ---------------- */
enum { MG_FRELAX_JACOBI = 0, MG_FRELAX_GAUSS_SEIDEL = 1, MG_FRELAX_AMG = 2, MG_FRELAX_EXACT = 3 };
enum { MG_COARSE_AMG = 0, MG_COARSE_EXACT = 1 };

typedef struct {
  const uint8_t *f_mask;   /* length = current level size, 1 = F point */
  int rp_kind;             /* MG_RP_* */
  int frelax_kind;         /* MG_FRELAX_* */
  int frelax_sweeps;
  int frelax_pre;
  int frelax_post;
  int frelax_max_levels;   /* 0 = no cap */
  int global_relax;        /* per-cell block-diagonal relaxation */
} mg_level_spec;

int mg_mgr_setup(mg_ctx *ctx, const mg_mat *a, const mg_level_spec *plan, int nlevels,
                 const mg_amg_opts *amg_opts, int coarse_kind, int post_smoothing,
                 const int64_t *cells, mg_mgr **out);
/* attach a per-cell block pre-scale: apply becomes MGR(Dinv v) */
int mg_mgr_set_prescale(mg_ctx *ctx, mg_mgr *h, const mg_mat *dinv);
int mg_mgr_apply(mg_ctx *ctx, mg_mgr *h, const double *r, double *e);
int mg_mgr_apply_dev(mg_ctx *ctx, mg_mgr *h, const double *r_dev, double *e_dev);
int mg_mgr_nlevels(mg_ctx *ctx, const mg_mgr *h, int *nlevels);
/* what: 0 = level A, 1 = R, 2 = P, 3 = coarse A, 4 = A_ff */
int mg_mgr_level_mat(mg_ctx *ctx, const mg_mgr *h, int level, int what, mg_mat **out);
/* borrowed view of the F-relaxation AMG at `level` (-1 = bottom coarse AMG);
 * release the view with mg_amg_free (the hierarchy keeps owning the data) */
int mg_mgr_level_amg(mg_ctx *ctx, const mg_mgr *h, int level, const mg_amg **out);
int mg_mgr_free(mg_ctx *ctx, mg_mgr *h);

/* ---- GMRES (krylov.py:20-144) --------------------------------------------- */
typedef struct {
  double rel_tol;          /* 1e-12 */
  int max_iter;            /* 400 */
  int restart;             /* 30 */
  int reorthogonalize;     /* 1: CGS2 via DCGS2 (one-reduction, delayed); 2: classic CGS2 (krylov.py:101-107
                              pass order); 0: single CGS pass */
  int check_every;         /* 25 */
} mg_gmres_opts;

typedef struct {
  int iterations;
  int converged;
  double residual_norm;
  double rhs_norm;
  int cycles;                  /* restart cycles run (Arnoldi loops) */
  int first_cycle_iterations;  /* iterations when the first cycle ended (-1: none ran) */
} mg_gmres_result;

/* right-preconditioned GMRES on `a` with preconditioner `m` (NULL = none).
 * a_norm < 0 means None (no backward-error acceptance). */
int mg_gmres(mg_ctx *ctx, const mg_mat *a, mg_mgr *m, const double *b, double *x,
             const mg_gmres_opts *opts, double a_norm, mg_gmres_result *res);
int mg_gmres_dev(mg_ctx *ctx, const mg_mat *a, mg_mgr *m, const double *b_dev, double *x_dev,
                 const mg_gmres_opts *opts, double a_norm, mg_gmres_result *res);
/* GMRES preconditioned by an ILU factorisation (GmresSolver(preconditioner='ilu'),
 * linsolve.py:79-84); host vectors */
int mg_gmres_ilu(mg_ctx *ctx, const mg_mat *a, mg_ilu *f, const double *b, double *x, const mg_gmres_opts *opts,
                 double a_norm, mg_gmres_result *out);

/* ---- device buffers (bench / e2e plumbing) --------------------------------- */
int mg_dev_alloc(mg_ctx *ctx, int64_t bytes, void **out);
int mg_dev_free(mg_ctx *ctx, void *p);
int mg_memcpy_h2d(mg_ctx *ctx, void *dst, const void *src, int64_t bytes);
int mg_memcpy_d2h(mg_ctx *ctx, void *dst, const void *src, int64_t bytes);

/* ---- timing: per-phase CUDA-event timing of the last setup / solve -------- */
typedef struct {
  double setup_ms;       /* last mg_mgr_setup (device time) */
  double solve_ms;       /* last mg_gmres (device time) */
  double spmv_ms;        /* accumulated BCSR SpMV kernel time in the last solve */
  int64_t spmv_calls;
  double vcycle_ms;      /* accumulated coarse-AMG V-cycle time in the last solve */
  int64_t vcycle_calls;
  double vcycle_bytes;   /* algorithmic bytes of one coarse V-cycle */
  double spmv_bytes;     /* algorithmic bytes of one BCSR SpMV */
  /* per-phase device time of the last solve when profiling is on:
   * 0 BCSR SpMV, 1 coarse AMG cycles, 2 F-relaxation, 3 GMRES orthogonalisation,
   * 4 MGR level transfers / residuals, 5 prescale, 6 GMRES host sync + Givens, 7 other */
  double phase_ms[8];
  /* the dominant single kernel: L1-Jacobi sweep on the coarse-AMG level-0 operator */
  double k0_ms;
  int64_t k0_calls;
  double k0_bytes;       /* algorithmic bytes per launch */
  /* MGR F-relaxation AMG V-cycles (phase_ms[2]): count and accumulated algorithmic
   * bytes (Amg::cycle_bytes of each cycle run) in the last profiled solve */
  int64_t frelax_calls;
  double frelax_bytes;
} mg_timing;
int mg_get_timing(mg_ctx *ctx, mg_timing *t);
/* CUDA-event timer on the context stream (bench timed regions) */
int mg_timer_start(mg_ctx *ctx);
int mg_timer_stop(mg_ctx *ctx, double *ms);
int mg_set_profiling(mg_ctx *ctx, int on);

#ifdef __cplusplus
}
#endif
#endif
