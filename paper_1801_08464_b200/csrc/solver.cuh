// Solver objects: AMG hierarchy, MGR hierarchy, GMRES driver.
#pragma once
#include <memory>
#include <vector>
#include "common.cuh"

namespace mg {

struct AmgOpts {
  double theta = 0.25;
  int max_levels = 25, cutoff = 50, pre = 1, post = 1, cycles = 1, max_elmts = 4;
  uint64_t seed = 0;
};

struct AmgLevel {
  Csr A;                  // level operator (level 0: row-sign-normalised copy)
  Csr P, R;               // interpolation from level l+1, R = P^T
  DBuf<int8_t> split;     // C/F marker of this level (0/1/2)
  DBuf<double> l1inv;     // 1 / sum_j |a_ij|
  DBuf<double> x, b, r, t;
  int n = 0;
};

struct Amg {
  AmgOpts opts;
  std::vector<AmgLevel> L;
  DBuf<double> sign;
  bool has_sign = false;
  DBuf<double> cinv;      // dense inverse of the coarsest operator
  int cn = 0;
  bool tag_k0 = false;    // time level-0 sweeps as the dominant kernel (MGR coarse AMG)
  double cycle_bytes() const;
  double k0_bytes() const {  // L1-Jacobi sweep on level 0: SpMV + b, D^-1 (x own counted in gather)
    return L.empty() ? 0.0 : L[0].A.bytes_spmv() + 16.0 * L[0].n;
  }
};

std::unique_ptr<Amg> amg_setup(const Csr &a, const AmgOpts &o);
// pre_done (x0 == nullptr only): the producer of b already formed the first
// pre-sweep from zero at the targets amg_pre_targets(h, x) returned
void amg_vcycle(Amg &h, const double *b, const double *x0, double *x, bool pre_done = false);
void amg_apply(Amg &h, const double *b, double *x, bool pre_done = false);
struct AmgPreTargets {
  bool ok = false;             // the hierarchy has a level-0 pre-sweep a producer can form
  const double *sign = nullptr;
  double *bs = nullptr;        // sign-normalised b (level-0 b buffer) when sign
  const double *d = nullptr;   // level-0 L1 inverse
  double *xo = nullptr;        // where the first pre-sweep writes for output x
};
AmgPreTargets amg_pre_targets(Amg &h, double *x);

enum { RP_INJECTIVE = 0, RP_NONINJECTIVE = 1, RP_INJECTION = 2, RP_IDEAL = 3 };
enum { FR_JACOBI = 0, FR_GS = 1, FR_AMG = 2, FR_EXACT = 3 };

struct LevelSpec {
  std::vector<uint8_t> fmask;
  int rp = RP_INJECTIVE, frelax = FR_JACOBI, sweeps = 1, pre = 1, post = 1, max_levels = 0;
  int global_relax = 0;
};

struct FSolver {
  int kind = FR_JACOBI, sweeps = 1;
  DBuf<double> invd;           // jacobi
  Csr tril;                    // gauss_seidel: lower triangle of A_ff (diagonal last)
  DBuf<int> ctrl;              // gauss_seidel: substitution ticket + ready flags
  std::unique_ptr<Amg> amg;    // amg
  DBuf<double> dinv;           // exact (dense inverse)
  DBuf<double> t1, t2;
  int nf = 0;
};

struct BlockDiag {             // per-cell block-diagonal relaxation (mgr.py:212-242)
  int nblk = 0, kmax = 0;      // blocks of size ioff[b+1]-ioff[b] <= 8 (mixed sizes allowed)
  DBuf<int> idx;               // unknowns of all blocks, concatenated
  DBuf<int> ioff;              // nblk + 1 offsets into idx
  DBuf<int64_t> moff;          // nblk + 1 offsets into inv (k*k per block)
  DBuf<double> inv;            // row-major block inverses
};

struct MgrLevel {
  Csr A, R, P, Aff;
  Csr AF;                      // A[:, F] (F-local columns): residual after F-relaxation from e = 0
  Csr AFr;                     // A[F, :] (post_smoothing): the F rows of the residual before the F-relaxation
  int n = 0, nf = 0, nc = 0, rp = 0;
  DBuf<int> flist, clist, fmap;
  FSolver fs;
  std::unique_ptr<BlockDiag> bd;
  DBuf<double> res, rF, eF, rc, ec;
};

struct Mgr {
  std::vector<MgrLevel> L;
  int coarse_kind = 0;
  std::unique_ptr<Amg> camg;
  DBuf<double> cinv;
  int cn = 0;
  Csr coarse_A;
  bool post_smoothing = false;
  int n0 = 0;
  Csr prescale;                // optional per-cell D^-1 (block diagonal)
  bool has_prescale = false;
  DBuf<double> pre_buf;
  // CUDA graph of one apply, captured on first use.  Output: the fixed buffer
  // gout.  Input: with a prescale, read through the device pointer slot in_slot
  // (set by a one-thread kernel before each replay: no copy); else copied into gin.
  cudaGraphExec_t gexec = nullptr;
  Ctx *gctx = nullptr;          // context whose stream the graph was captured on
  DBuf<double> gin, gout;
  DBuf<const double *> in_slot;
  int64_t graph_kernels = 0;
  bool graph_failed = false;
  ~Mgr();
  void drop_graph();
};

std::unique_ptr<Mgr> mgr_setup(const Csr &a, const std::vector<LevelSpec> &plan, const AmgOpts &ao,
                               int coarse_kind, bool post_smoothing, const int64_t *cells_host);
void mgr_apply(Mgr &h, const double *r, double *e);
// as mgr_apply, but the result may be left in the hierarchy's graph output buffer
// (valid until the next apply on h): returns where it is (e or that buffer)
const double *mgr_apply_result(Mgr &h, const double *r, double *e);

// ILU(k) comparator (ilu.cu; ilu.py:53-174)
struct Ilu {
  Csr LU;                      // combined factor, sorted columns, unit lower diagonal implicit
  DBuf<int> dpos;              // diagonal position per row
  DBuf<int> ctrl;              // substitution ticket + ready flags
  DBuf<double> t;              // intermediate of the two substitutions
  int n = 0, level = 0;
};
std::unique_ptr<Ilu> ilu_factor(const Csr &a, int level);
void ilu_apply(Ilu &f, const double *r, double *x);

struct GmresOpts {
  double rel_tol = 1e-12;
  int max_iter = 400, restart = 30, reorth = 1, check_every = 25;
};
struct GmresOut {
  int iterations = 0, converged = 0;
  double residual_norm = 0, rhs_norm = 0;
  int cycles = 0, first_cycle = -1;  // restart cycles run; iterations when the first one ended
};
GmresOut gmres(const Csr &a, Mgr *m, const double *b, double *x, const GmresOpts &o, double a_norm,
               Ilu *ilu = nullptr);

// build_rp (mgr_ops.cu)
void fc_split(const uint8_t *fmask_dev, int n, DBuf<int> &flist, DBuf<int> &clist, DBuf<int> &fmap,
              DBuf<int> &cmap, int &nf, int &nc);
void build_rp(const Csr &a, const int *fmap, const int *cmap, const int *flist, const int *clist, int nf,
              int nc, int kind, Csr &r, Csr &p);

// Gauss-Seidel F-relaxation (trisolve.cu)
void tril_setup(const Csr &a, Csr &l);
void trsv_lower(const Csr &l, const double *r, double *x, int *ctrl);

// profiling of the hot kernels inside a solve
struct ProfScope {
  int kind;  // 0 spmv, 1 vcycle
  cudaEvent_t a = nullptr, b = nullptr;
  explicit ProfScope(int k);
  ~ProfScope();
};
void prof_reset();
void prof_collect();

}  // namespace mg
