// Newton residual / Jacobian assembly of the two-phase NCP system on the device
// (SURVEY.md §8(f) item 3): replaces ncpflow/assembly.py:247-346
// (Problem._assemble, _flux_contributions) and the COO -> CSR merge of
// CsrMatrix.from_coo (sparse.py:88-93), which is the step immediately before
// the linear solve.
//
// * Constitutive laws per cell (physics.py relperm / capillary with the
//   Van Genuchten clamps and tangent extensions, power-law / linear variants),
//   the same formulas in the same operation order (libm-accurate pow/sqrt).
// * Two-point fluxes per face (interior faces a -> b, then the Dirichlet
//   boundary faces of each rule with the ghost state on side b).
// * Residual: per cell, the accumulation term plus the face fluxes gathered in
//   exactly the order np.add.at applies them in the reference (a-side faces in
//   face order, then b-side faces, Neumann groups, Dirichlet groups), scaled by
//   dt/V; complementarity rows min(1 - S_l, C_h P_g - rho_lh).
// * Jacobian: every COO triplet the reference emits (same rows, columns and
//   values, balance rows scaled by dt/V before the merge), sorted by
//   (row, column) and merged; duplicate sums in sorted order (scipy's merge
//   order is an unstable sort, so values agree to rounding, patterns exactly,
//   explicit zeros kept as the reference keeps them).
#include <cub/cub.cuh>
#include "ops.cuh"
#include "../../include/mgrgpu.h"

namespace mg {
namespace {

struct Models {
  // relperm
  int rp_vg;
  double s_lr, s_gr, rp_m, rp_eps;
  // capillary
  int cp_vg;
  double p_entry, cp_n, cp_m, cp_eps;
};

__device__ void vg_curves(double s, double m, double &krl, double &krg) {
  double u = pow(s, 1.0 / m);
  double w = 1.0 - pow(1.0 - u, m);
  krl = sqrt(s) * (w * w);
  krg = sqrt(1.0 - s) * pow(1.0 - u, 2.0 * m);
}

// relperm (physics.py:145-219): krl, krg and d/dS_l (times dse)
__device__ void relperm(double s_l, const Models &md, double &krl, double &krg, double &dkrl, double &dkrg) {
  const double span = 1.0 - md.s_lr - md.s_gr;
  const double se = (s_l - md.s_lr) / span;
  const double dse = 1.0 / span;
  const double sc = fmin(fmax(se, 0.0), 1.0);
  const bool interior = se > 0.0 && se < 1.0;
  dkrl = 0.0;
  dkrg = 0.0;
  if (!md.rp_vg) {
    krl = sc * sc;
    krg = (1.0 - sc) * (1.0 - sc);
    if (interior) {
      dkrl = 2.0 * sc;
      dkrg = -2.0 * (1.0 - sc);
    }
  } else {
    const double m = md.rp_m, eps = md.rp_eps;
    krl = 0.0;
    krg = 0.0;
    if (se <= 0.0) { krl = 0.0; krg = 1.0; }
    if (se >= 1.0) { krl = 1.0; krg = 0.0; }
    double krl_lo, krg_lo, krl_hi, krg_hi;
    vg_curves(eps, m, krl_lo, krg_lo);
    vg_curves(1.0 - eps, m, krl_hi, krg_hi);
    if (se >= eps && se <= 1.0 - eps) {
      const double s = sc;
      const double u = pow(s, 1.0 / m);
      const double omu = 1.0 - u;
      const double w = 1.0 - pow(omu, m);
      const double sqrt_s = sqrt(s);
      krl = sqrt_s * (w * w);
      const double dw = pow(omu, m - 1.0) * pow(s, 1.0 / m - 1.0);
      dkrl = 0.5 * (w * w) / sqrt_s + 2.0 * sqrt_s * w * dw;
      const double sqrt_1ms = sqrt(1.0 - s);
      krg = sqrt_1ms * pow(omu, 2.0 * m);
      dkrg = (-0.5 * pow(omu, 2.0 * m) / sqrt_1ms - 2.0 * sqrt_1ms * pow(omu, 2.0 * m - 1.0) * pow(s, 1.0 / m - 1.0));
    }
    if (interior && se < eps) {
      const double t = sc / eps;
      krl = krl_lo * t;
      dkrl = krl_lo / eps;
      krg = 1.0 + (krg_lo - 1.0) * t;
      dkrg = (krg_lo - 1.0) / eps;
    }
    if (interior && se > 1.0 - eps) {
      const double t = (sc - (1.0 - eps)) / eps;
      krl = krl_hi + (1.0 - krl_hi) * t;
      dkrl = (1.0 - krl_hi) / eps;
      krg = krg_hi * (1.0 - t);
      dkrg = -krg_hi / eps;
    }
  }
  dkrl = dkrl * dse;
  dkrg = dkrg * dse;
}

__device__ void vg_pc(double se, const Models &md, double &pc, double &dpc) {
  const double m = md.cp_m;
  const double t = pow(se, -1.0 / m) - 1.0;
  pc = md.p_entry * pow(t, 1.0 / md.cp_n);
  dpc = md.p_entry * (1.0 / md.cp_n) * pow(t, 1.0 / md.cp_n - 1.0) * (-1.0 / m) * pow(se, -1.0 / m - 1.0);
}

// capillary (physics.py:231-257)
__device__ void capillary(double s_l, const Models &md, double &pc, double &dpc) {
  const double span = 1.0 - md.s_lr - md.s_gr;
  const double se = (s_l - md.s_lr) / span;
  const double dse = 1.0 / span;
  if (!md.cp_vg) {
    pc = md.p_entry * (1.0 - se);
    dpc = -md.p_entry * dse;
    return;
  }
  const double eps = md.cp_eps;
  if (se < eps) {
    double pc_lo, slope_lo;
    vg_pc(eps, md, pc_lo, slope_lo);
    pc = pc_lo + slope_lo * (se - eps);
    dpc = slope_lo;
  } else if (se > 1.0 - eps) {
    double pc_hi, slope_hi;
    vg_pc(1.0 - eps, md, pc_hi, slope_hi);
    pc = pc_hi + slope_hi * (se - (1.0 - eps));
    dpc = slope_hi;
  } else {
    vg_pc(se, md, pc, dpc);
  }
  dpc = dpc * dse;
}

struct Params {
  double phi, diff_lh, mu_l, mu_g, rho_w_std, c_h, c_v;
};

// per-cell evaluation of the state (Problem._eval, assembly.py:205-214)
__global__ void k_eval(int n, const double *__restrict__ p, const double *__restrict__ s, Models md, Params pr,
                       double *pc, double *dpc, double *lam_l, double *dlam_l, double *lam_g, double *dlam_g) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double c, dc, krl, krg, dkrl, dkrg;
  capillary(s[i], md, c, dc);
  relperm(s[i], md, krl, krg, dkrl, dkrg);
  pc[i] = c;
  dpc[i] = dc;
  lam_l[i] = krl / pr.mu_l;
  dlam_l[i] = dkrl / pr.mu_l;
  lam_g[i] = krg / pr.mu_g;
  dlam_g[i] = dkrg / pr.mu_g;
  (void)p;
}

struct Cell {
  const double *p, *s, *r;                 // state
  const double *pc, *dpc, *lam_l, *dlam_l, *lam_g, *dlam_g;
};

struct Ghost {  // Dirichlet rule ghost state (b side)
  double p, s, r, pc, dpc, lam_l, lam_g;
};

// fluxes and the face's Jacobian triplets (_flux_contributions, assembly.py:348-470)
// writes fw, fh and (when rows != nullptr) 46 (interior) / 23 (boundary) triplets
__device__ void face_flux(int n, int a, int b, bool bnd, const Ghost &gh, double t, double tgeo, double gdx,
                          const Cell &c, const Params &pr, double &fw, double &fh, int64_t *rows, int *cols,
                          double *vals) {
  const double pa = c.p[a], sa = c.s[a], ra = c.r[a], pca = c.pc[a], dpca = c.dpc[a];
  const double lam_la = c.lam_l[a], dlam_la = c.dlam_l[a], lam_ga = c.lam_g[a], dlam_ga = c.dlam_g[a];
  double pb, sb, rb, pcb, dpcb, lam_lb, dlam_lb, lam_gb, dlam_gb;
  if (bnd) {
    pb = gh.p; sb = gh.s; rb = gh.r; pcb = gh.pc; dpcb = gh.dpc;
    lam_lb = gh.lam_l; dlam_lb = 0.0; lam_gb = gh.lam_g; dlam_gb = 0.0;
  } else {
    pb = c.p[b]; sb = c.s[b]; rb = c.r[b]; pcb = c.pc[b]; dpcb = c.dpc[b];
    lam_lb = c.lam_l[b]; dlam_lb = c.dlam_l[b]; lam_gb = c.lam_g[b]; dlam_gb = c.dlam_g[b];
  }
  const double pga = pa + pca, pgb = pb + pcb;
  const double rho_l_face = pr.rho_w_std + 0.5 * (ra + rb);
  const double rho_g_face = 0.5 * pr.c_v * (pga + pgb);
  const double dphi_l = (pa - pb) - rho_l_face * gdx;
  const double dphi_g = (pga - pgb) - rho_g_face * gdx;
  const bool up_l = dphi_l >= 0.0, up_g = dphi_g >= 0.0;
  const double lam_l_up = up_l ? lam_la : lam_lb;
  const double r_up = up_l ? ra : rb;
  const double lam_g_up = up_g ? lam_ga : lam_gb;
  const double pg_up = up_g ? pga : pgb;
  const double rho_g_up = pr.c_v * pg_up;
  const double dfac = tgeo * pr.phi * pr.diff_lh * 0.5 * (sa + sb);
  const double f_diff = dfac * (ra - rb);
  const double fw_adv = pr.rho_w_std * lam_l_up * t * dphi_l;
  const double fh_l = r_up * lam_l_up * t * dphi_l;
  const double fh_g = rho_g_up * lam_g_up * t * dphi_g;
  fw = fw_adv - f_diff;
  fh = fh_l + fh_g + f_diff;
  if (!rows) return;

  const double half_g = 0.5 * gdx;
  const double ddphil_dpa = 1.0, ddphil_dpb = -1.0;
  const double ddphil_dra = -half_g, ddphil_drb = -half_g;
  const double ddphig_dpa = 1.0 - pr.c_v * half_g;
  const double ddphig_dpb = -1.0 - pr.c_v * half_g;
  const double ddphig_dsa = dpca * (1.0 - pr.c_v * half_g);
  const double ddphig_dsb = -dpcb * (1.0 + pr.c_v * half_g);
  const double c_l = lam_l_up * t;
  const double live_l = bnd ? (up_l ? 1.0 : 0.0) : 1.0;
  const double live_g = bnd ? (up_g ? 1.0 : 0.0) : 1.0;
  const int bb = bnd ? a : b;
  const int col_pa = a, col_pb = bb, col_sa = n + a, col_sb = n + bb, col_ra = 2 * n + a, col_rb = 2 * n + bb;
  const int wrow_a = a, wrow_b = bb, hrow_a = n + a, hrow_b = n + bb;
  const double keep_b = bnd ? 0.0 : 1.0;
  int k = 0;
  auto scatter = [&](int ra_, int rb_, int col, double val) {
    rows[k] = ra_; cols[k] = col; vals[k] = val; ++k;
    if (!bnd) { rows[k] = rb_; cols[k] = col; vals[k] = -val; ++k; }
  };
  // water row
  double coef = pr.rho_w_std * c_l;
  scatter(wrow_a, wrow_b, col_pa, coef * ddphil_dpa);
  scatter(wrow_a, wrow_b, col_pb, keep_b * coef * ddphil_dpb);
  const double dlam_up = up_l ? dlam_la : dlam_lb;
  const int up_cols = up_l ? n + a : (bnd ? n + a : n + b);
  scatter(wrow_a, wrow_b, up_cols, live_l * pr.rho_w_std * dlam_up * t * dphi_l);
  const double ddfac = tgeo * pr.phi * pr.diff_lh * 0.5;
  scatter(wrow_a, wrow_b, col_sa, -ddfac * (ra - rb));
  scatter(wrow_a, wrow_b, col_sb, keep_b * (-ddfac * (ra - rb)));
  scatter(wrow_a, wrow_b, col_ra, -dfac + coef * ddphil_dra);
  scatter(wrow_a, wrow_b, col_rb, keep_b * (dfac + coef * ddphil_drb));
  // hydrogen row, liquid advection
  coef = r_up * c_l;
  scatter(hrow_a, hrow_b, col_pa, coef * ddphil_dpa);
  scatter(hrow_a, hrow_b, col_pb, keep_b * coef * ddphil_dpb);
  scatter(hrow_a, hrow_b, up_cols, live_l * r_up * dlam_up * t * dphi_l);
  const int up_cols_r = up_l ? 2 * n + a : (bnd ? 2 * n + a : 2 * n + b);
  scatter(hrow_a, hrow_b, up_cols_r, live_l * lam_l_up * t * dphi_l);
  scatter(hrow_a, hrow_b, col_ra, coef * ddphil_dra);
  scatter(hrow_a, hrow_b, col_rb, keep_b * coef * ddphil_drb);
  // hydrogen row, gas advection
  const double cg = rho_g_up * lam_g_up * t;
  scatter(hrow_a, hrow_b, col_pa, cg * ddphig_dpa);
  scatter(hrow_a, hrow_b, col_pb, keep_b * cg * ddphig_dpb);
  scatter(hrow_a, hrow_b, col_sa, cg * ddphig_dsa);
  scatter(hrow_a, hrow_b, col_sb, keep_b * cg * ddphig_dsb);
  const double dlam_g_up = up_g ? dlam_ga : dlam_gb;
  const double dpc_up = up_g ? dpca : dpcb;
  const int up_cols_s = up_g ? n + a : (bnd ? n + a : n + b);
  const int up_cols_p = up_g ? a : (bnd ? a : b);
  scatter(hrow_a, hrow_b, up_cols_s, live_g * (pr.c_v * dpc_up * lam_g_up + rho_g_up * dlam_g_up) * t * dphi_g);
  scatter(hrow_a, hrow_b, up_cols_p, live_g * pr.c_v * lam_g_up * t * dphi_g);
  // hydrogen row, diffusion
  scatter(hrow_a, hrow_b, col_sa, ddfac * (ra - rb));
  scatter(hrow_a, hrow_b, col_sb, keep_b * ddfac * (ra - rb));
  scatter(hrow_a, hrow_b, col_ra, dfac);
  scatter(hrow_a, hrow_b, col_rb, keep_b * (-dfac));
}

constexpr int FACE_NNZ = 46;   // triplets per interior face
constexpr int BFACE_NNZ = 23;  // triplets per Dirichlet face
constexpr int CELL_NNZ = 7;    // accumulation (4) + complementarity (<= 3), padded

struct Geo {
  int n, nf, nbd;                    // cells, interior faces, Dirichlet faces
  const int *fa, *fb;
  const double *t, *tgeo, *gdx;
  const int *bcell, *brule;          // Dirichlet faces: cell, rule index
  const double *bt, *btgeo, *bgdx;
  const Ghost *ghosts;               // per rule
};

__global__ void k_faces(Geo g, Cell c, Params pr, double *fw, double *fh, int64_t *rows, int *cols, double *vals) {
  int f = blockIdx.x * blockDim.x + threadIdx.x;
  if (f >= g.nf + g.nbd) return;
  Ghost none{};
  double w, h;
  if (f < g.nf) {
    size_t o = (size_t)f * FACE_NNZ;
    face_flux(g.n, g.fa[f], g.fb[f], false, none, g.t[f], g.tgeo[f], g.gdx[f], c, pr, w, h,
              rows ? rows + o : nullptr, cols ? cols + o : nullptr, vals ? vals + o : nullptr);
  } else {
    int q = f - g.nf;
    size_t o = (size_t)g.nf * FACE_NNZ + (size_t)q * BFACE_NNZ;
    face_flux(g.n, g.bcell[q], -1, true, g.ghosts[g.brule[q]], g.bt[q], g.btgeo[q], g.bgdx[q], c, pr, w, h,
              rows ? rows + o : nullptr, cols ? cols + o : nullptr, vals ? vals + o : nullptr);
  }
  fw[f] = w;
  fh[f] = h;
}

// per-cell residual in the reference's np.add.at order; incidence list per cell:
// entries (face index, +1 a-side / -1 b-side) for the interior faces (a-sides
// first), then Neumann entries (as negative -1 - k into neu_w / neu_h), then
// Dirichlet faces (nf + q)
struct Inc {
  const int *rp;       // n + 1
  const int *ent;      // encoded entries
  const double *neu_w, *neu_h;  // Neumann contributions -w*area, -h*area per entry
};

__global__ void k_cells(int n, double vphi_dt, double scale, Params pr, Cell c, const double *__restrict__ s_old,
                        const double *__restrict__ r_old, const double *__restrict__ pc_old,
                        const double *__restrict__ p_old, const double *__restrict__ fw,
                        const double *__restrict__ fh, Inc inc, double *res, int64_t *rows, int *cols,
                        double *vals, int *active) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double s = c.s[i], rho = c.r[i];
  const double rho_g = pr.c_v * (c.p[i] + c.pc[i]);
  const double rho_g_old = pr.c_v * (p_old[i] + pc_old[i]);
  double rw = vphi_dt * pr.rho_w_std * (s - s_old[i]);
  const double m_h = s * rho + (1.0 - s) * rho_g;
  const double m_h_old = s_old[i] * r_old[i] + (1.0 - s_old[i]) * rho_g_old;
  double rh = vphi_dt * (m_h - m_h_old);
  // the water row receives every face contribution before the hydrogen row in the
  // reference, but each row's own sequence is what matters: same order for both
  for (int q = inc.rp[i]; q < inc.rp[i + 1]; ++q) {
    const int e = inc.ent[q];
    if (e >= 0) {  // interior a-side (+) / b-side (encoded >= 2^30), or Dirichlet face
      const bool bside = e >= (1 << 30);
      const int f = bside ? e - (1 << 30) : e;
      if (bside) {
        rw = rw + (-fw[f]);
        rh = rh + (-fh[f]);
      } else {
        rw = rw + fw[f];
        rh = rh + fh[f];
      }
    } else {
      const int k = -1 - e;
      rw = rw + inc.neu_w[k];
      rh = rh + inc.neu_h[k];
    }
  }
  res[i] = rw * scale;
  res[n + i] = rh * scale;
  const double f_con = 1.0 - s;
  const double g_con = pr.c_h * (c.p[i] + c.pc[i]) - rho;
  res[2 * n + i] = fmin(f_con, g_con);
  const bool act = f_con >= g_con;
  active[i] = act;
  if (!rows) return;
  int64_t *r = rows + (size_t)i * CELL_NNZ;
  int *cc = cols + (size_t)i * CELL_NNZ;
  double *v = vals + (size_t)i * CELL_NNZ;
  r[0] = i;         cc[0] = n + i;     v[0] = (vphi_dt * pr.rho_w_std) * scale;
  r[1] = n + i;     cc[1] = i;         v[1] = (vphi_dt * (1.0 - s) * pr.c_v) * scale;
  r[2] = n + i;     cc[2] = n + i;     v[2] = (vphi_dt * (rho - rho_g + (1.0 - s) * pr.c_v * c.dpc[i])) * scale;
  r[3] = n + i;     cc[3] = 2 * n + i; v[3] = (vphi_dt * s) * scale;
  if (act) {
    r[4] = 2 * n + i; cc[4] = i;         v[4] = pr.c_h;
    r[5] = 2 * n + i; cc[5] = n + i;     v[5] = pr.c_h * c.dpc[i];
    r[6] = 2 * n + i; cc[6] = 2 * n + i; v[6] = -1.0;
  } else {
    r[4] = 2 * n + i; cc[4] = n + i;     v[4] = -1.0;
    r[5] = -1; cc[5] = 0; v[5] = 0.0;    // unused slots (dropped before the merge)
    r[6] = -1; cc[6] = 0; v[6] = 0.0;
  }
}

// balance rows (< 2n) of the face triplets scaled by dt/V (assembly.py:337-338)
__global__ void k_scale_face_vals(int64_t m, int two_n, double scale, const int64_t *rows, double *vals) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k < m && rows[k] < two_n) vals[k] = vals[k] * scale;
}

// key = row * ncols + col; unused cell slots get ncols * ncols (sorts last)
__global__ void k_coo_keys(int64_t m, int64_t ncols, const int64_t *rows, const int *cols, int64_t *keys) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  keys[k] = rows[k] < 0 ? ncols * ncols : rows[k] * ncols + cols[k];
}
__global__ void k_run_heads(int64_t m, int64_t none, const int64_t *keys, int *head) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m) return;
  head[k] = keys[k] != none && (k == 0 || keys[k] != keys[k - 1]);
}
// one thread per unique (row, col): sum its run in sorted (stable: emission) order
__global__ void k_merge_runs(int64_t m, int64_t ncols, const int64_t *keys, const double *vals, const int *pos,
                             const int *head, int *ci, double *v, int *rowcnt) {
  int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (k >= m || !head[k]) return;
  const int64_t key = keys[k];
  double s = 0.0;
  for (int64_t q = k; q < m && keys[q] == key; ++q) s = s + vals[q];
  const int o = pos[k];
  ci[o] = (int)(key % ncols);
  v[o] = s;
  atomicAdd(rowcnt + key / ncols, 1);
}

}  // namespace

struct AsmGeo {
  int n = 0, nf = 0, nbd = 0;
  DBuf<int> fa, fb, bcell, brule, inc_rp, inc_ent;
  DBuf<double> t, tgeo, gdx, bt, btgeo, bgdx, neu_w, neu_h;
  DBuf<Ghost> ghosts;
  Models md{};
  Params pr{};
  double cell_vol = 1.0;
};

AsmGeo *asm_create(const mg_asm_desc &d) {
  auto g = new AsmGeo();
  g->n = d.n_cells;
  g->nf = d.n_faces;
  g->nbd = d.n_dirichlet;
  g->cell_vol = d.cell_volume;
  g->md = Models{d.rp_van_genuchten, d.s_lr, d.s_gr, d.rp_m, d.rp_eps, d.cp_van_genuchten, d.p_entry, d.cp_n,
                 d.cp_m, d.cp_eps};
  g->pr = Params{d.phi, d.diff_lh, d.mu_l, d.mu_g, d.rho_w_std, d.c_h, d.c_v};
  auto up_i = [](DBuf<int> &b, const int *h, int64_t m) {
    b.alloc((size_t)(m ? m : 1));
    if (m) h2d(b.p, h, sizeof(int) * m);
  };
  auto up_d = [](DBuf<double> &b, const double *h, int64_t m) {
    b.alloc((size_t)(m ? m : 1));
    if (m) h2d(b.p, h, sizeof(double) * m);
  };
  up_i(g->fa, d.face_a, g->nf);
  up_i(g->fb, d.face_b, g->nf);
  up_d(g->t, d.trans, g->nf);
  up_d(g->tgeo, d.tgeo, g->nf);
  up_d(g->gdx, d.gdx, g->nf);
  up_i(g->bcell, d.dir_cell, g->nbd);
  up_i(g->brule, d.dir_rule, g->nbd);
  up_d(g->bt, d.dir_trans, g->nbd);
  up_d(g->btgeo, d.dir_tgeo, g->nbd);
  up_d(g->bgdx, d.dir_gdx, g->nbd);
  up_i(g->inc_rp, d.inc_rp, (int64_t)g->n + 1);
  up_i(g->inc_ent, d.inc_ent, d.inc_rp[g->n]);
  up_d(g->neu_w, d.neu_w, d.n_neumann);
  up_d(g->neu_h, d.neu_h, d.n_neumann);
  std::vector<Ghost> gh(d.n_rules);
  for (int r = 0; r < d.n_rules; ++r)
    gh[r] = Ghost{d.rule_p[r], d.rule_s[r], d.rule_rho[r], d.rule_pc[r], d.rule_dpc[r], d.rule_lam_l[r],
                  d.rule_lam_g[r]};
  g->ghosts.alloc((size_t)(d.n_rules ? d.n_rules : 1));
  if (d.n_rules) h2d(g->ghosts.p, gh.data(), sizeof(Ghost) * d.n_rules);
  return g;
}

void asm_destroy(AsmGeo *g) { delete g; }

// residual (3n, device) and, when jac != nullptr, the Jacobian (3n x 3n CSR)
void asm_assemble(AsmGeo &g, const double *p, const double *s, const double *r, const double *p_old,
                  const double *s_old, const double *r_old, double dt, double *res, int *active, Csr *jac) {
  if (!(dt > 0.0)) throw MgError(MG_ERR_BAD_OPTION, "dt must be positive");
  const int n = g.n;
  DBuf<double> pc(n), dpc(n), ll(n), dll(n), lg(n), dlg(n), pco(n), dpco(n), t1(n), t2(n), t3(n), t4(n);
  k_eval<<<grid_for(n, 256), 256, 0, stream()>>>(n, p, s, g.md, g.pr, pc.p, dpc.p, ll.p, dll.p, lg.p, dlg.p);
  check_launch("asm_eval");
  k_eval<<<grid_for(n, 256), 256, 0, stream()>>>(n, p_old, s_old, g.md, g.pr, pco.p, dpco.p, t1.p, t2.p, t3.p,
                                                 t4.p);
  check_launch("asm_eval_old");
  Cell c{p, s, r, pc.p, dpc.p, ll.p, dll.p, lg.p, dlg.p};
  Geo geo{n, g.nf, g.nbd, g.fa.p, g.fb.p, g.t.p, g.tgeo.p, g.gdx.p, g.bcell.p, g.brule.p, g.bt.p, g.btgeo.p,
          g.bgdx.p, g.ghosts.p};
  const int nfaces = g.nf + g.nbd;
  DBuf<double> fw((size_t)(nfaces ? nfaces : 1)), fh((size_t)(nfaces ? nfaces : 1));
  const int64_t mface = (int64_t)g.nf * FACE_NNZ + (int64_t)g.nbd * BFACE_NNZ;
  const int64_t mtot = mface + (int64_t)n * CELL_NNZ;
  DBuf<int64_t> rows;
  DBuf<int> cols;
  DBuf<double> vals;
  if (jac) {
    rows.alloc((size_t)mtot);
    cols.alloc((size_t)mtot);
    vals.alloc((size_t)mtot);
  }
  if (nfaces) {
    k_faces<<<grid_for(nfaces, 128), 128, 0, stream()>>>(geo, c, g.pr, fw.p, fh.p, jac ? rows.p : nullptr,
                                                         jac ? cols.p : nullptr, jac ? vals.p : nullptr);
    check_launch("asm_faces");
  }
  const double vphi_dt = g.cell_vol * g.pr.phi / dt;
  const double scale = dt / g.cell_vol;
  Inc inc{g.inc_rp.p, g.inc_ent.p, g.neu_w.p, g.neu_h.p};
  k_cells<<<grid_for(n, 256), 256, 0, stream()>>>(n, vphi_dt, scale, g.pr, c, s_old, r_old, pco.p, p_old, fw.p,
                                                  fh.p, inc, res, jac ? rows.p + mface : nullptr,
                                                  jac ? cols.p + mface : nullptr, jac ? vals.p + mface : nullptr,
                                                  active);
  check_launch("asm_cells");
  if (!jac) return;
  if (mface) {
    k_scale_face_vals<<<grid_for(mface, 256), 256, 0, stream()>>>(mface, 2 * n, scale, rows.p, vals.p);
    check_launch("asm_scale");
  }
  // COO -> CSR: stable sort by (row, col), merge runs (CsrMatrix.from_coo)
  const int64_t N3 = 3 * (int64_t)n;
  DBuf<int64_t> keys((size_t)mtot), keys_s((size_t)mtot);
  DBuf<double> vals_s((size_t)mtot);
  k_coo_keys<<<grid_for(mtot, 256), 256, 0, stream()>>>(mtot, N3, rows.p, cols.p, keys.p);
  check_launch("coo_keys");
  int bits = 1;
  while (bits < 63 && (int64_t(1) << bits) <= N3 * N3) ++bits;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.p, keys_s.p, vals.p, vals_s.p, (int)mtot, 0, bits, stream());
  void *tmp = cub_scratch(tb);
  MG_CUDA(cub::DeviceRadixSort::SortPairs(tmp, tb, keys.p, keys_s.p, vals.p, vals_s.p, (int)mtot, 0, bits,
                                          stream()));
  count_launch(4);
  DBuf<int> head((size_t)mtot), pos((size_t)mtot + 1);
  k_run_heads<<<grid_for(mtot, 256), 256, 0, stream()>>>(mtot, N3 * N3, keys_s.p, head.p);
  check_launch("run_heads");
  const int64_t nnz = exclusive_scan_i32_to_i32(head.p, pos.p, (int)mtot);
  jac->alloc((int)N3, (int)N3, nnz);
  DBuf<int> rowcnt((size_t)N3 + 1);
  dzero(rowcnt.p, sizeof(int) * ((size_t)N3 + 1));
  k_merge_runs<<<grid_for(mtot, 256), 256, 0, stream()>>>(mtot, N3, keys_s.p, vals_s.p, pos.p, head.p, jac->ci.p,
                                                          jac->v.p, rowcnt.p);
  check_launch("merge_runs");
  exclusive_scan_i32_to_i32(rowcnt.p, jac->rp.p, (int)N3);
}

}  // namespace mg
