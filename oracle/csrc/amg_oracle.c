/*
 * CPU oracle for the AMG pieces the reference does not contain.
 * TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference leg; never by the product path.
 *
 * The reference AMG (ncpflow/amg.py) uses Ruge-Stueben coarsening
 * (amg.py:106-158), classical interpolation (amg.py:206-276) and
 * Gauss-Seidel (amg.py:279-286).  The north star replaces those with PMIS,
 * extended+i interpolation and L1-Jacobi; SURVEY.md §8(c) fixes the
 * contract restated here.  This file pins every operation order, because the
 * GPU kernels (paper_1801_08464_b200/csrc/amg_setup.cu) reproduce it bit for
 * bit: compile with -ffp-contract=off (no FMA), as the GPU side uses
 * --fmad=false.
 *
 * Layout: CSR, int32 indptr/indices, sorted columns, f64 values; the
 * strength mask is int8 aligned with the stored entries (as
 * ncpflow.amg.strength_graph returns, amg.py:88-103).  State codes follow
 * amg.py:24 (0 undecided, 1 F, 2 C).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

#define UNDECIDED 0
#define FPOINT 1
#define CPOINT 2

/* splitmix64 finaliser; the PMIS random measure is pinned to it. */
static inline uint64_t splitmix64(uint64_t x) {
    uint64_t z = x + 0x9E3779B97F4A7C15ULL;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

/* u_i in [0,1): (splitmix64(seed ^ level*0x9E37.. ^ i) >> 11) * 2^-53 */
double pmis_u(uint64_t seed, int level, int64_t i) {
    uint64_t x = seed ^ ((uint64_t)(uint32_t)level * 0x9E3779B97F4A7C15ULL) ^ (uint64_t)i;
    return (double)(splitmix64(x) >> 11) * (1.0 / 9007199254740992.0);
}

/* i beats j: mu_i > mu_j, ties broken by the larger index. */
static inline int beats(double mi, int64_t i, double mj, int64_t j) {
    return mi > mj || (mi == mj && i > j);
}

/*
 * PMIS C/F splitting (synchronous rounds).
 *   S_i = {j != i : strong(i,j)},  S^T_i = {j : i in S_j}
 *   mu_i = |S^T_i| + u_i;  |S^T_i| == 0  =>  F.
 *   round: undecided i becomes C iff it beats every undecided
 *          j in S_i u S^T_i; then every undecided j with a C in S_j becomes F.
 * Returns the number of rounds; state_out[n].
 */
int pmis(int n, const int *indptr, const int *indices, const int8_t *strong,
         uint64_t seed, int level, int8_t *state) {
    int *tcnt = (int *)calloc((size_t)n + 1, sizeof(int));
    for (int i = 0; i < n; ++i)
        for (int e = indptr[i]; e < indptr[i + 1]; ++e)
            if (strong[e] && indices[e] != i) tcnt[indices[e] + 1]++;
    for (int i = 0; i < n; ++i) tcnt[i + 1] += tcnt[i];
    int *tind = (int *)malloc(sizeof(int) * (size_t)(tcnt[n] > 0 ? tcnt[n] : 1));
    int *fill = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) fill[i] = tcnt[i];
    for (int i = 0; i < n; ++i)
        for (int e = indptr[i]; e < indptr[i + 1]; ++e)
            if (strong[e] && indices[e] != i) tind[fill[indices[e]]++] = i;
    double *mu = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    int undecided = 0;
    for (int i = 0; i < n; ++i) {
        int st = tcnt[i + 1] - tcnt[i];
        mu[i] = (double)st + pmis_u(seed, level, i);
        state[i] = st == 0 ? FPOINT : UNDECIDED;
        undecided += st != 0;
    }
    int8_t *newc = (int8_t *)calloc((size_t)n + 1, 1);
    int rounds = 0;
    while (undecided > 0) {
        rounds++;
        for (int i = 0; i < n; ++i) {
            newc[i] = 0;
            if (state[i] != UNDECIDED) continue;
            int best = 1;
            for (int e = indptr[i]; e < indptr[i + 1] && best; ++e) {
                int j = indices[e];
                if (!strong[e] || j == i || state[j] != UNDECIDED) continue;
                if (!beats(mu[i], i, mu[j], j)) best = 0;
            }
            for (int e = tcnt[i]; e < tcnt[i + 1] && best; ++e) {
                int j = tind[e];
                if (state[j] != UNDECIDED) continue;
                if (!beats(mu[i], i, mu[j], j)) best = 0;
            }
            newc[i] = (int8_t)best;
        }
        for (int i = 0; i < n; ++i)
            if (newc[i]) { state[i] = CPOINT; undecided--; }
        for (int j = 0; j < n; ++j) {
            if (state[j] != UNDECIDED) continue;
            for (int e = indptr[j]; e < indptr[j + 1]; ++e) {
                int k = indices[e];
                if (strong[e] && k != j && state[k] == CPOINT) {
                    state[j] = FPOINT; undecided--; break;
                }
            }
        }
    }
    free(tcnt); free(tind); free(fill); free(mu); free(newc);
    return rounds;
}

/*
 * Pinned summation order for the extended+i scalar sums: TREE(t_0..t_{m-1})
 * = acc, acc = 0 then acc = acc + tree32(chunk) for each chunk of 32 terms
 * (zero padded), tree32(w) = for off in 16,8,4,2,1: w[l] = w[l] + w[l+off]
 * (l < off); return w[0].  This is the GPU's warp shuffle-down tree, so a
 * warp can form these sums in parallel and still match bit for bit.
 */
static double tree32(const double *t, int n) {
    double w[32];
    for (int l = 0; l < 32; ++l) w[l] = l < n ? t[l] : 0.0;
    for (int off = 16; off > 0; off >>= 1)
        for (int l = 0; l < off; ++l) w[l] = w[l] + w[l + off];
    return w[0];
}

static double tree_sum(const double *t, int m) {
    double acc = 0.0;
    for (int c = 0; c < m; c += 32) acc = acc + tree32(t + c, m - c < 32 ? m - c : 32);
    return acc;
}

static double row_diag(const int *indptr, const int *indices, const double *data, int k) {
    double d = 0.0;
    for (int e = indptr[k]; e < indptr[k + 1]; ++e)
        if (indices[e] == k) d = d + data[e];
    return d;
}

/* a_kl has the opposite sign of a_kk (zero entries never qualify). */
static inline int opposite(double v, double dkk) {
    return (v < 0.0 && dkk > 0.0) || (v > 0.0 && dkk < 0.0);
}

static int cmp_int(const void *a, const void *b) {
    int x = *(const int *)a, y = *(const int *)b;
    return (x > y) - (x < y);
}

typedef struct { double absw; int col; } wsel_t;
static int cmp_sel(const void *a, const void *b) {
    const wsel_t *x = (const wsel_t *)a, *y = (const wsel_t *)b;
    if (x->absw > y->absw) return -1;
    if (x->absw < y->absw) return 1;
    return (x->col > y->col) - (x->col < y->col);
}

/*
 * Extended+i interpolation, one F row:
 *   Chat_i = C^s_i  u  U_{k in F^s_i} C^s_k             (sorted, no value drop)
 *   abar_kl = a_kl if sign(a_kl) != sign(a_kk) else 0
 *   beta_k  = sum_{l in Chat_i u {i}} abar_kl            (row-k stored order)
 *   dt      = a_ii + sum_{weak n not in Chat_i} a_in
 *                  + sum_{k in F^s_i} (beta_k == 0 ? a_ik : (a_ik/beta_k)*abar_ki)
 *   w_ij    = -(a_ij + sum_k (a_ik/beta_k)*abar_kj) / dt   for j in Chat_i
 * Operation order: dt = a_ii + TREE(row-i lumps, row order), then per
 * strong-F k in row-i order either + a_ik (beta_k == 0) or + f*abar_ki;
 * beta_k = TREE(row k terms, row order); num[j] starts at 0, adds a_ij (if
 * stored), then f*abar_kj per k in row-i order.  TREE is the warp tree sum
 * defined at tree_sum() above.
 * Optional truncation to max_elmts largest |w| (ties: smaller column), kept
 * weights scaled by TREE(all w)/TREE(kept w) (column order) when the kept
 * sum is nonzero.
 * mode 0: count (cnt[i] = row length), mode 1: fill rows at p_indptr.
 * Columns are written as FINE indices (the caller maps to coarse ids).
 * Returns -1 on success, else the row with a zero interpolation pivot.
 */
static int ext_interp_impl(int n, const int *indptr, const int *indices, const double *data,
                           const int8_t *strong, const int8_t *state, int max_elmts,
                           int mode, int *cnt, const int64_t *p_indptr, int *p_col,
                           double *p_val) {
    int *mark = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int *pos = (int *)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) mark[i] = -1;
    int cap = 64;
    int *chat = (int *)malloc(sizeof(int) * cap);
    double *num = (double *)malloc(sizeof(double) * cap);
    wsel_t *sel = (wsel_t *)malloc(sizeof(wsel_t) * cap);
    int tcap = 64;
    double *terms = (double *)malloc(sizeof(double) * tcap);
    int bad = -1;
    for (int i = 0; i < n && bad < 0; ++i) {
        if (state[i] == CPOINT) {
            if (mode == 0) cnt[i] = 1;
            else { p_col[p_indptr[i]] = i; p_val[p_indptr[i]] = 1.0; }
            continue;
        }
        int m = 0;
#define PUSH(j) do { if (m == cap) { cap *= 2; chat = (int*)realloc(chat, sizeof(int)*cap); \
        num = (double*)realloc(num, sizeof(double)*cap); sel = (wsel_t*)realloc(sel, sizeof(wsel_t)*cap);} \
        chat[m++] = (j); mark[(j)] = i; } while (0)
        for (int e = indptr[i]; e < indptr[i + 1]; ++e) {
            int j = indices[e];
            if (j != i && strong[e] && state[j] == CPOINT && mark[j] != i) PUSH(j);
        }
        for (int e = indptr[i]; e < indptr[i + 1]; ++e) {
            int k = indices[e];
            if (k == i || !strong[e] || state[k] != FPOINT) continue;
            for (int e2 = indptr[k]; e2 < indptr[k + 1]; ++e2) {
                int l = indices[e2];
                if (l != k && strong[e2] && state[l] == CPOINT && mark[l] != i) PUSH(l);
            }
        }
#undef PUSH
        if (m == 0) { if (mode == 0) cnt[i] = 0; continue; }
        int outlen = (max_elmts > 0 && m > max_elmts) ? max_elmts : m;
        if (mode == 0) { cnt[i] = outlen; continue; }
        qsort(chat, (size_t)m, sizeof(int), cmp_int);
        for (int q = 0; q < m; ++q) { pos[chat[q]] = q; num[q] = 0.0; }
        /* scratch for TREE sums (row lengths and m) */
        int need = m;
        for (int e = indptr[i]; e < indptr[i + 1]; ++e) {
            int k = indices[e];
            int len = indptr[k + 1] - indptr[k];
            if (len > need) need = len;
        }
        if (indptr[i + 1] - indptr[i] > need) need = indptr[i + 1] - indptr[i];
        if (need > tcap) { tcap = need; terms = (double *)realloc(terms, sizeof(double) * tcap); }
        /* direct numerators */
        for (int e = indptr[i]; e < indptr[i + 1]; ++e) {
            int j = indices[e];
            if (j != i && mark[j] == i) num[pos[j]] = num[pos[j]] + data[e];
        }
        /* dt = a_ii + TREE(weak lumps in row order) */
        int nt = 0;
        for (int e = indptr[i]; e < indptr[i + 1]; ++e) {
            int j = indices[e];
            double t = 0.0;
            if (j != i && mark[j] != i && !(strong[e] && state[j] == FPOINT)) t = data[e];
            terms[nt++] = t;
        }
        double dt = row_diag(indptr, indices, data, i) + tree_sum(terms, nt);
        for (int e = indptr[i]; e < indptr[i + 1]; ++e) {
            int k = indices[e];
            if (k == i || !strong[e] || state[k] != FPOINT) continue;
            double akk = row_diag(indptr, indices, data, k);
            /* beta = TREE over row k of abar_kl, l in Chat u {i} */
            nt = 0;
            int at_i = -1;
            for (int e2 = indptr[k]; e2 < indptr[k + 1]; ++e2) {
                int l = indices[e2];
                double t = 0.0;
                if (l != k && opposite(data[e2], akk) && (l == i || mark[l] == i)) t = data[e2];
                if (l != k && l == i && opposite(data[e2], akk)) at_i = e2;
                terms[nt++] = t;
            }
            double beta = tree_sum(terms, nt);
            if (beta == 0.0) { dt = dt + data[e]; continue; }
            double f = data[e] / beta;
            for (int e2 = indptr[k]; e2 < indptr[k + 1]; ++e2) {
                int l = indices[e2];
                if (l == k || !opposite(data[e2], akk)) continue;
                if (mark[l] == i) num[pos[l]] = num[pos[l]] + f * data[e2];
            }
            if (at_i >= 0) dt = dt + f * data[at_i];
        }
        if (dt == 0.0) { bad = i; break; }
        for (int q = 0; q < m; ++q) num[q] = -num[q] / dt;
        int64_t o = p_indptr[i];
        if (outlen == m) {
            for (int q = 0; q < m; ++q) { p_col[o + q] = chat[q]; p_val[o + q] = num[q]; }
        } else {
            double s_all = tree_sum(num, m);
            for (int q = 0; q < m; ++q) { sel[q].absw = fabs(num[q]); sel[q].col = q; }
            qsort(sel, (size_t)m, sizeof(wsel_t), cmp_sel);
            /* kept positions, back in column order */
            int *keep = (int *)malloc(sizeof(int) * (size_t)outlen);
            for (int q = 0; q < outlen; ++q) keep[q] = sel[q].col;
            qsort(keep, (size_t)outlen, sizeof(int), cmp_int);
            for (int q = 0; q < m; ++q) terms[q] = 0.0;
            for (int q = 0; q < outlen; ++q) terms[keep[q]] = num[keep[q]];
            double s_kept = tree_sum(terms, m);
            double scale = s_kept != 0.0 ? s_all / s_kept : 1.0;
            for (int q = 0; q < outlen; ++q) {
                p_col[o + q] = chat[keep[q]];
                p_val[o + q] = num[keep[q]] * scale;
            }
            free(keep);
        }
    }
    free(mark); free(pos); free(chat); free(num); free(sel); free(terms);
    return bad;
}

int ext_interp_count(int n, const int *indptr, const int *indices, const double *data,
                     const int8_t *strong, const int8_t *state, int max_elmts, int *cnt) {
    return ext_interp_impl(n, indptr, indices, data, strong, state, max_elmts, 0, cnt,
                           NULL, NULL, NULL);
}

int ext_interp_fill(int n, const int *indptr, const int *indices, const double *data,
                    const int8_t *strong, const int8_t *state, int max_elmts,
                    const int64_t *p_indptr, int *p_col, double *p_val) {
    return ext_interp_impl(n, indptr, indices, data, strong, state, max_elmts, 1, NULL,
                           p_indptr, p_col, p_val);
}

/*
 * scipy-order SpGEMM C = A*B (the csr_matmat order):
 * for each row i, for j in A_i (stored order), for k in B_j (stored order)
 * sums[k] = sums[k] + a_ij*b_jk (separate multiply and add); exact zeros
 * dropped; columns sorted.  Used to cross-check the GPU SpGEMM and scipy.
 * mode 0 counts nonzeros per row into cnt; mode 1 fills.
 */
static int spgemm_impl(int m, int ncols, const int *ap, const int *aj, const double *ax,
                       const int *bp, const int *bj, const double *bx, int mode,
                       int *cnt, const int64_t *cp, int *cj, double *cx) {
    int *mark = (int *)malloc(sizeof(int) * (size_t)(ncols > 0 ? ncols : 1));
    double *sums = (double *)calloc((size_t)(ncols > 0 ? ncols : 1), sizeof(double));
    int *list = (int *)malloc(sizeof(int) * (size_t)(ncols > 0 ? ncols : 1));
    for (int k = 0; k < ncols; ++k) mark[k] = -1;
    for (int i = 0; i < m; ++i) {
        int len = 0;
        for (int e = ap[i]; e < ap[i + 1]; ++e) {
            int j = aj[e];
            double a = ax[e];
            for (int e2 = bp[j]; e2 < bp[j + 1]; ++e2) {
                int k = bj[e2];
                if (mark[k] != i) { mark[k] = i; sums[k] = 0.0; list[len++] = k; }
                sums[k] = sums[k] + a * bx[e2];
            }
        }
        qsort(list, (size_t)len, sizeof(int), cmp_int);
        int64_t o = mode ? cp[i] : 0;
        int c = 0;
        for (int q = 0; q < len; ++q) {
            int k = list[q];
            if (sums[k] != 0.0) {
                if (mode) { cj[o + c] = k; cx[o + c] = sums[k]; }
                c++;
            }
        }
        if (!mode) cnt[i] = c;
    }
    free(mark); free(sums); free(list);
    return 0;
}

int spgemm_count(int m, int ncols, const int *ap, const int *aj, const double *ax,
                 const int *bp, const int *bj, const double *bx, int *cnt) {
    return spgemm_impl(m, ncols, ap, aj, ax, bp, bj, bx, 0, cnt, NULL, NULL, NULL);
}

int spgemm_fill(int m, int ncols, const int *ap, const int *aj, const double *ax,
                const int *bp, const int *bj, const double *bx, const int64_t *cp,
                int *cj, double *cx) {
    return spgemm_impl(m, ncols, ap, aj, ax, bp, bj, bx, 1, NULL, cp, cj, cx);
}
