/*
 * oracle.c — plain, slow, single-threaded CPU oracle of the paper's method.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load or call this file.  The product library
 * (paper_2511_21268_b200/) shares no code with it and never calls it.
 *
 * Paper: D'Ambra, Durastante, Filippone, "Parallel matching-based AMG preconditioners for elliptic
 * equations discretized by IgA", arXiv 2511.21268.  Citations "P:Lnnn" are lines of PAPER.md;
 * "c.N" are the rows of SURVEY.md §8(c) whose readings DESIGN.md §3 adopts.
 *
 * Compile: gcc -O2 -ffp-contract=off -fPIC -shared (NO FMA contraction: the canonical arithmetic
 * contract of DESIGN.md §3 — every expression is evaluated exactly in the order written here,
 * every sum is sequential in ascending index order starting from +0.0).
 *
 * Functions and the passage each follows:
 *   or_assemble      c.4  K = K1⊗M1⊗M1 + M1⊗K1⊗M1 + M1⊗M1⊗K1 (eq:matrix_and_vector_values
 *                         P:L646-650), Dirichlet DOFs eliminated
 *   or_spmv          y = A x
 *   or_setup         c.6-c.15: compatible weighted matching (eq:cij P:L766-771, eq:maxprod
 *                    P:L794-809), pairwise prolongation (eq:prolongation P:L811-834), 3-step
 *                    aggregation, smoothed prolongator, Galerkin
 *                    K_{l+1} = R K_l P (eq:galerkin_matrix_projection P:L664-667), ℓ1 diagonal
 *                    (P:L877-880), coarse stop
 *   or_vcycle        c.16-c.18: V-cycle with 4th-kind Chebyshev-ℓ1-Jacobi smoothing
 *                     and 30 ℓ1-Jacobi sweeps on the coarsest level
 *   or_pcg           c.19: preconditioned CG, rtol test on the
 *                    recurrence residual
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_MAX_LEVELS 32

typedef struct {
    int64_t nrows, ncols, nnz;
    int64_t *rp;   /* nrows+1 */
    int32_t *ci;   /* nnz, ascending within each row */
    double *v;     /* nnz */
} ocsr;

typedef struct {
    int agg_steps;          /* pairwise matching steps per level (3 -> aggregates <= 8) */
    int smooth_prolong;     /* 1: P̄ = (I - ω D_f^{-1} K_f) P ; 0: tentative P */
    double match_threshold; /* edge (i,j) eligible iff c_ij > threshold (1.0) */
    double filter_theta;    /* strong iff |k_ij| >= θ sqrt(k_ii k_jj) (0.01) */
    int cheb_degree;        /* m: number of SpMVs per smoothing application */
    int coarse_sweeps;      /* ℓ1-Jacobi sweeps on the coarsest level (30) */
    int64_t coarse_size;    /* stop when N_l <= coarse_size (50) */
    int max_levels;         /* 20 */
    /* coarsest-level solver: 0 = coarse_sweeps ℓ1-Jacobi sweeps (§4; c.17);
     * 1 = CG preconditioned by one weighted-Jacobi sweep, to coarse_tol relative or coarse_maxit
     *     iterations (§5.1) */
    int coarse_solver;
    double coarse_tol;      /* 1e-4 */
    int coarse_maxit;       /* 30 */
    /* Study knobs for readings the paper leaves open (c.8 / c.12); 0 = the canonical
     * reading every parity test uses.  Only oracle/scripts/opc_study.py sets them.
     *   tie_break : order of edges with equal c_ij.  0: (i asc, j asc) for i < j — each vertex prefers
     *               its smaller-index partner; 1: (j desc, i desc) — prefers the larger index;
     *               2 + s: a fixed pseudo-random order (splitmix64 of (i, j) with seed s, then i, j).
     *   omega_norm: 0: λ̂ = ‖D_f⁻¹K_f‖∞ of the filtered matrix (c.12); 1: ‖D⁻¹K‖∞ of K itself. */
    int tie_break;
    int omega_norm;
} oparams;

typedef struct {
    int64_t N;
    ocsr K;          /* level operator K_l */
    ocsr P;          /* prolongator P̄_l: N_l x N_{l+1} (empty on the coarsest level) */
    ocsr R;          /* R_l = P̄_lᵀ */
    int32_t *agg;    /* composite aggregate of each row (tentative P column) */
    double *ptent;   /* composite tentative P value of each row */
    double *dhat;    /* ℓ1 diagonal */
    double *w;       /* test vector used on this level */
    double omega;    /* prolongator damping (0 if unsmoothed / coarsest) */
} olevel;

typedef struct {
    oparams prm;
    int nlevels;
    olevel lev[OR_MAX_LEVELS];
} ohier;

/* ------------------------------------------------------------------------------------------ */
/* CSR helpers                                                                                 */
/* ------------------------------------------------------------------------------------------ */

static void csr_free(ocsr *A) {
    free(A->rp); free(A->ci); free(A->v);
    memset(A, 0, sizeof(*A));
}

static int csr_alloc(ocsr *A, int64_t nrows, int64_t ncols, int64_t nnz) {
    A->nrows = nrows; A->ncols = ncols; A->nnz = nnz;
    A->rp = (int64_t *)calloc((size_t)nrows + 1, sizeof(int64_t));
    A->ci = (int32_t *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(int32_t));
    A->v = (double *)malloc((size_t)(nnz > 0 ? nnz : 1) * sizeof(double));
    return (A->rp && A->ci && A->v) ? 0 : -2;
}

/* Transpose; row J of the result lists the source rows i in ascending order. */
static int csr_transpose(const ocsr *A, ocsr *T) {
    if (csr_alloc(T, A->ncols, A->nrows, A->nnz)) return -2;
    for (int64_t k = 0; k < A->nnz; k++) T->rp[A->ci[k] + 1]++;
    for (int64_t j = 0; j < A->ncols; j++) T->rp[j + 1] += T->rp[j];
    int64_t *pos = (int64_t *)malloc(((size_t)A->ncols + 1) * sizeof(int64_t));
    if (!pos) return -2;
    memcpy(pos, T->rp, ((size_t)A->ncols + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < A->nrows; i++)
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; k++) {
            int64_t d = pos[A->ci[k]]++;
            T->ci[d] = (int32_t)i;
            T->v[d] = A->v[k];
        }
    free(pos);
    return 0;
}

/* Row-wise sparse accumulator ("Gustavson"): acc starts at +0.0 for every touched column and
 * receives contributions in the order they are produced; the row's pattern is the set of
 * touched columns (structural, even where the sum is 0), emitted in ascending order. */
typedef struct {
    double *acc;
    int64_t *stamp;
    int32_t *cols;
    int64_t ncols_touched;
    int64_t row;
} spa;

static int spa_init(spa *s, int64_t ncols) {
    s->acc = (double *)malloc((size_t)(ncols > 0 ? ncols : 1) * sizeof(double));
    s->stamp = (int64_t *)malloc((size_t)(ncols > 0 ? ncols : 1) * sizeof(int64_t));
    s->cols = (int32_t *)malloc((size_t)(ncols > 0 ? ncols : 1) * sizeof(int32_t));
    if (!s->acc || !s->stamp || !s->cols) return -2;
    for (int64_t j = 0; j < ncols; j++) s->stamp[j] = -1;
    s->ncols_touched = 0;
    s->row = 0;
    return 0;
}
static void spa_free(spa *s) { free(s->acc); free(s->stamp); free(s->cols); }
static void spa_start(spa *s, int64_t row) { s->row = row; s->ncols_touched = 0; }
static void spa_add(spa *s, int32_t j, double x) {
    if (s->stamp[j] != s->row) {
        s->stamp[j] = s->row;
        s->acc[j] = 0.0;
        s->cols[s->ncols_touched++] = j;
    }
    s->acc[j] = s->acc[j] + x;
}
static int cmp_i32(const void *a, const void *b) {
    int32_t x = *(const int32_t *)a, y = *(const int32_t *)b;
    return (x > y) - (x < y);
}

/* Growable CSR builder used by the products below. */
typedef struct {
    ocsr A;
    int64_t cap;
} cbuild;

static int cb_init(cbuild *b, int64_t nrows, int64_t ncols, int64_t cap) {
    if (cap < 16) cap = 16;
    if (csr_alloc(&b->A, nrows, ncols, cap)) return -2;
    b->A.nnz = 0;
    b->cap = cap;
    return 0;
}
static int cb_push(cbuild *b, int32_t j, double v) {
    if (b->A.nnz == b->cap) {
        b->cap *= 2;
        int32_t *ci = (int32_t *)realloc(b->A.ci, (size_t)b->cap * sizeof(int32_t));
        double *vv = (double *)realloc(b->A.v, (size_t)b->cap * sizeof(double));
        if (!ci || !vv) return -2;
        b->A.ci = ci; b->A.v = vv;
    }
    b->A.ci[b->A.nnz] = j;
    b->A.v[b->A.nnz] = v;
    b->A.nnz++;
    return 0;
}
/* Flush the accumulator as row i (ascending columns). */
static int cb_flush(cbuild *b, spa *s, int64_t i) {
    qsort(s->cols, (size_t)s->ncols_touched, sizeof(int32_t), cmp_i32);
    for (int64_t t = 0; t < s->ncols_touched; t++)
        if (cb_push(b, s->cols[t], s->acc[s->cols[t]])) return -2;
    b->A.rp[i + 1] = b->A.nnz;
    return 0;
}

static double csr_get(const ocsr *A, int64_t i, int32_t j, int *found) {
    int64_t lo = A->rp[i], hi = A->rp[i + 1] - 1;
    while (lo <= hi) {
        int64_t mid = (lo + hi) / 2;
        if (A->ci[mid] == j) { *found = 1; return A->v[mid]; }
        if (A->ci[mid] < j) lo = mid + 1; else hi = mid - 1;
    }
    *found = 0;
    return 0.0;
}

/* A <- 0.5 (A + Aᵀ) entrywise on the structural union of the two patterns (c.10, c.13;
 * SPEC S:L57).  Missing entries count as +0.0.  (a + b) * 0.5 is commutative in IEEE
 * arithmetic, so the result is bitwise symmetric. */
static int csr_symmetrize(ocsr *A) {
    ocsr T;
    if (csr_transpose(A, &T)) return -2;
    cbuild b;
    if (cb_init(&b, A->nrows, A->ncols, A->nnz + 16)) return -2;
    for (int64_t i = 0; i < A->nrows; i++) {
        int64_t ka = A->rp[i], kt = T.rp[i];
        while (ka < A->rp[i + 1] || kt < T.rp[i + 1]) {
            int32_t ja = ka < A->rp[i + 1] ? A->ci[ka] : INT32_MAX;
            int32_t jt = kt < T.rp[i + 1] ? T.ci[kt] : INT32_MAX;
            double a = 0.0, t = 0.0;
            int32_t j;
            if (ja == jt) { j = ja; a = A->v[ka++]; t = T.v[kt++]; }
            else if (ja < jt) { j = ja; a = A->v[ka++]; }
            else { j = jt; t = T.v[kt++]; }
            if (cb_push(&b, j, (a + t) * 0.5)) return -2;
        }
        b.A.rp[i + 1] = b.A.nnz;
    }
    csr_free(&T);
    csr_free(A);
    *A = b.A;
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* c.4 — stiffness by the Kronecker sum of exact 1-D tables                                    */
/* ------------------------------------------------------------------------------------------ */

/* M1, K1: band storage (m x (2p+1)), band[a*(2p+1) + (b-a+p)] = table(a,b), m = n+p.
 * dirmask: bit s-1 set <=> side s Dirichlet (1:x=0 2:x=1 3:y=0 4:y=1 5:z=0 6:z=1).
 * Free DOFs numbered lexicographically, x fastest (c.1). For free rows (a,b,c), (a',b',c') with
 * |a-a'|,|b-b'|,|c-c'| <= p (structural pattern, c.4):
 *   t1 = (K1[a,a']·M1[b,b'])·M1[c,c'];  t2 = (M1[a,a']·K1[b,b'])·M1[c,c'];
 *   t3 = (M1[a,a']·M1[b,b'])·K1[c,c'];  k = (t1 + t2) + t3.
 * 2-D: k = K1[a,a']·M1[b,b'] + M1[a,a']·K1[b,b']. */
int or_assemble(int dim, int p, int n, int dirmask, const double *M1, const double *K1, ocsr *K) {
    const int m = n + p, bw = 2 * p + 1;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0}, nf[3] = {1, 1, 1};
    if (dim != 2 && dim != 3) return -1;
    for (int ax = 0; ax < dim; ax++) {
        lo[ax] = (dirmask >> (2 * ax)) & 1 ? 1 : 0;
        hi[ax] = m - 1 - ((dirmask >> (2 * ax + 1)) & 1 ? 1 : 0);
        nf[ax] = hi[ax] - lo[ax] + 1;
    }
    int64_t N = (int64_t)nf[0] * nf[1] * nf[2];
    /* count */
    int64_t nnz = 0;
    int64_t *rp = (int64_t *)calloc((size_t)N + 1, sizeof(int64_t));
    if (!rp) return -2;
    for (int c = lo[2]; c <= hi[2]; c++)
        for (int b = lo[1]; b <= hi[1]; b++)
            for (int a = lo[0]; a <= hi[0]; a++) {
                int64_t row = (int64_t)(a - lo[0]) + (int64_t)nf[0] * ((b - lo[1]) + (int64_t)nf[1] * (c - lo[2]));
                int64_t cnt = 1;
                for (int ax = 0; ax < dim; ax++) {
                    int x = ax == 0 ? a : ax == 1 ? b : c;
                    int l = x - p > lo[ax] ? x - p : lo[ax];
                    int h = x + p < hi[ax] ? x + p : hi[ax];
                    cnt *= (h - l + 1);
                }
                rp[row + 1] = cnt;
            }
    for (int64_t i = 0; i < N; i++) rp[i + 1] += rp[i];
    nnz = rp[N];
    K->nrows = K->ncols = N;
    K->nnz = nnz;
    K->rp = rp;
    K->ci = (int32_t *)malloc((size_t)nnz * sizeof(int32_t));
    K->v = (double *)malloc((size_t)nnz * sizeof(double));
    if (!K->ci || !K->v) return -2;
    int64_t k = 0;
    for (int c = lo[2]; c <= hi[2]; c++)
        for (int b = lo[1]; b <= hi[1]; b++)
            for (int a = lo[0]; a <= hi[0]; a++) {
                int cl = dim == 3 ? (c - p > lo[2] ? c - p : lo[2]) : c;
                int ch = dim == 3 ? (c + p < hi[2] ? c + p : hi[2]) : c;
                for (int c2 = cl; c2 <= ch; c2++) {
                    int bl = b - p > lo[1] ? b - p : lo[1];
                    int bh = b + p < hi[1] ? b + p : hi[1];
                    for (int b2 = bl; b2 <= bh; b2++) {
                        int al = a - p > lo[0] ? a - p : lo[0];
                        int ah = a + p < hi[0] ? a + p : hi[0];
                        for (int a2 = al; a2 <= ah; a2++) {
                            double Ka = K1[a * bw + (a2 - a + p)], Ma = M1[a * bw + (a2 - a + p)];
                            double Kb = K1[b * bw + (b2 - b + p)], Mb = M1[b * bw + (b2 - b + p)];
                            double val;
                            if (dim == 3) {
                                double Kc = K1[c * bw + (c2 - c + p)], Mc = M1[c * bw + (c2 - c + p)];
                                double t1 = (Ka * Mb) * Mc;
                                double t2 = (Ma * Kb) * Mc;
                                double t3 = (Ma * Mb) * Kc;
                                val = (t1 + t2) + t3;
                            } else {
                                double t1 = Ka * Mb;
                                double t2 = Ma * Kb;
                                val = t1 + t2;
                            }
                            K->ci[k] = (int32_t)((a2 - lo[0]) + (int64_t)nf[0] * ((b2 - lo[1]) + (int64_t)nf[1] * (c2 - lo[2])));
                            K->v[k] = val;
                            k++;
                        }
                    }
                }
            }
    return k == nnz ? 0 : -3;
}

/* y_i = Σ_j a_ij x_j, j ascending, from +0.0. */
void or_spmv(const ocsr *A, const double *x, double *y) {
    for (int64_t i = 0; i < A->nrows; i++) {
        double s = 0.0;
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; k++) s = s + A->v[k] * x[A->ci[k]];
        y[i] = s;
    }
}

/* ------------------------------------------------------------------------------------------ */
/* c.7/c.8 — compatibility weights and the greedy (= locally dominant) matching                 */
/* ------------------------------------------------------------------------------------------ */

typedef struct { double c; int32_t i, j; } oedge;

static int g_tie_break = 0; /* oparams.tie_break of the running or_setup (study knob; 0 = canonical) */

static uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

/* Strict total order: c descending, then i ascending, then j ascending (c.8).  (tie_break 1 / 2:
 * the study orders of the oparams comment.) */
static int cmp_edge(const void *pa, const void *pb) {
    const oedge *a = (const oedge *)pa, *b = (const oedge *)pb;
    if (a->c > b->c) return -1;
    if (a->c < b->c) return 1;
    if (g_tie_break == 1) {
        if (a->j != b->j) return a->j > b->j ? -1 : 1;
        if (a->i != b->i) return a->i > b->i ? -1 : 1;
        return 0;
    }
    if (g_tie_break >= 2) { /* seed = tie_break − 2 */
        const uint64_t seed = (uint64_t)(g_tie_break - 2) * 0xD1B54A32D192ED03ull;
        uint64_t ha = mix64(seed ^ (((uint64_t)(uint32_t)a->i << 32) | (uint32_t)a->j));
        uint64_t hb = mix64(seed ^ (((uint64_t)(uint32_t)b->i << 32) | (uint32_t)b->j));
        if (ha != hb) return ha < hb ? -1 : 1;
    }
    if (a->i != b->i) return a->i < b->i ? -1 : 1;
    if (a->j != b->j) return a->j < b->j ? -1 : 1;
    return 0;
}

static int get_diag(const ocsr *A, double *diag) {
    for (int64_t i = 0; i < A->nrows; i++) {
        int found;
        diag[i] = csr_get(A, i, (int32_t)i, &found);
        if (!found) return -5;
    }
    return 0;
}

/* eq:cij, evaluated for the ordered pair i < j exactly as written in c.7:
 *   num = ((2·k_ij)·w_i)·w_j ;  den = (k_ii·w_i)·w_i + (k_jj·w_j)·w_j ;  c = 1 − num/den. */
double or_cij(double kij, double kii, double kjj, double wi, double wj) {
    double num = ((2.0 * kij) * wi) * wj;
    double den = (kii * wi) * wi + (kjj * wj) * wj;
    return 1.0 - num / den;
}

/* One pairwise aggregation step (c.7-c.9).  Outputs:
 *   mate[i]  : matched partner or -1;
 *   agg[i]   : aggregate index, aggregates numbered in ascending order of their minimum member;
 *   pv[i]    : P[i, agg[i]] (eq:prolongation P:L811-834, "no reordering");
 *   wn[I]    : coarse test vector (‖w_e‖ for a pair, |w_s| for a singleton).
 * Returns the number of aggregates, or < 0 on error. */
int64_t or_pairwise(const ocsr *A, const double *w, double thr, int32_t *mate, int32_t *agg,
                    double *pv, double *wn) {
    const int64_t N = A->nrows;
    double *diag = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    if (!diag) return -2;
    if (get_diag(A, diag)) { free(diag); return -5; }
    int64_t ne = 0;
    for (int64_t i = 0; i < N; i++)
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; k++)
            if (A->ci[k] > i) ne++;
    oedge *E = (oedge *)malloc((size_t)(ne > 0 ? ne : 1) * sizeof(oedge));
    if (!E) { free(diag); return -2; }
    int64_t m = 0;
    for (int64_t i = 0; i < N; i++)
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; k++) {
            int32_t j = A->ci[k];
            if (j <= i) continue;
            double c = or_cij(A->v[k], diag[i], diag[j], w[i], w[j]);
            if (c > thr) { E[m].c = c; E[m].i = (int32_t)i; E[m].j = j; m++; }
        }
    qsort(E, (size_t)m, sizeof(oedge), cmp_edge);
    for (int64_t i = 0; i < N; i++) mate[i] = -1;
    for (int64_t e = 0; e < m; e++)
        if (mate[E[e].i] < 0 && mate[E[e].j] < 0) {
            mate[E[e].i] = E[e].j;
            mate[E[e].j] = E[e].i;
        }
    free(E);
    free(diag);
    int64_t nc = 0;
    for (int64_t i = 0; i < N; i++) {
        int32_t j = mate[i];
        if (j < 0) {
            agg[i] = (int32_t)nc;
            pv[i] = w[i] / fabs(w[i]);
            wn[nc] = fabs(w[i]);
            nc++;
        } else if (i < j) {
            double nrm = sqrt(w[i] * w[i] + w[j] * w[j]);
            agg[i] = agg[j] = (int32_t)nc;
            pv[i] = w[i] / nrm;
            pv[j] = w[j] / nrm;
            wn[nc] = nrm;
            nc++;
        }
    }
    return nc;
}

/* c.10: A_{s+1}[I,J] = Σ_{i∈I asc} Σ_{j stored in row i, asc} P[i,I]·(A_s[i,j]·P[j,J]); then
 * symmetrised. */
static int galerkin_pairwise(const ocsr *A, const int32_t *agg, const double *pv, int64_t nc, ocsr *Ac) {
    const int64_t N = A->nrows;
    /* members of each aggregate, ascending */
    int64_t *mp = (int64_t *)calloc((size_t)nc + 1, sizeof(int64_t));
    int32_t *mem = (int32_t *)malloc((size_t)(N > 0 ? N : 1) * sizeof(int32_t));
    if (!mp || !mem) return -2;
    for (int64_t i = 0; i < N; i++) mp[agg[i] + 1]++;
    for (int64_t I = 0; I < nc; I++) mp[I + 1] += mp[I];
    int64_t *pos = (int64_t *)malloc(((size_t)nc + 1) * sizeof(int64_t));
    memcpy(pos, mp, ((size_t)nc + 1) * sizeof(int64_t));
    for (int64_t i = 0; i < N; i++) mem[pos[agg[i]]++] = (int32_t)i;
    free(pos);
    spa s;
    cbuild b;
    if (spa_init(&s, nc) || cb_init(&b, nc, nc, A->nnz)) return -2;
    for (int64_t I = 0; I < nc; I++) {
        spa_start(&s, I);
        for (int64_t t = mp[I]; t < mp[I + 1]; t++) {
            int32_t i = mem[t];
            for (int64_t k = A->rp[i]; k < A->rp[i + 1]; k++) {
                int32_t j = A->ci[k];
                spa_add(&s, agg[j], pv[i] * (A->v[k] * pv[j]));
            }
        }
        if (cb_flush(&b, &s, I)) return -2;
    }
    spa_free(&s);
    free(mp); free(mem);
    *Ac = b.A;
    return csr_symmetrize(Ac);
}

/* ------------------------------------------------------------------------------------------ */
/* c.12 — filtered smoothed prolongator;  c.13 — Galerkin coarse operator                     */
/* ------------------------------------------------------------------------------------------ */

/* K_f: keep the diagonal and the strong entries (|k_ij| >= θ·sqrt(k_ii·k_jj)); weak entries are
 * lumped onto the diagonal: K_f[i,i] = k_ii + s, s = Σ_{weak j asc} k_ij (from +0.0). */
static int filter_matrix(const ocsr *K, double theta, ocsr *Kf) {
    const int64_t N = K->nrows;
    double *diag = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    if (!diag) return -2;
    if (get_diag(K, diag)) { free(diag); return -5; }
    cbuild b;
    if (cb_init(&b, N, K->ncols, K->nnz)) return -2;
    for (int64_t i = 0; i < N; i++) {
        double s = 0.0;
        for (int64_t k = K->rp[i]; k < K->rp[i + 1]; k++) {
            int32_t j = K->ci[k];
            if (j == i) continue;
            if (!(fabs(K->v[k]) >= theta * sqrt(diag[i] * diag[j]))) s = s + K->v[k];
        }
        for (int64_t k = K->rp[i]; k < K->rp[i + 1]; k++) {
            int32_t j = K->ci[k];
            if (j == i) {
                if (cb_push(&b, j, diag[i] + s)) return -2;
            } else if (fabs(K->v[k]) >= theta * sqrt(diag[i] * diag[j])) {
                if (cb_push(&b, j, K->v[k])) return -2;
            }
        }
        b.A.rp[i + 1] = b.A.nnz;
    }
    free(diag);
    *Kf = b.A;
    return 0;
}

/* P̄ = (I − ω D⁻¹ K_f) P with D = diag(K_f), ω = 4/(3 λ̂), λ̂ = ‖D⁻¹K_f‖_∞ (c.12).
 *   t_iJ = Σ_{j in K_f row i, asc} K_f[i,j]·P[j,J];   P̄[i,J] = P[i,J] − (ω·t_iJ)/K_f[i,i]. */
static int smoothed_prolongator(const ocsr *K, const int32_t *agg, const double *pt, int64_t nc,
                                double theta, int omega_norm, ocsr *Pb, double *omega_out) {
    ocsr Kf;
    int rc = filter_matrix(K, theta, &Kf);
    if (rc) return rc;
    const int64_t N = K->nrows;
    double *df = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    if (!df) return -2;
    if (get_diag(&Kf, df)) return -5;
    double lam = 0.0;
    const ocsr *Kn = omega_norm == 1 ? K : &Kf; /* study knob: norm of K itself instead of K_f */
    for (int64_t i = 0; i < N; i++) {
        double s = 0.0, dii = 0.0;
        for (int64_t k = Kn->rp[i]; k < Kn->rp[i + 1]; k++) {
            s = s + fabs(Kn->v[k]);
            if (Kn->ci[k] == i) dii = Kn->v[k];
        }
        double q = s / (omega_norm == 1 ? dii : df[i]);
        if (q > lam) lam = q;
    }
    double omega = 4.0 / (3.0 * lam);
    spa s;
    cbuild b;
    if (spa_init(&s, nc) || cb_init(&b, N, nc, Kf.nnz)) return -2;
    for (int64_t i = 0; i < N; i++) {
        spa_start(&s, i);
        for (int64_t k = Kf.rp[i]; k < Kf.rp[i + 1]; k++) {
            int32_t j = Kf.ci[k];
            spa_add(&s, agg[j], Kf.v[k] * pt[j]);
        }
        qsort(s.cols, (size_t)s.ncols_touched, sizeof(int32_t), cmp_i32);
        for (int64_t t = 0; t < s.ncols_touched; t++) {
            int32_t J = s.cols[t];
            double pij = (J == agg[i]) ? pt[i] : 0.0;
            if (cb_push(&b, J, pij - (omega * s.acc[J]) / df[i])) return -2;
        }
        b.A.rp[i + 1] = b.A.nnz;
    }
    spa_free(&s);
    free(df);
    csr_free(&Kf);
    *Pb = b.A;
    *omega_out = omega;
    return 0;
}

/* C = A·B, row-wise, contributions in the order (k in row i of A ascending, then row k of B
 * ascending), each product a_ik·b_kj (c.13). */
static int csr_matmul(const ocsr *A, const ocsr *B, ocsr *C) {
    spa s;
    cbuild b;
    if (spa_init(&s, B->ncols) || cb_init(&b, A->nrows, B->ncols, A->nnz + B->nnz)) return -2;
    for (int64_t i = 0; i < A->nrows; i++) {
        spa_start(&s, i);
        for (int64_t k = A->rp[i]; k < A->rp[i + 1]; k++) {
            int32_t j = A->ci[k];
            double a = A->v[k];
            for (int64_t t = B->rp[j]; t < B->rp[j + 1]; t++) spa_add(&s, B->ci[t], a * B->v[t]);
        }
        if (cb_flush(&b, &s, i)) return -2;
    }
    spa_free(&s);
    *C = b.A;
    return 0;
}

static void l1_diag(const ocsr *K, double *d) {
    for (int64_t i = 0; i < K->nrows; i++) {
        double s = 0.0;
        for (int64_t k = K->rp[i]; k < K->rp[i + 1]; k++) s = s + fabs(K->v[k]);
        d[i] = s;
    }
}

static int csr_copy(const ocsr *A, ocsr *B) {
    if (csr_alloc(B, A->nrows, A->ncols, A->nnz)) return -2;
    memcpy(B->rp, A->rp, ((size_t)A->nrows + 1) * sizeof(int64_t));
    memcpy(B->ci, A->ci, (size_t)A->nnz * sizeof(int32_t));
    memcpy(B->v, A->v, (size_t)A->nnz * sizeof(double));
    return 0;
}

void or_hier_free(ohier *H) {
    if (!H) return;
    for (int l = 0; l < H->nlevels; l++) {
        olevel *L = &H->lev[l];
        csr_free(&L->K); csr_free(&L->P); csr_free(&L->R);
        free(L->agg); free(L->ptent); free(L->dhat); free(L->w);
    }
    free(H);
}

/* Hierarchy (c.6-c.15).  Level l: if N_l <= coarse_size or l == max_levels-1 -> coarsest.
 * Otherwise agg_steps pairwise steps on the intermediate Galerkin operators with the carried test
 * vector (w^(0) = 1, c.6), composite P (c.11), P̄ (c.12), R = P̄ᵀ, K_{l+1} = sym(R (K P̄)) (c.13).
 * A composite step that does not reduce N makes the level the coarsest (c.14). */
int or_setup(const ocsr *K0, const oparams *prm, ohier **out) {
    ohier *H = (ohier *)calloc(1, sizeof(ohier));
    if (!H) return -2;
    H->prm = *prm;
    g_tie_break = prm->tie_break;
    int rc = csr_copy(K0, &H->lev[0].K);
    if (rc) return rc;
    int64_t N0 = K0->nrows;
    H->lev[0].N = N0;
    H->lev[0].w = (double *)malloc((size_t)(N0 > 0 ? N0 : 1) * sizeof(double));
    for (int64_t i = 0; i < N0; i++) H->lev[0].w[i] = 1.0;
    int l = 0;
    for (;;) {
        olevel *L = &H->lev[l];
        const int64_t N = L->N;
        L->dhat = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
        l1_diag(&L->K, L->dhat);
        H->nlevels = l + 1;
        if (N <= prm->coarse_size || l + 1 >= prm->max_levels || l + 1 >= OR_MAX_LEVELS) break;
        /* agg_steps pairwise matchings (c.7-c.11) */
        int32_t *agg = (int32_t *)malloc((size_t)N * sizeof(int32_t));
        double *pt = (double *)malloc((size_t)N * sizeof(double));
        int32_t *mate = (int32_t *)malloc((size_t)N * sizeof(int32_t));
        int32_t *aggs = (int32_t *)malloc((size_t)N * sizeof(int32_t));
        double *pvs = (double *)malloc((size_t)N * sizeof(double));
        double *w = (double *)malloc((size_t)N * sizeof(double));
        double *wn = (double *)malloc((size_t)N * sizeof(double));
        if (!agg || !pt || !mate || !aggs || !pvs || !w || !wn) return -2;
        for (int64_t i = 0; i < N; i++) { agg[i] = (int32_t)i; pt[i] = 1.0; }
        memcpy(w, L->w, (size_t)N * sizeof(double));
        ocsr A;
        if (csr_copy(&L->K, &A)) return -2;
        int64_t nc = N;
        for (int s = 0; s < prm->agg_steps; s++) {
            int64_t ncs = or_pairwise(&A, w, prm->match_threshold, mate, aggs, pvs, wn);
            if (ncs < 0) return (int)ncs;
            /* compose: P[i, a_s(agg(i))] = P[i,agg(i)] · p_s[agg(i)]  (left to right, c.11) */
            for (int64_t i = 0; i < N; i++) {
                int32_t a = agg[i];
                pt[i] = pt[i] * pvs[a];
                agg[i] = aggs[a];
            }
            if (s + 1 < prm->agg_steps) {
                ocsr Ac;
                rc = galerkin_pairwise(&A, aggs, pvs, ncs, &Ac);
                if (rc) return rc;
                csr_free(&A);
                A = Ac;
            }
            memcpy(w, wn, (size_t)ncs * sizeof(double));
            nc = ncs;
        }
        csr_free(&A);
        free(mate); free(aggs); free(pvs); free(wn);
        if (nc == N) { free(agg); free(pt); free(w); break; }
        L->agg = agg;
        L->ptent = pt;
        /* c.12 */
        if (prm->smooth_prolong) {
            rc = smoothed_prolongator(&L->K, agg, pt, nc, prm->filter_theta, prm->omega_norm, &L->P, &L->omega);
            if (rc) return rc;
        } else {
            if (csr_alloc(&L->P, N, nc, N)) return -2;
            for (int64_t i = 0; i < N; i++) { L->P.rp[i + 1] = i + 1; L->P.ci[i] = agg[i]; L->P.v[i] = pt[i]; }
            L->omega = 0.0;
        }
        /* c.13 */
        if (csr_transpose(&L->P, &L->R)) return -2;
        ocsr AP, Kc;
        if (csr_matmul(&L->K, &L->P, &AP)) return -2;
        if (csr_matmul(&L->R, &AP, &Kc)) return -2;
        csr_free(&AP);
        if (csr_symmetrize(&Kc)) return -2;
        olevel *C = &H->lev[l + 1];
        C->K = Kc;
        C->N = nc;
        C->w = (double *)realloc(w, (size_t)(nc > 0 ? nc : 1) * sizeof(double));
        l++;
    }
    g_tie_break = 0;
    *out = H;
    return 0;
}

/* ------------------------------------------------------------------------------------------ */
/* c.16 — 4th-kind Chebyshev-accelerated ℓ1-Jacobi, ρ = 1 (Lottes)         */
/* ------------------------------------------------------------------------------------------ */

/* x <- S(b, x): m SpMVs.  x_is_zero: x on entry is 0 (r0 = b without an SpMV).
 *   r0 = b − K x;  d0 = (4/3)·(r0/d̂);  x += d0;
 *   for i = 1..m−1:  r −= K d_{i−1};  d_i = ((2i−1)/(2i+3))·d_{i−1} + ((8i+4)/(2i+3))·(r/d̂);  x += d_i. */
static void smooth(const olevel *L, int m, const double *b, double *x, int x_is_zero, double *r,
                   double *d, double *t) {
    const int64_t N = L->N;
    if (x_is_zero) {
        for (int64_t i = 0; i < N; i++) r[i] = b[i];
    } else {
        or_spmv(&L->K, x, t);
        for (int64_t i = 0; i < N; i++) r[i] = b[i] - t[i];
    }
    for (int64_t i = 0; i < N; i++) {
        d[i] = (4.0 / 3.0) * (r[i] / L->dhat[i]);
        x[i] = x[i] + d[i];
    }
    for (int i = 1; i < m; i++) {
        double ai = (double)(2 * i - 1) / (double)(2 * i + 3);
        double bi = (double)(8 * i + 4) / (double)(2 * i + 3);
        or_spmv(&L->K, d, t);
        for (int64_t k = 0; k < N; k++) {
            r[k] = r[k] - t[k];
            d[k] = ai * d[k] + bi * (r[k] / L->dhat[k]);
            x[k] = x[k] + d[k];
        }
    }
}

/* c.17: x = 0; repeat sweeps times: x_i <- x_i + (b_i − Σ_j k_ij x_j)/d̂_i  (Jacobi, old x). */
static void coarse_solve(const olevel *L, int sweeps, const double *b, double *x, double *t) {
    const int64_t N = L->N;
    for (int64_t i = 0; i < N; i++) x[i] = 0.0;
    for (int s = 0; s < sweeps; s++) {
        or_spmv(&L->K, x, t);
        for (int64_t i = 0; i < N; i++) x[i] = x[i] + (b[i] - t[i]) / L->dhat[i];
    }
}

/* §5.1 coarsest solver ("the CG preconditioned by a single sweep of weighted Jacobi as coarse
 * solver set to achieve a tolerance of 10^{-4} or stop in 30 iterations"): PCG from x = 0 with
 * z = D⁻¹ r, D = diag(K_L).  One weighted-Jacobi sweep from 0 is ω D⁻¹ r; CG is invariant under the
 * scalar ω, so the (unstated) weight does not matter.  Stops when ‖r‖₂ <= tol·‖b‖₂ or after maxit. */
static void coarse_cg(const olevel *L, double tol, int maxit, const double *b, double *x) {
    const int64_t N = L->N;
    double *r = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    double *z = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    double *p = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    double *q = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    double *dg = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    for (int64_t i = 0; i < N; i++) {
        int found = 0;
        dg[i] = csr_get(&L->K, i, (int32_t)i, &found);
        x[i] = 0.0;
        r[i] = b[i];
    }
    double bn = 0.0, rz = 0.0;
    for (int64_t i = 0; i < N; i++) bn = bn + b[i] * b[i];
    bn = sqrt(bn);
    if (bn > 0.0) {
        for (int64_t i = 0; i < N; i++) {
            z[i] = r[i] / dg[i];
            p[i] = z[i];
            rz = rz + r[i] * z[i];
        }
        for (int k = 0; k < maxit; k++) {
            or_spmv(&L->K, p, q);
            double pq = 0.0;
            for (int64_t i = 0; i < N; i++) pq = pq + p[i] * q[i];
            if (!(pq > 0.0)) break;
            const double alpha = rz / pq;
            double rn = 0.0;
            for (int64_t i = 0; i < N; i++) {
                x[i] = x[i] + alpha * p[i];
                r[i] = r[i] - alpha * q[i];
                rn = rn + r[i] * r[i];
            }
            if (sqrt(rn) <= tol * bn) break;
            double rz_new = 0.0;
            for (int64_t i = 0; i < N; i++) {
                z[i] = r[i] / dg[i];
                rz_new = rz_new + r[i] * z[i];
            }
            const double beta = rz_new / rz;
            for (int64_t i = 0; i < N; i++) p[i] = z[i] + beta * p[i];
            rz = rz_new;
        }
    }
    free(r); free(z); free(p); free(q); free(dg);
}

/* c.18: V(l, b): l = L: coarse solve.  Else x = S(b, 0); r = b − K x; e = V(l+1, R r);
 * x += P̄ e; x = S(b, x). */
static void vcycle_level(const ohier *H, int l, const double *b, double *x) {
    const olevel *L = &H->lev[l];
    const int64_t N = L->N;
    double *t = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    if (l == H->nlevels - 1) {
        if (H->prm.coarse_solver == 1) coarse_cg(L, H->prm.coarse_tol, H->prm.coarse_maxit, b, x);
        else coarse_solve(L, H->prm.coarse_sweeps, b, x, t);
        free(t);
        return;
    }
    const int64_t Nc = H->lev[l + 1].N;
    double *r = (double *)malloc((size_t)N * sizeof(double));
    double *d = (double *)malloc((size_t)N * sizeof(double));
    double *bc = (double *)malloc((size_t)Nc * sizeof(double));
    double *xc = (double *)malloc((size_t)Nc * sizeof(double));
    for (int64_t i = 0; i < N; i++) x[i] = 0.0;
    smooth(L, H->prm.cheb_degree, b, x, 1, r, d, t);
    or_spmv(&L->K, x, t);
    for (int64_t i = 0; i < N; i++) r[i] = b[i] - t[i];
    or_spmv(&L->R, r, bc);
    vcycle_level(H, l + 1, bc, xc);
    or_spmv(&L->P, xc, t);
    for (int64_t i = 0; i < N; i++) x[i] = x[i] + t[i];
    smooth(L, H->prm.cheb_degree, b, x, 0, r, d, t);
    free(r); free(d); free(bc); free(xc); free(t);
}

void or_vcycle(const ohier *H, const double *b, double *x) { vcycle_level(H, 0, b, x); }

static double dot(int64_t n, const double *a, const double *b) {
    double s = 0.0;
    for (int64_t i = 0; i < n; i++) s = s + a[i] * b[i];
    return s;
}

/* c.19: PCG.  u: initial guess in, solution out.  Stops when
 * ‖r_k‖₂ <= rtol·‖F‖₂ (recurrence residual) or k == maxit.  hist (nullable, maxit+1): ‖r_k‖/‖F‖.
 * Returns 0 (converged), 1 (maxit reached), -5 (breakdown: pᵀKp <= 0 or rᵀz <= 0). */
int or_pcg(const ohier *H, const double *F, double *u, double rtol, int maxit, int *iters,
           double *relres, double *hist) {
    const olevel *L = &H->lev[0];
    const int64_t N = L->N;
    double *r = (double *)malloc((size_t)N * sizeof(double));
    double *z = (double *)malloc((size_t)N * sizeof(double));
    double *p = (double *)malloc((size_t)N * sizeof(double));
    double *q = (double *)malloc((size_t)N * sizeof(double));
    int rc = 0;
    double nF = sqrt(dot(N, F, F));
    *iters = 0;
    if (nF == 0.0) {
        for (int64_t i = 0; i < N; i++) u[i] = 0.0;
        *relres = 0.0;
        if (hist) hist[0] = 0.0;
        goto done;
    }
    or_spmv(&L->K, u, q);
    for (int64_t i = 0; i < N; i++) r[i] = F[i] - q[i];
    double rn = sqrt(dot(N, r, r));
    if (hist) hist[0] = rn / nF;
    *relres = rn / nF;
    if (rn <= rtol * nF) goto done;
    or_vcycle(H, r, z);
    double rho = dot(N, r, z);
    if (!(rho > 0.0)) { rc = -5; goto done; }
    for (int64_t i = 0; i < N; i++) p[i] = z[i];
    rc = 1;
    for (int k = 1; k <= maxit; k++) {
        or_spmv(&L->K, p, q);
        double pq = dot(N, p, q);
        if (!(pq > 0.0)) { rc = -5; break; }
        double alpha = rho / pq;
        for (int64_t i = 0; i < N; i++) {
            u[i] = u[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
        rn = sqrt(dot(N, r, r));
        *iters = k;
        *relres = rn / nF;
        if (hist) hist[k] = rn / nF;
        if (rn <= rtol * nF) { rc = 0; break; }
        or_vcycle(H, r, z);
        double rho_new = dot(N, r, z);
        if (!(rho_new > 0.0)) { rc = -5; break; }
        double beta = rho_new / rho;
        for (int64_t i = 0; i < N; i++) p[i] = z[i] + beta * p[i];
        rho = rho_new;
    }
done:
    free(r); free(z); free(p); free(q);
    return rc;
}

/* Flexible CG (the paper's outer solver: "the flexible variant of the CG algorithm"), in
 * Notay's FCG(1) form (truncation 1): α_k = (p_kᵀ r_k)/(p_kᵀ q_k), p_{k+1} = z_{k+1} − ((z_{k+1}ᵀ q_k)/
 * (p_kᵀ q_k)) p_k.  With a fixed SPD preconditioner it generates the CG iterates; it stays a descent
 * method when the preconditioner varies (the §5.1 coarse CG makes the V-cycle nonlinear).  Same
 * stopping test, history and return codes as or_pcg; breakdown if pᵀKp <= 0. */
typedef int (*or_iter_cb)(int k, void *ctx);
int or_fcg_cb(const ohier *H, const double *F, double *u, double rtol, int maxit, int *iters,
              double *relres, double *hist, or_iter_cb cb, void *ctx);
int or_fcg(const ohier *H, const double *F, double *u, double rtol, int maxit, int *iters,
           double *relres, double *hist) {
    return or_fcg_cb(H, F, u, rtol, maxit, iters, relres, hist, 0, 0);
}
/* or_fcg with an observer: cb(k, ctx) is called after iteration k's stopping test (not after the
 * final, converged one); a non-zero return stops the solve there (return code 1, as at maxit).  The
 * observer only reads the clock (bench.py's oracle arm times the iterations one by one); the
 * arithmetic is or_fcg's. */
int or_fcg_cb(const ohier *H, const double *F, double *u, double rtol, int maxit, int *iters,
              double *relres, double *hist, or_iter_cb cb, void *ctx) {
    const olevel *L = &H->lev[0];
    const int64_t N = L->N;
    double *r = (double *)malloc((size_t)N * sizeof(double));
    double *z = (double *)malloc((size_t)N * sizeof(double));
    double *p = (double *)malloc((size_t)N * sizeof(double));
    double *q = (double *)malloc((size_t)N * sizeof(double));
    int rc = 0;
    double nF = sqrt(dot(N, F, F));
    *iters = 0;
    if (nF == 0.0) {
        for (int64_t i = 0; i < N; i++) u[i] = 0.0;
        *relres = 0.0;
        if (hist) hist[0] = 0.0;
        goto done;
    }
    or_spmv(&L->K, u, q);
    for (int64_t i = 0; i < N; i++) r[i] = F[i] - q[i];
    double rn = sqrt(dot(N, r, r));
    if (hist) hist[0] = rn / nF;
    *relres = rn / nF;
    if (rn <= rtol * nF) goto done;
    or_vcycle(H, r, z);
    for (int64_t i = 0; i < N; i++) p[i] = z[i];
    rc = 1;
    for (int k = 1; k <= maxit; k++) {
        or_spmv(&L->K, p, q);
        const double pq = dot(N, p, q);
        if (!(pq > 0.0)) { rc = -5; break; }
        const double alpha = dot(N, p, r) / pq;
        for (int64_t i = 0; i < N; i++) {
            u[i] = u[i] + alpha * p[i];
            r[i] = r[i] - alpha * q[i];
        }
        rn = sqrt(dot(N, r, r));
        *iters = k;
        *relres = rn / nF;
        if (hist) hist[k] = rn / nF;
        if (rn <= rtol * nF) { rc = 0; break; }
        if (cb && cb(k, ctx)) break;
        or_vcycle(H, r, z);
        const double beta = -dot(N, z, q) / pq;
        for (int64_t i = 0; i < N; i++) p[i] = z[i] + beta * p[i];
    }
done:
    free(r); free(z); free(p); free(q);
    return rc;
}

/* ------------------------------------------------------------------------------------------ */
/* Accessors for the Python side                                                              */
/* ------------------------------------------------------------------------------------------ */

ocsr *or_csr_new(void) { return (ocsr *)calloc(1, sizeof(ocsr)); }
void or_csr_delete(ocsr *A) { if (A) { csr_free(A); free(A); } }
int or_hier_nlevels(const ohier *H) { return H->nlevels; }
/* c.10 on its own (for its pin, tests/test_oracle_setup.py): the intermediate Galerkin operator of
 * one pairwise step, written into *Ac (free with or_csr_delete). */
int or_galerkin_pairwise(const ocsr *A, const int32_t *agg, const double *pv, int64_t nc, ocsr *Ac) {
    return galerkin_pairwise(A, agg, pv, nc, Ac);
}
const olevel *or_hier_level(const ohier *H, int l) { return &H->lev[l]; }

/* Smoother alone (tests): x <- S(b, x) on level l (c.16). */
void or_smooth(const ohier *H, int l, const double *b, double *x, int x_is_zero) {
    const olevel *L = &H->lev[l];
    const int64_t N = L->N;
    double *r = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    double *d = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    double *t = (double *)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
    if (x_is_zero)
        for (int64_t i = 0; i < N; i++) x[i] = 0.0;
    smooth(L, H->prm.cheb_degree, b, x, x_is_zero, r, d, t);
    free(r); free(d); free(t);
}
