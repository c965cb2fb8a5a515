// setup.cpp — host-side hierarchy setup (deterministic, OpenMP, bitwise reproducible).
//
// Paper: compatible weighted matching (eq:cij P:L766-771, eq:maxprod P:L794-809), pairwise
// prolongation (eq:prolongation P:L811-834, "no such reordering is performed" P:L834), m-step
// aggregation P1P2P3 ("aggregates of size 8" P:L1114), smoothed prolongation
// P̄ = (I − ωD⁻¹K)P, Galerkin K_{l+1} = R K_l P with R = P̄ᵀ
// (eq:galerkin_matrix_projection P:L664-667), ℓ1 diagonal, coarse stop.
//
// The readings c.6-c.15 of DESIGN.md §3 fix every choice the paper leaves open, and the canonical
// arithmetic contract fixes every floating-point evaluation order, so this parallel implementation
// produces the same bits for every thread count:
//   * every reduction that feeds a stored value is sequential, in ascending index order, from +0.0;
//   * products are evaluated as written (c.7, c.10, c.12, c.13), with no FMA (-ffp-contract=off);
//   * the matching is the unique locally-dominant matching under the strict order
//     (c_ij desc, min(i,j) asc, max(i,j) asc), computed here by the parallel pointer algorithm
//     (mutual heaviest pairs, re-pointing only the neighbours of newly matched vertices); it equals
//     the greedy matching of that order (Preis; DESIGN.md §3 c.8).
#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <atomic>
#include <cmath>
#include <vector>

#include "common.hpp"

namespace amgb {
namespace {

// ------------------------------------------------------------------------------------------------
// Parallel row builder: rows are produced independently (each by fn into a sparse accumulator) in
// contiguous chunks, then concatenated.  Row content never depends on the thread count.
// ------------------------------------------------------------------------------------------------
struct Spa {
    std::vector<double> acc;
    std::vector<int64_t> stamp;
    std::vector<int32_t> cols;
    int64_t row = -1;
    void init(int64_t ncols) {
        acc.resize(ncols > 0 ? ncols : 1);
        stamp.assign(ncols > 0 ? ncols : 1, -1);
        cols.clear();
    }
    void start(int64_t r) { row = r; cols.clear(); }
    inline void add(int32_t j, double x) {
        if (stamp[j] != row) {
            stamp[j] = row;
            acc[j] = 0.0;
            cols.push_back(j);
        }
        acc[j] = acc[j] + x;
    }
    void sort() { std::sort(cols.begin(), cols.end()); }
};

struct Chunk {
    std::vector<int64_t> cnt;
    std::vector<int32_t> ci;
    std::vector<double> v;
};

// Two-pass assembly for the largest levels (fine levels of C5-sized problems, or AMG_SETUP_LEAN=1):
// every row is computed twice, once to count and once straight into the exactly-sized output, so the
// peak holds the output once instead of the chunk buffers (with vector growth slack) plus the output.
// The rows are the same computation both times, so the result is bitwise the single-pass one.
inline bool lean_rows(int64_t nrows) {
    static const int forced = [] {
        const char *e = std::getenv("AMG_SETUP_LEAN");
        return e ? std::atoi(e) : -1;
    }();
    return forced >= 0 ? forced != 0 : nrows >= 8000000;
}

// fn(row, spa, out_ci, out_v): append the row's entries (ascending columns) to out_ci/out_v.
template <class Fn>
void build_rows(int64_t nrows, int64_t ncols, HCsr &out, Fn fn) {
    out.nrows = nrows;
    out.ncols = ncols;
    if (lean_rows(nrows)) {
        out.rp.alloc(nrows + 1);
        out.rp[0] = 0;
#pragma omp parallel
        {
            Spa spa;
            spa.init(ncols);
            std::vector<int32_t> ci;
            std::vector<double> v;
#pragma omp for schedule(dynamic, 2048)
            for (int64_t r = 0; r < nrows; r++) {
                ci.clear();
                v.clear();
                fn(r, spa, ci, v);
                out.rp[r + 1] = (int64_t)ci.size();
            }
        }
        for (int64_t r = 0; r < nrows; r++) out.rp[r + 1] += out.rp[r];
        out.ci.alloc(out.rp[nrows]);
        out.v.alloc(out.rp[nrows]);
#pragma omp parallel
        {
            Spa spa;
            spa.init(ncols);
            std::vector<int32_t> ci;
            std::vector<double> v;
#pragma omp for schedule(dynamic, 2048)
            for (int64_t r = 0; r < nrows; r++) {
                ci.clear();
                v.clear();
                fn(r, spa, ci, v);
                std::memcpy(out.ci.data() + out.rp[r], ci.data(), ci.size() * sizeof(int32_t));
                std::memcpy(out.v.data() + out.rp[r], v.data(), v.size() * sizeof(double));
            }
        }
        return;
    }
    const int64_t CH = 2048;
    const int64_t nch = (nrows + CH - 1) / CH;
    std::vector<Chunk> chunks(nch);
#pragma omp parallel
    {
        Spa spa;
        spa.init(ncols);
#pragma omp for schedule(dynamic, 1)
        for (int64_t c = 0; c < nch; c++) {
            Chunk &ch = chunks[c];
            const int64_t r0 = c * CH, r1 = std::min(nrows, r0 + CH);
            ch.cnt.resize(r1 - r0);
            for (int64_t r = r0; r < r1; r++) {
                size_t before = ch.ci.size();
                fn(r, spa, ch.ci, ch.v);
                ch.cnt[r - r0] = (int64_t)(ch.ci.size() - before);
            }
        }
    }
    out.rp.alloc(nrows + 1);
    out.rp[0] = 0;
    std::vector<int64_t> base(nch + 1, 0);
    for (int64_t c = 0; c < nch; c++) base[c + 1] = base[c] + (int64_t)chunks[c].ci.size();
    out.ci.alloc(base[nch]);
    out.v.alloc(base[nch]);
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t c = 0; c < nch; c++) {
        Chunk &ch = chunks[c];
        int64_t off = base[c];
        const int64_t r0 = c * CH;
        for (size_t t = 0; t < ch.cnt.size(); t++) {
            off += ch.cnt[t];
            out.rp[r0 + (int64_t)t + 1] = off;
        }
        if (!ch.ci.empty()) {
            std::memcpy(out.ci.data() + base[c], ch.ci.data(), ch.ci.size() * sizeof(int32_t));
            std::memcpy(out.v.data() + base[c], ch.v.data(), ch.v.size() * sizeof(double));
        }
        Chunk().cnt.swap(ch.cnt);
        std::vector<int32_t>().swap(ch.ci);
        std::vector<double>().swap(ch.v);
    }
}

// Emit the accumulator's row in ascending column order.
inline void flush(Spa &s, std::vector<int32_t> &ci, std::vector<double> &v) {
    s.sort();
    for (int32_t j : s.cols) {
        ci.push_back(j);
        v.push_back(s.acc[j]);
    }
}

// Transpose (row J lists source rows ascending).
void transpose(const HCsr &A, HCsr &T) {
    const int64_t nnz = A.nnz();
    T.nrows = A.ncols;
    T.ncols = A.nrows;
    T.rp.alloc(T.nrows + 1);
    std::memset(T.rp.data(), 0, sizeof(int64_t) * (T.nrows + 1));
    for (int64_t k = 0; k < nnz; k++) T.rp[A.ci[k] + 1]++;
    for (int64_t j = 0; j < T.nrows; j++) T.rp[j + 1] += T.rp[j];
    T.ci.alloc(nnz);
    T.v.alloc(nnz);
    Buf<int64_t> pos(T.nrows + 1);
    std::memcpy(pos.data(), T.rp.data(), sizeof(int64_t) * (T.nrows + 1));
    for (int64_t i = 0; i < A.nrows; i++)
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++) {
            int64_t d = pos[A.ci[k]]++;
            T.ci[d] = (int32_t)i;
            T.v[d] = A.v[k];
        }
}

// A <- 0.5 (A + Aᵀ) on the structural union (c.10, c.13); (a + t) * 0.5 is commutative.
void symmetrize(HCsr &A) {
    HCsr T;
    transpose(A, T);
    HCsr S;
    build_rows(A.nrows, A.ncols, S, [&](int64_t i, Spa &, std::vector<int32_t> &ci, std::vector<double> &v) {
        int64_t ka = A.rp[i], ea = A.rp[i + 1], kt = T.rp[i], et = T.rp[i + 1];
        while (ka < ea || kt < et) {
            int32_t ja = ka < ea ? A.ci[ka] : INT32_MAX;
            int32_t jt = kt < et ? T.ci[kt] : INT32_MAX;
            double a = 0.0, t = 0.0;
            int32_t j;
            if (ja == jt) { j = ja; a = A.v[ka++]; t = T.v[kt++]; }
            else if (ja < jt) { j = ja; a = A.v[ka++]; }
            else { j = jt; t = T.v[kt++]; }
            ci.push_back(j);
            v.push_back((a + t) * 0.5);
        }
    });
    A = std::move(S);
}

void diagonal(const HCsr &A, Buf<double> &d) {
    d.alloc(A.nrows);
    std::atomic<int> bad{0};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < A.nrows; i++) {
        const int32_t *b = A.ci.data() + A.rp[i], *e = A.ci.data() + A.rp[i + 1];
        const int32_t *f = std::lower_bound(b, e, (int32_t)i);
        if (f == e || *f != i || !(A.v[A.rp[i] + (f - b)] > 0.0)) {
            bad = 1;
            d[i] = 0.0;
        } else {
            d[i] = A.v[A.rp[i] + (f - b)];
        }
    }
    if (bad) throw Error{AMG_ENOTSPD, "missing or non-positive diagonal entry"};
}

// ------------------------------------------------------------------------------------------------
// c.7 / c.8 — compatibility weights and the locally-dominant matching
// ------------------------------------------------------------------------------------------------

// eq:cij for the ordered pair lo < hi, evaluated exactly as c.7 writes it.
inline double cij(double k, double kll, double khh, double wl, double wh) {
    const double num = ((2.0 * k) * wl) * wh;
    const double den = (kll * wl) * wl + (khh * wh) * wh;
    return 1.0 - num / den;
}

// Heaviest eligible unmatched neighbour of i under (c desc, lo asc, hi asc); -1 if none.
inline int32_t best_candidate(const HCsr &A, int64_t i, const double *diag, const double *w,
                              const int32_t *mate, double thr) {
    int32_t best = -1;
    double bc = 0.0;
    int64_t blo = 0, bhi = 0;
    for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++) {
        const int32_t j = A.ci[k];
        if (j == i || mate[j] >= 0) continue;
        const int64_t lo = std::min<int64_t>(i, j), hi = std::max<int64_t>(i, j);
        const double c = cij(A.v[k], diag[lo], diag[hi], w[lo], w[hi]);
        if (!(c > thr)) continue;
        if (best < 0 || c > bc || (c == bc && (lo < blo || (lo == blo && hi < bhi)))) {
            best = j;
            bc = c;
            blo = lo;
            bhi = hi;
        }
    }
    return best;
}

template <class T>
void concat(std::vector<std::vector<T>> &parts, std::vector<T> &out) {
    out.clear();
    for (auto &p : parts) {
        out.insert(out.end(), p.begin(), p.end());
        p.clear();
    }
}

// One pairwise step (c.7-c.9).  Returns the number of aggregates.
int64_t pairwise_step(const HCsr &A, const double *w, double thr, Buf<int32_t> &agg, Buf<double> &pv,
                      Buf<double> &wn) {
    const int64_t N = A.nrows;
    Buf<double> diag;
    diagonal(A, diag);
    Buf<int32_t> mate(N), cand(N);
    Buf<uint8_t> flag(N);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) { mate[i] = -1; flag[i] = 0; }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < N; i++) cand[i] = best_candidate(A, i, diag.data(), w, mate.data(), thr);
    std::vector<int32_t> work(N);
    for (int64_t i = 0; i < N; i++) work[i] = (int32_t)i;
    const int T = omp_get_max_threads();
    std::vector<std::vector<int32_t>> part(T);
    std::vector<int32_t> newly, next;
    while (!work.empty()) {
        const bool par = work.size() > 8192;
        // phase 1: match mutual pairs (the smaller endpoint writes; no two threads touch a pair)
#pragma omp parallel if (par)
        {
            auto &mine = part[omp_get_thread_num()];
#pragma omp for schedule(static)
            for (size_t t = 0; t < work.size(); t++) {
                const int32_t i = work[t];
                const int32_t j = cand[i];
                if (j > i && mate[i] < 0 && cand[j] == i) {
                    mate[i] = j;
                    mate[j] = i;
                    mine.push_back(i);
                    mine.push_back(j);
                }
            }
        }
        concat(part, newly);
        if (newly.empty()) break;
        // phase 2: unmatched vertices that pointed at a newly matched vertex are re-pointed
#pragma omp parallel if (newly.size() > 4096)
        {
            auto &mine = part[omp_get_thread_num()];
#pragma omp for schedule(dynamic, 64)
            for (size_t t = 0; t < newly.size(); t++) {
                const int32_t v = newly[t];
                for (int64_t k = A.rp[v]; k < A.rp[v + 1]; k++) {
                    const int32_t u = A.ci[k];
                    if (u == v || mate[u] >= 0 || cand[u] != v) continue;
                    uint8_t expected = 0;
                    if (__atomic_compare_exchange_n(&flag[u], &expected, (uint8_t)1, false, __ATOMIC_RELAXED,
                                                    __ATOMIC_RELAXED))
                        mine.push_back(u);
                }
            }
        }
        concat(part, next);
#pragma omp parallel for schedule(dynamic, 256) if (next.size() > 4096)
        for (size_t t = 0; t < next.size(); t++)
            cand[next[t]] = best_candidate(A, next[t], diag.data(), w, mate.data(), thr);
        // next work list: re-pointed vertices and their new targets (deduplicated by flag)
        work.clear();
        for (int32_t u : next) work.push_back(u);
        for (int32_t u : next) {
            const int32_t c = cand[u];
            if (c >= 0 && !flag[c]) {
                flag[c] = 1;
                work.push_back(c);
            }
        }
        for (int32_t u : work) flag[u] = 0;
    }
    // aggregates numbered in ascending order of their minimum member (c.9)
    agg.alloc(N);
    pv.alloc(N);
    wn.alloc(N);
    int64_t nc = 0;
    for (int64_t i = 0; i < N; i++) {
        const int32_t j = mate[i];
        if (j < 0) {
            agg[i] = (int32_t)nc;
            pv[i] = w[i] / std::fabs(w[i]);
            wn[nc] = std::fabs(w[i]);
            nc++;
        } else if (i < j) {
            const double nrm = std::sqrt(w[i] * w[i] + w[j] * w[j]);
            agg[i] = agg[j] = (int32_t)nc;
            pv[i] = w[i] / nrm;
            pv[j] = w[j] / nrm;
            wn[nc] = nrm;
            nc++;
        }
    }
    wn.shrink(nc);
    return nc;
}

// c.10: A_{s+1}[I,J] = Σ_{i∈I asc} Σ_{j in row i asc} P[i,I]·(A[i,j]·P[j,J]), then symmetrised.
void galerkin_pairwise(const HCsr &A, const Buf<int32_t> &agg, const Buf<double> &pv, int64_t nc, HCsr &Ac) {
    const int64_t N = A.nrows;
    // members: at most two per aggregate, ascending
    Buf<int32_t> m0(nc), m1(nc);
    for (int64_t I = 0; I < nc; I++) m0[I] = m1[I] = -1;
    for (int64_t i = 0; i < N; i++) {
        const int32_t I = agg[i];
        if (m0[I] < 0) m0[I] = (int32_t)i;
        else m1[I] = (int32_t)i;
    }
    build_rows(nc, nc, Ac, [&](int64_t I, Spa &s, std::vector<int32_t> &ci, std::vector<double> &v) {
        s.start(I);
        for (int t = 0; t < 2; t++) {
            const int32_t i = t == 0 ? m0[I] : m1[I];
            if (i < 0) continue;
            for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++) {
                const int32_t j = A.ci[k];
                s.add(agg[j], pv[i] * (A.v[k] * pv[j]));
            }
        }
        flush(s, ci, v);
    });
    symmetrize(Ac);
}

// ------------------------------------------------------------------------------------------------
// c.12 — smoothed prolongator with the θ-filtered smoothing matrix
// ------------------------------------------------------------------------------------------------
void smoothed_prolongator(const HCsr &K, const Buf<int32_t> &agg, const Buf<double> &pt, int64_t nc,
                          double theta, HCsr &P, double &omega) {
    const int64_t N = K.nrows;
    Buf<double> diag;
    diagonal(K, diag);
    // K_f diagonal: k_ii + Σ_{weak j asc} k_ij
    Buf<double> df(N);
    Buf<double> rowq(N);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < N; i++) {
        double s = 0.0;
        for (int64_t k = K.rp[i]; k < K.rp[i + 1]; k++) {
            const int32_t j = K.ci[k];
            if (j == i) continue;
            if (!(std::fabs(K.v[k]) >= theta * std::sqrt(diag[i] * diag[j]))) s = s + K.v[k];
        }
        df[i] = diag[i] + s;
        // Σ_j |K_f[i,j]| in ascending column order
        double a = 0.0;
        for (int64_t k = K.rp[i]; k < K.rp[i + 1]; k++) {
            const int32_t j = K.ci[k];
            if (j == i) a = a + std::fabs(df[i]);
            else if (std::fabs(K.v[k]) >= theta * std::sqrt(diag[i] * diag[j])) a = a + std::fabs(K.v[k]);
        }
        rowq[i] = a / df[i];
    }
    double lam = 0.0;
    for (int64_t i = 0; i < N; i++)
        if (rowq[i] > lam) lam = rowq[i];
    omega = 4.0 / (3.0 * lam);
    const double om = omega;
    build_rows(N, nc, P, [&](int64_t i, Spa &s, std::vector<int32_t> &ci, std::vector<double> &v) {
        s.start(i);
        for (int64_t k = K.rp[i]; k < K.rp[i + 1]; k++) {
            const int32_t j = K.ci[k];
            double kf;
            if (j == i) kf = df[i];
            else if (std::fabs(K.v[k]) >= theta * std::sqrt(diag[i] * diag[j])) kf = K.v[k];
            else continue;
            s.add(agg[j], kf * pt[j]);
        }
        s.sort();
        for (int32_t J : s.cols) {
            const double pij = (J == agg[i]) ? pt[i] : 0.0;
            ci.push_back(J);
            v.push_back(pij - (om * s.acc[J]) / df[i]);
        }
    });
}

// C = A·B (c.13 order: k in row i of A ascending, then row k of B ascending).
void spgemm(const HCsr &A, const HCsr &B, HCsr &C) {
    build_rows(A.nrows, B.ncols, C, [&](int64_t i, Spa &s, std::vector<int32_t> &ci, std::vector<double> &v) {
        s.start(i);
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++) {
            const int32_t j = A.ci[k];
            const double a = A.v[k];
            for (int64_t t = B.rp[j]; t < B.rp[j + 1]; t++) s.add(B.ci[t], a * B.v[t]);
        }
        flush(s, ci, v);
    });
}

void l1_diagonal(const HCsr &K, Buf<double> &d) {
    d.alloc(K.nrows);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < K.nrows; i++) {
        double s = 0.0;
        for (int64_t k = K.rp[i]; k < K.rp[i + 1]; k++) s = s + std::fabs(K.v[k]);
        if (!(s > 0.0)) s = 0.0;
        d[i] = s;
    }
    for (int64_t i = 0; i < K.nrows; i++)
        if (!(d[i] > 0.0)) throw Error{AMG_ENOTSPD, "zero row (ℓ1 diagonal <= 0)"};
}

void copy_in(const amg_csr &K, HCsr &A) {
    const int64_t n = K.n_rows, nnz = K.nnz;
    A.nrows = n;
    A.ncols = K.n_cols;
    A.rp.alloc(n + 1);
    A.ci.alloc(nnz);
    A.v.alloc(nnz);
    std::memcpy(A.rp.data(), K.row_ptr, sizeof(int64_t) * (n + 1));
    std::memcpy(A.ci.data(), K.col, sizeof(int32_t) * nnz);
    std::memcpy(A.v.data(), K.val, sizeof(double) * nnz);
}

void validate(const HCsr &A) {
    if (A.nrows != A.ncols) throw Error{AMG_EINVAL, "K must be square"};
    if (A.rp[0] != 0) throw Error{AMG_EINVAL, "row_ptr[0] must be 0"};
    std::atomic<int> bad{0};
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < A.nrows; i++) {
        if (A.rp[i + 1] < A.rp[i]) { bad = 1; continue; }
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++) {
            if (A.ci[k] < 0 || A.ci[k] >= A.ncols || (k > A.rp[i] && A.ci[k] <= A.ci[k - 1])) bad = 1;
        }
    }
    if (bad) throw Error{AMG_EINVAL, "K: columns must be in range and strictly ascending per row"};
    // exact (bitwise) symmetry: every stored (i, j) has a stored (j, i) with the same bits — found by
    // binary search in row j (ascending columns), so no transposed copy of K is built (K₀ of C5 at 4
    // GPUs is 94 GB); (i, j) ↦ (j, i) is then an involution of the stored entries, i.e. K == Kᵀ bitwise
    std::atomic<int> asym{0};
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t i = 0; i < A.nrows; i++) {
        for (int64_t k = A.rp[i]; k < A.rp[i + 1] && !asym; k++) {
            const int32_t j = A.ci[k];
            const int32_t *b = A.ci.data() + A.rp[j], *e = A.ci.data() + A.rp[j + 1];
            const int32_t *f = std::lower_bound(b, e, (int32_t)i);
            if (f == e || *f != i ||
                std::memcmp(&A.v[k], &A.v[A.rp[j] + (f - b)], sizeof(double)) != 0)
                asym = 1;
        }
    }
    if (asym) throw Error{AMG_EINVAL, "K must be exactly (bitwise) symmetric"};
    Buf<double> d;
    diagonal(A, d);  // throws AMG_ENOTSPD on a missing or non-positive diagonal entry
}

}  // namespace

// Hierarchy (c.6-c.15): level l is the coarsest if N_l <= coarse_size, l+1 == max_levels, or the
// composite aggregation does not reduce N_l.  w^(0) = 1 (c.6); the test vector is carried through the
// pairwise steps (w_{s+1} = ‖w_e‖) and on to the next level.
static void build_levels(const amg_params &prm, HHierarchy &H);

void build_hierarchy(const amg_csr &Kin, const amg_params &prm, HHierarchy &H) {
    if (prm.num_threads > 0) omp_set_num_threads(prm.num_threads);
    copy_in(Kin, H.lev[0].K);
    build_levels(prm, H);
}

void build_hierarchy_take(amg_csr &Kin, const amg_params &prm, HHierarchy &H) {
    if (prm.num_threads > 0) omp_set_num_threads(prm.num_threads);
    HCsr &A = H.lev[0].K;
    A.nrows = Kin.n_rows;
    A.ncols = Kin.n_cols;
    A.rp.adopt(Kin.row_ptr, Kin.n_rows + 1);
    A.ci.adopt(Kin.col, Kin.nnz);
    A.v.adopt(Kin.val, Kin.nnz);
    Kin.row_ptr = nullptr;
    Kin.col = nullptr;
    Kin.val = nullptr;
    build_levels(prm, H);
}

// AMG_SETUP_TRACE=1: resident host memory (GB) and seconds at every phase boundary of the setup, to
// stderr (the largest runs are bounded by the host RAM of the box)
static void trace(const char *what, int l) {
    static const bool on = [] {
        const char *e = std::getenv("AMG_SETUP_TRACE");
        return e && std::atoi(e) != 0;
    }();
    if (!on) return;
    long rss = 0;
    if (FILE *f = std::fopen("/proc/self/statm", "r")) {
        long sz = 0;
        if (std::fscanf(f, "%ld %ld", &sz, &rss) != 2) rss = 0;
        std::fclose(f);
    }
    static const auto t0 = std::chrono::steady_clock::now();
    const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::fprintf(stderr, "[setup] %-18s level %d  rss %.2f GB  t %.1f s\n", what, l, rss * 4096.0 / 1e9, sec);
}

static void build_levels(const amg_params &prm, HHierarchy &H) {
    trace("start", 0);
    H.prm = prm;
    H.nlevels = 0;
    HLevel &L0 = H.lev[0];
    validate(L0.K);
    trace("validated", 0);
    L0.N = L0.K.nrows;
    Buf<double> w(L0.N);
    for (int64_t i = 0; i < L0.N; i++) w[i] = 1.0;
    const int maxl = std::min(prm.max_levels, 32);
    int l = 0;
    for (;;) {
        HLevel &L = H.lev[l];
        const int64_t N = L.N;
        l1_diagonal(L.K, L.dhat);
        H.nlevels = l + 1;
        if (N <= prm.coarse_size || l + 1 >= maxl) break;
        Buf<int32_t> agg(N);
        Buf<double> pt(N);
        for (int64_t i = 0; i < N; i++) { agg[i] = (int32_t)i; pt[i] = 1.0; }
        HCsr A;  // intermediate operator; starts as K_l (borrowed view by copy of pointers avoided)
        const HCsr *Acur = &L.K;
        int64_t nc = N;
        Buf<double> wc(N);
        std::memcpy(wc.data(), w.data(), sizeof(double) * N);
        for (int s = 0; s < prm.agg_steps; s++) {
            Buf<int32_t> aggs;
            Buf<double> pvs, wn;
            const int64_t ncs = pairwise_step(*Acur, wc.data(), prm.match_threshold, aggs, pvs, wn);
            // compose (c.11): P[i, a_s(agg(i))] = P[i, agg(i)] · p_s[agg(i)]
#pragma omp parallel for schedule(static)
            for (int64_t i = 0; i < N; i++) {
                const int32_t a = agg[i];
                pt[i] = pt[i] * pvs[a];
                agg[i] = aggs[a];
            }
            trace("pairwise", l);
            if (s + 1 < prm.agg_steps) {
                HCsr Ac;
                galerkin_pairwise(*Acur, aggs, pvs, ncs, Ac);
                A = std::move(Ac);
                Acur = &A;
                trace("galerkin_pairwise", l);
            }
            wc = std::move(wn);
            nc = ncs;
        }
        if (nc == N) break;
        if (prm.smooth_prolong) {
            smoothed_prolongator(L.K, agg, pt, nc, prm.filter_theta, L.P, L.omega);
        } else {
            L.P.nrows = N;
            L.P.ncols = nc;
            L.P.rp.alloc(N + 1);
            L.P.ci.alloc(N);
            L.P.v.alloc(N);
            for (int64_t i = 0; i <= N; i++) L.P.rp[i] = i;
            for (int64_t i = 0; i < N; i++) { L.P.ci[i] = agg[i]; L.P.v[i] = pt[i]; }
            L.omega = 0.0;
        }
        trace("prolongator", l);
        L.agg = std::move(agg);
        L.ptent = std::move(pt);
        transpose(L.P, L.R);
        HCsr AP, Kc;
        spgemm(L.K, L.P, AP);
        trace("AP", l);
        spgemm(L.R, AP, Kc);
        trace("RAP", l);
        { HCsr tmp = std::move(AP); }
        symmetrize(Kc);
        trace("symmetrized", l);
        HLevel &C = H.lev[l + 1];
        C.K = std::move(Kc);
        C.N = nc;
        w = std::move(wc);
        l++;
    }
}

}  // namespace amgb
