// dist.cpp — multi-GPU plumbing on the host: row-block partition of every level, the replication cut,
// and each rank's local operators with their halo plans.
//
// * Every level is split into contiguous row blocks balanced by nnz(K_l).  The fine ordering is
//   lexicographic with z slowest, so level-0 blocks are z-slabs; coarse levels are numbered by minimum
//   member (c.9), so their blocks stay aligned with the fine slabs and halos stay neighbour-to-neighbour.
// * Levels with nnz(K_l) <= replicate_nnz (and every level below the first such one, and always the
//   coarsest) are REPLICATED: held whole on every rank and computed redundantly, bitwise identically.
// * A local operator keeps the global row's entry order and only renumbers columns, so every row sum
//   is bitwise the single-GPU one; only the dot products (per-rank partials + all-reduce) differ in
//   rounding order from the 1-GPU run.
#include <algorithm>

#include "common.hpp"

namespace amgb {
namespace {

std::vector<int64_t> balanced_bounds(const HCsr &A, int nranks) {
    std::vector<int64_t> b(nranks + 1, A.nrows);
    b[0] = 0;
    const int64_t tot = A.nnz();
    int k = 1;
    for (int64_t i = 0; i < A.nrows && k < nranks; i++) {
        // first row whose prefix nnz reaches k/nranks of the total starts block k
        while (k < nranks && A.rp[i] * (int64_t)nranks >= tot * (int64_t)k) b[k++] = i;
    }
    for (; k < nranks; k++) b[k] = A.nrows;
    return b;
}

// Local share of A for rank k: rows [rb[k], rb[k+1]); columns partitioned by cb (nullptr: full).
void make_local(const HCsr &A, const std::vector<int64_t> &rb, const std::vector<int64_t> *cb, int k, int nr,
                LocalOp &L) {
    const int64_t r0 = rb[k], r1 = rb[k + 1];
    L.row_begin = r0;
    L.row_end = r1;
    L.full_cols = (cb == nullptr);
    L.A.nrows = r1 - r0;
    L.A.rp.alloc(r1 - r0 + 1);
    const int64_t base = A.rp[r0], nnz = A.rp[r1] - base;
    for (int64_t i = r0; i <= r1; i++) L.A.rp[i - r0] = A.rp[i] - base;
    L.A.ci.alloc(nnz);
    L.A.v.alloc(nnz);
    std::memcpy(L.A.v.data(), A.v.data() + base, sizeof(double) * nnz);
    L.send_count.assign(nr, 0);
    L.send_off.assign(nr + 1, 0);
    L.recv_count.assign(nr, 0);
    L.recv_off.assign(nr + 1, 0);
    L.ghost.clear();
    L.send_idx.clear();
    if (L.full_cols) {
        L.col_begin = 0;
        L.col_end = A.ncols;
        L.A.ncols = A.ncols;
        std::memcpy(L.A.ci.data(), A.ci.data() + base, sizeof(int32_t) * nnz);
        return;
    }
    const int64_t c0 = (*cb)[k], c1 = (*cb)[k + 1], nown = c1 - c0;
    L.col_begin = c0;
    L.col_end = c1;
    // ghosts: columns of my rows outside my owned range, ascending
    {
        std::vector<int64_t> g;
        for (int64_t t = base; t < A.rp[r1]; t++) {
            const int64_t c = A.ci[t];
            if (c < c0 || c >= c1) g.push_back(c);
        }
        std::sort(g.begin(), g.end());
        g.erase(std::unique(g.begin(), g.end()), g.end());
        L.ghost.swap(g);
    }
    L.A.ncols = nown + (int64_t)L.ghost.size();
    L.nlo = std::lower_bound(L.ghost.begin(), L.ghost.end(), c0) - L.ghost.begin();
    for (int64_t t = 0; t < nnz; t++) {
        const int64_t c = A.ci[base + t];
        int64_t lc;
        if (c >= c0 && c < c1) {
            lc = c - c0;
        } else {
            const int64_t g = std::lower_bound(L.ghost.begin(), L.ghost.end(), c) - L.ghost.begin();
            lc = g < L.nlo ? g - L.nlo : nown + (g - L.nlo);
        }
        L.A.ci[t] = (int32_t)lc;
    }
    // receive segments: ghosts owned by rank q are contiguous
    for (int q = 0; q < nr; q++) {
        const auto lo = std::lower_bound(L.ghost.begin(), L.ghost.end(), (*cb)[q]);
        const auto hi = std::lower_bound(L.ghost.begin(), L.ghost.end(), (*cb)[q + 1]);
        L.recv_count[q] = (int32_t)(hi - lo);
        L.recv_off[q] = (int32_t)(lo - L.ghost.begin());
    }
    L.recv_off[nr] = (int32_t)L.ghost.size();
    // send lists: the columns I own that rank q's rows reference, ascending (= q's ghost order)
    std::vector<uint8_t> mark(nown > 0 ? nown : 1, 0);
    for (int q = 0; q < nr; q++) {
        L.send_off[q] = (int32_t)L.send_idx.size();
        if (q == k) continue;
        std::vector<int32_t> mine;
        for (int64_t t = A.rp[rb[q]]; t < A.rp[rb[q + 1]]; t++) {
            const int64_t c = A.ci[t];
            if (c >= c0 && c < c1 && !mark[c - c0]) {
                mark[c - c0] = 1;
                mine.push_back((int32_t)(c - c0));
            }
        }
        std::sort(mine.begin(), mine.end());
        for (int32_t j : mine) mark[j] = 0;
        L.send_count[q] = (int32_t)mine.size();
        L.send_idx.insert(L.send_idx.end(), mine.begin(), mine.end());
    }
    L.send_off[nr] = (int32_t)L.send_idx.size();
}

}  // namespace

void build_dist_plan(const HHierarchy &H, int rank, int nranks, int64_t replicate_nnz, DistPlan &P) {
    P.rank = rank;
    P.nranks = nranks;
    const int L = H.nlevels;
    for (int l = 0; l < L; l++) P.lev[l].bounds = balanced_bounds(H.lev[l].K, nranks);
    // replication cut: level 0 always distributed; the coarsest always replicated when nranks > 1
    int ld = L - 1;
    if (nranks > 1) {
        ld = 0;
        while (ld + 1 < L - 1 && H.lev[ld + 1].K.nnz() > replicate_nnz) ld++;
        if (L == 1) throw Error{AMG_EINVAL, "a single-level hierarchy cannot be distributed"};
    }
    P.last_dist = ld;
    for (int l = 0; l < L; l++) {
        DistLevel &D = P.lev[l];
        D.replicated = l > ld;
        if (D.replicated) continue;
        make_local(H.lev[l].K, D.bounds, &D.bounds, rank, nranks, D.K);
        if (l + 1 < L) {
            const std::vector<int64_t> &cb = P.lev[l + 1].bounds;
            make_local(H.lev[l].P, D.bounds, (l + 1 <= ld) ? &cb : nullptr, rank, nranks, D.P);
            make_local(H.lev[l].R, cb, &D.bounds, rank, nranks, D.R);
        }
    }
}

}  // namespace amgb
