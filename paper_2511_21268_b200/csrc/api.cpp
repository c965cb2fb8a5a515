// api.cpp — host-side C-ABI entry points (generator, parameters, setup, export, errors).
#include <omp.h>

#include <cstdio>
#include <string>

#include "common.hpp"

namespace amgb {
static thread_local std::string g_err;
void set_error(const std::string &msg) { g_err = msg; }
const char *get_error() { return g_err.c_str(); }
}  // namespace amgb

using namespace amgb;

#define API_BEGIN \
    try {         \
        set_error("");
#define API_END                                                  \
    }                                                            \
    catch (const Error &e) {                                     \
        set_error(e.msg);                                        \
        return e.st;                                             \
    }                                                            \
    catch (const std::bad_alloc &) {                             \
        set_error("out of host memory");                         \
        return AMG_ENOMEM;                                       \
    }                                                            \
    catch (...) {                                                \
        set_error("unknown internal error");                     \
        return AMG_EINVAL;                                       \
    }

namespace {
int64_t replicate_nnz() {  // replicate levels below ~7e6 non-zeros
    int64_t rep = 7000000;
    if (const char *e = std::getenv("AMG_REPLICATE_NNZ")) rep = std::atoll(e);
    return rep;
}

void check_params(const amg_params &prm) {
    if (prm.agg_steps < 1 || prm.cheb_degree < 1 || prm.coarse_sweeps < 0 || prm.max_levels < 1 ||
        prm.coarse_size < 1 || !(prm.filter_theta >= 0.0) || prm.krylov < 0 || prm.krylov > 1 ||
        prm.coarse_solver < 0 || prm.coarse_solver > 1 || !(prm.coarse_tol >= 0.0) || prm.coarse_maxit < 0 ||
        prm.format < 0 || prm.format > 6)
        throw Error{AMG_EINVAL, "bad parameter"};
}

amg_csr *export_csr(const HCsr &A) {
    amg_csr *c = static_cast<amg_csr *>(std::calloc(1, sizeof(amg_csr)));
    if (!c) throw Error{AMG_ENOMEM, "host allocation failed"};
    const int64_t nnz = A.nnz();
    c->n_rows = A.nrows;
    c->n_cols = A.ncols;
    c->nnz = nnz;
    c->row_ptr = static_cast<int64_t *>(std::malloc(sizeof(int64_t) * (A.nrows + 1)));
    c->col = static_cast<int32_t *>(std::malloc(sizeof(int32_t) * (nnz > 0 ? nnz : 1)));
    c->val = static_cast<double *>(std::malloc(sizeof(double) * (nnz > 0 ? nnz : 1)));
    if (!c->row_ptr || !c->col || !c->val) {
        amg_csr_free(c);
        throw Error{AMG_ENOMEM, "host allocation failed"};
    }
    std::memcpy(c->row_ptr, A.rp.data(), sizeof(int64_t) * (A.nrows + 1));
    std::memcpy(c->col, A.ci.data(), sizeof(int32_t) * nnz);
    std::memcpy(c->val, A.v.data(), sizeof(double) * nnz);
    return c;
}
}  // namespace

namespace {
// amg_setup_from_share(_take): import the blob (freed right after when `take`), then the device setup,
// which frees this rank's host operators once they are on the device and before its first collective
amg_hierarchy *from_share(const void *share, int64_t bytes, const amg_dist *dist, int host_only, void *take) {
    struct Free {
        void *p;
        ~Free() { std::free(p); }
    } own{take};
    if (!share) throw Error{AMG_EINVAL, "NULL argument"};
    if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
        throw Error{AMG_EINVAL, "bad amg_dist (rank/nranks)"};
    const int rank = dist ? dist->rank : 0, nranks = dist ? dist->nranks : 1;
    amg_hierarchy *H = new amg_hierarchy();
    try {
        share_import(share, bytes, rank, nranks, H->host, H->plan);
        if (take) {  // the imported copy is all that is needed from here on
            std::free(own.p);
            own.p = nullptr;
        }
        H->host.prm.host_only = host_only ? 1 : 0;
        H->distributed = nranks > 1;
        if (!host_only) {
            // the device holds everything the solve needs: free this rank's host operators (the ranks of
            // one job share one host, whose RAM is what bounds the largest runs) before the first
            // collective of the device setup, where a rank waits for the others; the sizes, nnz counts
            // and row bounds stay for amg_hierarchy_info / amg_local_rows
            auto release = [H] {
                auto drop = [](HCsr &A) {
                    A.ci = Buf<int32_t>();
                    A.v = Buf<double>();
                };
                for (int l = 0; l < H->host.nlevels; l++) {
                    HLevel &L = H->host.lev[l];
                    drop(L.K);
                    drop(L.P);
                    drop(L.R);
                    drop(H->plan.lev[l].K.A);
                    drop(H->plan.lev[l].P.A);
                    drop(H->plan.lev[l].R.A);
                }
                H->host.released = true;
            };
            H->dev = dev_create(H->host, dist, H->distributed ? &H->plan : nullptr, release);
        }
    } catch (...) {
        delete H;
        throw;
    }
    return H;
}
}  // namespace

extern "C" {

const char *amg_last_error(void) { return get_error(); }

void amg_free(void *p) { std::free(p); }

void amg_csr_free(amg_csr *K) {
    if (!K) return;
    std::free(K->row_ptr);
    std::free(K->col);
    std::free(K->val);
    std::free(K);
}

amg_status amg_set_num_threads(int n) {
    API_BEGIN
    if (n < 1) throw Error{AMG_EINVAL, "thread count must be >= 1"};
    omp_set_num_threads(n);
    return AMG_OK;
    API_END
}

amg_status amg_iga_tables(int degree, int n_elem, double *mhat, double *khat) {
    API_BEGIN
    if (degree < 1 || degree > 8 || n_elem < 1 || !mhat || !khat) throw Error{AMG_EINVAL, "bad argument"};
    iga_tables_hat(degree, n_elem, mhat, khat);
    return AMG_OK;
    API_END
}

amg_status amg_iga_poisson(const amg_iga_desc *d, amg_csr **K, double **F) {
    API_BEGIN
    if (!d || !K || !F) throw Error{AMG_EINVAL, "NULL argument"};
    if (d->dim != 2 && d->dim != 3) throw Error{AMG_EINVAL, "dim must be 2 or 3"};
    if (d->degree < 1 || d->degree > 8) throw Error{AMG_EINVAL, "degree must be in [1, 8]"};
    if (d->n_elem < 1) throw Error{AMG_EINVAL, "n_elem must be >= 1"};
    if (d->dirichlet_sides >> (2 * d->dim)) throw Error{AMG_EINVAL, "dirichlet_sides names a side > 2*dim"};
    if (d->rhs < 0 || d->rhs > 2) throw Error{AMG_EINVAL, "rhs must be 0, 1 or 2"};
    if (d->geometry < 0 || d->geometry > 2)
        throw Error{AMG_EINVAL, "geometry must be 0 (cube), 1 (quarter ring) or 2 (three-patch L-shape)"};
    if (d->geometry == 2 && (d->dim != 3 || d->dirichlet_sides != 0b000111u))
        throw Error{AMG_EINVAL, "the L-shape is 3-D with its fixed boundary layout (dirichlet_sides = 0x7)"};
    if (d->geometry == 1 && (d->dim != 3 || d->rhs == 0 || d->dirichlet_sides != 0b000111u))
        throw Error{AMG_EINVAL, "the quarter ring is 3-D with Dirichlet sides 1,2,3 and rhs = 1 (F = 0) or 2 (its paper data)"};
    HCsr A;
    Buf<double> f;
    iga_assemble(*d, A, f);
    // hand the assembled arrays over (no second copy of K: C5's K₀ alone is 94 GB at 4 GPUs)
    amg_csr *c = static_cast<amg_csr *>(std::calloc(1, sizeof(amg_csr)));
    if (!c) throw Error{AMG_ENOMEM, "host allocation failed"};
    c->n_rows = A.nrows;
    c->n_cols = A.ncols;
    c->nnz = A.nnz();
    c->row_ptr = A.rp.release();
    c->col = A.ci.release();
    c->val = A.v.release();
    double *fo = static_cast<double *>(std::malloc(sizeof(double) * (A.nrows > 0 ? A.nrows : 1)));
    if (!fo) {
        amg_csr_free(c);
        throw Error{AMG_ENOMEM, "host allocation failed"};
    }
    std::memcpy(fo, f.data(), sizeof(double) * A.nrows);
    *K = c;
    *F = fo;
    return AMG_OK;
    API_END
}

amg_status amg_params_default(amg_params *prm, int p) {
    API_BEGIN
    if (!prm || p < 1 || p > 8) throw Error{AMG_EINVAL, "bad argument"};
    static const int cheb[9] = {0, 2, 4, 8, 12, 14, 16, 16, 16};  // P:L1117 (p>=3); p=2 -> 4 (c.16)
    prm->agg_steps = 3;
    prm->smooth_prolong = 1;
    prm->match_threshold = 1.0;
    prm->filter_theta = 0.01;
    prm->cheb_degree = cheb[p];
    prm->coarse_sweeps = 30;
    prm->coarse_size = 50;
    prm->max_levels = 20;
    prm->format = 0;
    prm->host_only = 0;
    prm->num_threads = 0;
    prm->krylov = 0;
    prm->coarse_solver = 0;
    prm->coarse_tol = 1e-4;
    prm->coarse_maxit = 30;
    return AMG_OK;
    API_END
}

amg_status amg_setup(const amg_csr *K, const amg_params *prm_in, const amg_dist *dist, amg_hierarchy **Hout) {
    API_BEGIN
    if (!K || !Hout || !K->row_ptr || (K->nnz && (!K->col || !K->val))) throw Error{AMG_EINVAL, "NULL argument"};
    if (K->n_rows < 1 || K->n_rows > INT32_MAX) throw Error{AMG_EINVAL, "n_rows out of range"};
    amg_params prm;
    if (prm_in) prm = *prm_in;
    else amg_params_default(&prm, 2);
    check_params(prm);
    if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
        throw Error{AMG_EINVAL, "bad amg_dist (rank/nranks)"};
    amg_hierarchy *H = new amg_hierarchy();
    try {
        build_hierarchy(*K, prm, H->host);
        if (dist && dist->nranks > 1) {
            build_dist_plan(H->host, dist->rank, dist->nranks, replicate_nnz(), H->plan);
            H->distributed = true;
        }
        if (!prm.host_only) H->dev = dev_create(H->host, dist, H->distributed ? &H->plan : nullptr);
    } catch (...) {
        delete H;
        throw;
    }
    *Hout = H;
    return AMG_OK;
    API_END
}

amg_status amg_setup_take(amg_csr *K, const amg_params *prm_in, const amg_dist *dist, amg_hierarchy **Hout) {
    // as amg_setup, with K's arrays taken over by the hierarchy instead of copied; K is released in
    // every case (its arrays are owned by the hierarchy or freed)
    if (!K) {
        set_error("NULL argument");
        return AMG_EINVAL;
    }
    amg_status st = AMG_OK;
    try {
        if (!Hout || !K->row_ptr || (K->nnz && (!K->col || !K->val))) throw Error{AMG_EINVAL, "NULL argument"};
        if (K->n_rows < 1 || K->n_rows > INT32_MAX) throw Error{AMG_EINVAL, "n_rows out of range"};
        amg_params prm;
        if (prm_in) prm = *prm_in;
        else amg_params_default(&prm, 2);
        check_params(prm);
        if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
            throw Error{AMG_EINVAL, "bad amg_dist (rank/nranks)"};
        amg_hierarchy *H = new amg_hierarchy();
        try {
            build_hierarchy_take(*K, prm, H->host);
            if (dist && dist->nranks > 1) {
                build_dist_plan(H->host, dist->rank, dist->nranks, replicate_nnz(), H->plan);
                H->distributed = true;
            }
            if (!prm.host_only) H->dev = dev_create(H->host, dist, H->distributed ? &H->plan : nullptr);
        } catch (...) {
            delete H;
            throw;
        }
        *Hout = H;
    } catch (const Error &e) {
        set_error(e.msg);
        st = e.st;
    } catch (const std::bad_alloc &) {
        set_error("out of host memory");
        st = AMG_ENOMEM;
    } catch (...) {
        set_error("unknown internal error");
        st = AMG_EINVAL;
    }
    amg_csr_free(K);  // arrays already taken over are NULL here
    return st;
}

amg_status amg_share_export(const amg_hierarchy *H, int rank, int nranks, void **share, int64_t *bytes) {
    API_BEGIN
    if (!H || !share || !bytes) throw Error{AMG_EINVAL, "NULL argument"};
    uint8_t *p = nullptr;
    share_export(H->host, rank, nranks, replicate_nnz(), &p, bytes);
    *share = p;
    return AMG_OK;
    API_END
}


amg_status amg_setup_from_share(const void *share, int64_t bytes, const amg_dist *dist, int host_only,
                                amg_hierarchy **Hout) {
    API_BEGIN
    if (!Hout) throw Error{AMG_EINVAL, "NULL argument"};
    *Hout = from_share(share, bytes, dist, host_only, nullptr);
    return AMG_OK;
    API_END
}

amg_status amg_setup_from_share_take(void *share, int64_t bytes, const amg_dist *dist, int host_only,
                                     amg_hierarchy **Hout) {
    if (!Hout) {
        std::free(share);
        set_error("NULL argument");
        return AMG_EINVAL;
    }
    API_BEGIN
    *Hout = from_share(share, bytes, dist, host_only, share);
    return AMG_OK;
    API_END
}

void *amg_malloc(int64_t bytes) { return std::malloc(bytes > 0 ? (size_t)bytes : 1); }

void amg_hierarchy_free(amg_hierarchy *H) {
    if (!H) return;
    if (H->dev) dev_destroy(H->dev);
    delete H;
}

amg_status amg_hierarchy_info(const amg_hierarchy *H, int64_t *n_levels, int64_t *N, int64_t *nnz, int64_t *nnz_P,
                              double *opc) {
    API_BEGIN
    if (!H) throw Error{AMG_EINVAL, "NULL hierarchy"};
    const HHierarchy &h = H->host;
    if (n_levels) *n_levels = h.nlevels;
    double tot = 0.0;
    for (int l = 0; l < h.nlevels; l++) {
        if (N) N[l] = h.lev[l].N;
        if (nnz) nnz[l] = level_nnz_K(h, l);
        if (nnz_P) nnz_P[l] = level_nnz_P(h, l);
        tot += (double)level_nnz_K(h, l);
    }
    if (opc) *opc = tot / (double)level_nnz_K(h, 0);
    return AMG_OK;
    API_END
}

amg_status amg_hierarchy_export(const amg_hierarchy *H, int level, amg_csr **K_l, amg_csr **P_l,
                                int32_t **aggregate_of, double **dhat, double *omega) {
    API_BEGIN
    if (!H || level < 0 || level >= H->host.nlevels) throw Error{AMG_EINVAL, "bad level"};
    if (H->host.thin) throw Error{AMG_EINVAL, "a hierarchy built from a share holds only this rank's operators"};
    const HLevel &L = H->host.lev[level];
    const bool last = level == H->host.nlevels - 1;
    if (K_l) *K_l = export_csr(L.K);
    if (P_l) *P_l = last ? nullptr : export_csr(L.P);
    if (aggregate_of) {
        if (last) {
            *aggregate_of = nullptr;
        } else {
            *aggregate_of = static_cast<int32_t *>(std::malloc(sizeof(int32_t) * L.N));
            if (!*aggregate_of) throw Error{AMG_ENOMEM, "host allocation failed"};
            std::memcpy(*aggregate_of, L.agg.data(), sizeof(int32_t) * L.N);
        }
    }
    if (dhat) {
        *dhat = static_cast<double *>(std::malloc(sizeof(double) * L.N));
        if (!*dhat) throw Error{AMG_ENOMEM, "host allocation failed"};
        std::memcpy(*dhat, L.dhat.data(), sizeof(double) * L.N);
    }
    if (omega) *omega = L.omega;
    return AMG_OK;
    API_END
}

amg_status amg_dist_view_get(const amg_hierarchy *H, int level, int op, amg_dist_view *v) {
    API_BEGIN
    if (!H || !v || !H->distributed) throw Error{AMG_EINVAL, "hierarchy is not distributed"};
    if (level < 0 || level >= H->host.nlevels || op < 0 || op > 2) throw Error{AMG_EINVAL, "bad level/op"};
    if (op > 0 && level == H->host.nlevels - 1) throw Error{AMG_EINVAL, "no transfer operator on the coarsest level"};
    if (H->host.released) throw Error{AMG_EINVAL, "host operators released after the device upload (use host_only)"};
    const DistLevel &D = H->plan.lev[level];
    std::memset(v, 0, sizeof(*v));
    v->nranks = H->plan.nranks;
    v->replicated = D.replicated ? 1 : 0;
    if (D.replicated) return AMG_OK;
    const LocalOp &L = op == 0 ? D.K : op == 1 ? D.P : D.R;
    v->full_cols = L.full_cols ? 1 : 0;
    v->row_begin = L.row_begin;
    v->row_end = L.row_end;
    v->col_begin = L.col_begin;
    v->col_end = L.col_end;
    v->n_ghost = (int64_t)L.ghost.size();
    v->n_ghost_lo = L.nlo;
    v->ghost = L.ghost.data();
    v->send_count = L.send_count.data();
    v->send_off = L.send_off.data();
    v->send_idx = L.send_idx.data();
    v->recv_count = L.recv_count.data();
    v->recv_off = L.recv_off.data();
    v->local.n_rows = L.A.nrows;
    v->local.n_cols = L.A.ncols;
    v->local.nnz = L.A.nnz();
    v->local.row_ptr = const_cast<int64_t *>(L.A.rp.data());
    v->local.col = const_cast<int32_t *>(L.A.ci.data());
    v->local.val = const_cast<double *>(L.A.v.data());
    return AMG_OK;
    API_END
}

}  // extern "C"
