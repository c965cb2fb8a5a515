// common.hpp — internal host-side types of the B200 AMG library (not part of the C ABI).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <functional>
#include <string>
#include <utility>
#include <vector>

#include "amg_b200.h"

namespace amgb {

// Thread-local error message behind amg_last_error().
void set_error(const std::string &msg);
const char *get_error();

struct Error {
    amg_status st;
    std::string msg;
};

// Uninitialised heap array (std::vector would zero-fill multi-GB arrays).
template <class T>
struct Buf {
    T *p = nullptr;
    int64_t n = 0;
    Buf() = default;
    explicit Buf(int64_t count) { alloc(count); }
    void alloc(int64_t count) {
        std::free(p);
        n = count;
        p = static_cast<T *>(std::malloc(static_cast<size_t>(count > 0 ? count : 1) * sizeof(T)));
        if (!p) throw Error{AMG_ENOMEM, "host allocation failed"};
    }
    void shrink(int64_t count) {  // keep the first `count` elements
        T *q = static_cast<T *>(std::realloc(p, static_cast<size_t>(count > 0 ? count : 1) * sizeof(T)));
        if (q) p = q;
        n = count;
    }
    Buf(const Buf &) = delete;
    Buf &operator=(const Buf &) = delete;
    Buf(Buf &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
    Buf &operator=(Buf &&o) noexcept {
        if (this != &o) { std::free(p); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
        return *this;
    }
    ~Buf() { std::free(p); }
    // hand the malloc'd array over (to an amg_csr the caller frees) / take one over (from an amg_csr)
    T *release() {
        T *q = p;
        p = nullptr;
        n = 0;
        return q;
    }
    void adopt(T *q, int64_t count) {
        std::free(p);
        p = q;
        n = count;
    }
    T &operator[](int64_t i) { return p[i]; }
    const T &operator[](int64_t i) const { return p[i]; }
    T *data() { return p; }
    const T *data() const { return p; }
};

// Host CSR (0-based, int64 row pointers, int32 ascending columns, fp64 values).
struct HCsr {
    int64_t nrows = 0, ncols = 0;
    Buf<int64_t> rp;
    Buf<int32_t> ci;
    Buf<double> v;
    int64_t nnz() const { return nrows ? rp[nrows] : 0; }
};

// One level of the host hierarchy (c.6-c.15).
struct HLevel {
    int64_t N = 0;
    HCsr K;              // K_l
    HCsr P;              // P̄_l (N_l x N_{l+1}); empty on the coarsest level
    HCsr R;              // R_l = P̄_lᵀ
    Buf<int32_t> agg;    // composite aggregate map
    Buf<double> ptent;   // composite tentative P value per row
    Buf<double> dhat;    // ℓ1 diagonal
    double omega = 0.0;
    int64_t nnz_K = 0, nnz_P = 0;  // thin hierarchies only (K, P of distributed levels not held)
};

struct HHierarchy {
    amg_params prm{};
    int nlevels = 0;
    bool thin = false;  // built from one rank's share (share.cpp): distributed levels held as LocalOps
    bool released = false;  // thin + device: the host operators were freed once uploaded (amg_setup_from_share)
    HLevel lev[32];
};

inline int64_t level_nnz_K(const HHierarchy &H, int l) { return H.thin ? H.lev[l].nnz_K : H.lev[l].K.nnz(); }
inline int64_t level_nnz_P(const HHierarchy &H, int l) {
    if (l + 1 >= H.nlevels) return 0;
    return H.thin ? H.lev[l].nnz_P : H.lev[l].P.nnz();
}

// ---- multi-GPU plumbing (dist.cpp) ------------------------------------------------------------
// One rank's share of a distributed operator: its rows [row_begin, row_end), columns renumbered in
// GLOBAL order: lower ghosts −nlo..−1, owned columns 0..nown−1 (global col_begin..col_end−1), upper
// ghosts nown.. (so a row's local column span equals its global span up to the gaps, which keeps the
// 16-bit column encoding available), and the halo plan that fills the ghost slots.  Ghosts owned by
// rank q are contiguous (global order = rank order).
struct LocalOp {
    int64_t row_begin = 0, row_end = 0;
    int64_t col_begin = 0, col_end = 0;  // owned column range; full_cols: [0, ncols)
    bool full_cols = false;              // columns index a replicated (whole) vector: no ghosts
    HCsr A;                              // local rows x (owned + ghost) columns
    std::vector<int64_t> ghost;          // global ids of the ghost columns, ascending
    int64_t nlo = 0;                     // ghosts below col_begin (lower ranks): local indices −nlo..−1
    std::vector<int32_t> send_count, send_off, send_idx;  // per destination rank; local owned indices
    std::vector<int32_t> recv_count, recv_off;            // per source rank; offsets into the ghost area
};

struct DistLevel {
    bool replicated = false;       // whole level on every rank (coarse levels)
    std::vector<int64_t> bounds;   // row partition (nranks+1) of the level (also for replicated levels)
    LocalOp K, P, R;               // R: rows = this level's coarse rows partition of level l+1
};

struct DistPlan {
    int rank = 0, nranks = 1;
    int last_dist = 0;             // last distributed level (levels > last_dist are replicated)
    DistLevel lev[32];
};

// Row partition of every level balanced by nnz, the replication cut, and this rank's local
// operators + halo plans.  Deterministic; identical on every rank given the same hierarchy.
void build_dist_plan(const HHierarchy &H, int rank, int nranks, int64_t replicate_nnz, DistPlan &P);

// share.cpp: one rank's share of a global host hierarchy as a malloc'd blob, and back (thin H + plan)
void share_export(const HHierarchy &H, int rank, int nranks, int64_t replicate_nnz, uint8_t **blob, int64_t *bytes);
void share_import(const void *blob, int64_t bytes, int rank, int nranks, HHierarchy &H, DistPlan &plan);

// iga_gen.cpp
void iga_tables_hat(int p, int n, double *mhat, double *khat);
void iga_assemble(const amg_iga_desc &d, HCsr &K, Buf<double> &F);

// setup.cpp
void build_hierarchy(const amg_csr &K, const amg_params &prm, HHierarchy &H);
// The same, taking K's arrays over instead of copying them (amg_setup_take): K's pointers are nulled.
void build_hierarchy_take(amg_csr &K, const amg_params &prm, HHierarchy &H);

// device.cu
struct DevState;
// release (may be null): called once every operator is on the device, before the first collective
// (NCCL init): a share-built hierarchy frees its host operators there, so the ranks that wait in the
// collective for the others do not hold them
DevState *dev_create(const HHierarchy &H, const amg_dist *dist, const DistPlan *plan,
                     const std::function<void()> &release = {});
void dev_destroy(DevState *D);

}  // namespace amgb

struct amg_hierarchy {
    amgb::HHierarchy host;
    amgb::DevState *dev = nullptr;
    amgb::DistPlan plan;  // host view of this rank's share (multi-GPU setups)
    bool distributed = false;
};
