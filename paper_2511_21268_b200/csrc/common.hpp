// common.hpp — internal host-side types of the B200 AMG library (not part of the C ABI).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <utility>

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
};

struct HHierarchy {
    amg_params prm{};
    int nlevels = 0;
    HLevel lev[32];
};

// iga_gen.cpp
void iga_tables_hat(int p, int n, double *mhat, double *khat);
void iga_assemble(const amg_iga_desc &d, HCsr &K, Buf<double> &F);

// setup.cpp
void build_hierarchy(const amg_csr &K, const amg_params &prm, HHierarchy &H);

// device.cu
struct DevState;
DevState *dev_create(const HHierarchy &H, const amg_dist *dist);
void dev_destroy(DevState *D);

}  // namespace amgb

struct amg_hierarchy {
    amgb::HHierarchy host;
    amgb::DevState *dev = nullptr;
};
