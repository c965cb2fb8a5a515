// share.cpp — one rank's share of a host hierarchy as a flat byte blob.
//
// With one process per GPU, every rank used to build the same global hierarchy on the host: g copies
// of the fine operator in host RAM and g setups competing for the cores.  Instead, one process builds
// the hierarchy once (amg_setup with host_only), and for each rank serialises exactly what that rank's
// device state needs: its DistPlan (local operators + halo plans of the distributed levels, row bounds
// of every level), the replicated levels whole, every level's size / nnz / ω and ℓ1 diagonal.  The
// rank rebuilds a "thin" hierarchy from the blob and creates its device state from it.  The plan in
// the blob is the one build_dist_plan computes on the global hierarchy, so the device state — and the
// solve — is bitwise the one of the all-ranks-build path.
#include "common.hpp"

namespace amgb {
namespace {

constexpr uint64_t kMagic = 0x31304852534d4741ull;  // "AMGSHR01"

// Two-pass writer: p == nullptr counts bytes, else copies.
struct Out {
    uint8_t *p = nullptr;
    size_t n = 0;
    void put(const void *src, size_t b) {
        if (p && b) std::memcpy(p + n, src, b);
        n += b;
    }
    template <class T>
    void val(const T &x) { put(&x, sizeof(T)); }
    template <class T>
    void arr(const T *a, int64_t cnt) {
        val(cnt);
        put(a, sizeof(T) * (size_t)cnt);
    }
    template <class T>
    void vec(const std::vector<T> &v) { arr(v.data(), (int64_t)v.size()); }
    void csr(const HCsr &A) {
        val(A.nrows);
        val(A.ncols);
        if (A.nrows == 0) {
            arr<int64_t>(nullptr, 0);
            arr<int32_t>(nullptr, 0);
            arr<double>(nullptr, 0);
            return;
        }
        arr(A.rp.data(), A.nrows + 1);
        arr(A.ci.data(), A.nnz());
        arr(A.v.data(), A.nnz());
    }
    void local(const LocalOp &L) {
        val(L.row_begin);
        val(L.row_end);
        val(L.col_begin);
        val(L.col_end);
        val((int32_t)L.full_cols);
        csr(L.A);
        vec(L.ghost);
        val(L.nlo);
        vec(L.send_count);
        vec(L.send_off);
        vec(L.send_idx);
        vec(L.recv_count);
        vec(L.recv_off);
    }
};

struct In {
    const uint8_t *p;
    size_t n, at = 0;
    void get(void *dst, size_t b) {
        if (b > n - at) throw Error{AMG_EINVAL, "truncated hierarchy share"};
        if (b) std::memcpy(dst, p + at, b);
        at += b;
    }
    template <class T>
    T val() {
        T x;
        get(&x, sizeof(T));
        return x;
    }
    int64_t count() {
        const int64_t c = val<int64_t>();
        if (c < 0) throw Error{AMG_EINVAL, "corrupt hierarchy share"};
        return c;
    }
    template <class T>
    void buf(Buf<T> &b) {
        const int64_t c = count();
        b.alloc(c);
        get(b.data(), sizeof(T) * (size_t)c);
    }
    template <class T>
    void vec(std::vector<T> &v) {
        const int64_t c = count();
        v.resize((size_t)c);
        get(v.data(), sizeof(T) * (size_t)c);
    }
    void csr(HCsr &A) {
        A.nrows = val<int64_t>();
        A.ncols = val<int64_t>();
        buf(A.rp);
        buf(A.ci);
        buf(A.v);
        if (A.nrows > 0 && (A.rp.n != A.nrows + 1 || A.ci.n != A.rp[A.nrows] || A.v.n != A.ci.n))
            throw Error{AMG_EINVAL, "corrupt hierarchy share (CSR sizes)"};
    }
    void local(LocalOp &L) {
        L.row_begin = val<int64_t>();
        L.row_end = val<int64_t>();
        L.col_begin = val<int64_t>();
        L.col_end = val<int64_t>();
        L.full_cols = val<int32_t>() != 0;
        csr(L.A);
        vec(L.ghost);
        L.nlo = val<int64_t>();
        vec(L.send_count);
        vec(L.send_off);
        vec(L.send_idx);
        vec(L.recv_count);
        vec(L.recv_off);
    }
};

void write_share(Out &o, const HHierarchy &H, const DistPlan &plan, int rank, int nranks) {
    const int L = H.nlevels;
    o.val(kMagic);
    o.val((int32_t)rank);
    o.val((int32_t)nranks);
    o.val((int32_t)L);
    o.val((int32_t)plan.last_dist);
    o.val(H.prm);
    for (int l = 0; l < L; l++) {
        const HLevel &h = H.lev[l];
        const bool coarsest = l + 1 == L;
        const bool whole = nranks == 1 || l > plan.last_dist;
        o.val(h.N);
        o.val(level_nnz_K(H, l));
        o.val(level_nnz_P(H, l));
        o.val(h.omega);
        o.arr(h.dhat.data(), h.N);
        o.val((int32_t)whole);
        if (nranks > 1) o.vec(plan.lev[l].bounds);
        if (whole) {
            o.csr(h.K);
            if (!coarsest) {
                o.csr(h.P);
                o.csr(h.R);
            }
        } else {
            const DistLevel &D = plan.lev[l];
            o.local(D.K);
            if (!coarsest) {
                o.local(D.P);
                o.local(D.R);
            }
        }
    }
    o.val(kMagic);
}

}  // namespace

void share_export(const HHierarchy &H, int rank, int nranks, int64_t replicate_nnz, uint8_t **blob, int64_t *bytes) {
    if (H.thin) throw Error{AMG_EINVAL, "a hierarchy built from a share cannot be re-shared"};
    if (nranks < 1 || rank < 0 || rank >= nranks) throw Error{AMG_EINVAL, "bad rank/nranks"};
    DistPlan plan;
    plan.last_dist = H.nlevels - 1;
    if (nranks > 1) build_dist_plan(H, rank, nranks, replicate_nnz, plan);
    Out cnt;
    write_share(cnt, H, plan, rank, nranks);
    uint8_t *p = static_cast<uint8_t *>(std::malloc(cnt.n));
    if (!p) throw Error{AMG_ENOMEM, "host allocation failed"};
    Out o;
    o.p = p;
    write_share(o, H, plan, rank, nranks);
    *blob = p;
    *bytes = (int64_t)o.n;
}

void share_import(const void *blob, int64_t bytes, int rank, int nranks, HHierarchy &H, DistPlan &plan) {
    if (!blob || bytes < 0) throw Error{AMG_EINVAL, "NULL share"};
    In in{static_cast<const uint8_t *>(blob), (size_t)bytes};
    if (in.val<uint64_t>() != kMagic) throw Error{AMG_EINVAL, "not a hierarchy share"};
    const int r = in.val<int32_t>(), nr = in.val<int32_t>(), L = in.val<int32_t>(), ld = in.val<int32_t>();
    if (r != rank || nr != nranks) throw Error{AMG_EINVAL, "the share was exported for another rank / rank count"};
    if (L < 1 || L > 32 || ld < 0 || ld >= L) throw Error{AMG_EINVAL, "corrupt hierarchy share"};
    H.prm = in.val<amg_params>();
    H.nlevels = L;
    H.thin = true;
    plan.rank = r;
    plan.nranks = nr;
    plan.last_dist = ld;
    for (int l = 0; l < L; l++) {
        HLevel &h = H.lev[l];
        const bool coarsest = l + 1 == L;
        h.N = in.val<int64_t>();
        h.nnz_K = in.val<int64_t>();
        h.nnz_P = in.val<int64_t>();
        h.omega = in.val<double>();
        in.buf(h.dhat);
        if (h.dhat.n != h.N) throw Error{AMG_EINVAL, "corrupt hierarchy share (diagonal)"};
        const bool whole = in.val<int32_t>() != 0;
        DistLevel &D = plan.lev[l];
        D.replicated = whole;
        if (nr > 1) in.vec(D.bounds);
        if (whole) {
            in.csr(h.K);
            if (!coarsest) {
                in.csr(h.P);
                in.csr(h.R);
            }
        } else {
            in.local(D.K);
            if (!coarsest) {
                in.local(D.P);
                in.local(D.R);
            }
        }
    }
    if (in.val<uint64_t>() != kMagic || in.at != in.n) throw Error{AMG_EINVAL, "corrupt hierarchy share (trailer)"};
}

}  // namespace amgb
