// device.cu — device runtime of the solve phase: level storage in HBM, the V-cycle (c.18) and PCG
// (c.19) as a fixed sequence of fused streaming kernels (kernels.cuh), and the C-ABI entry points
// that need the GPU.
//
// Everything is device-resident after amg_setup: per iteration the host only enqueues kernels and
// reads back one 64-byte scalar block (‖r‖² and breakdown flags) for the convergence test.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"

namespace amgb {

// ---------------------------------------------------------------------------------------------
// allocator hook
// ---------------------------------------------------------------------------------------------
static amg_alloc_fn g_alloc = nullptr;
static amg_free_fn g_free = nullptr;

void set_allocator(amg_alloc_fn a, amg_free_fn f) {
    g_alloc = a;
    g_free = f;
}

#define CUDA_OK(call)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw Error{AMG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};            \
    } while (0)

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// A device operator in one of two streaming formats (kernels.cuh):
//   CSR2 (fmt 0): rows padded to even length; warp per group of G rows.
//   SELL2 (fmt 1): 32-row slices, one row per lane, pair-interleaved columns; soff = slice offsets.
struct DCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;  // stored: entries incl. padding
    int fmt = 0;
    int64_t *rp = nullptr;    // CSR2 row pointers (entries)
    int64_t *soff = nullptr;  // SELL2 slice offsets (pairs)
    int32_t *ci = nullptr;
    double *v = nullptr;
    int G = 32;
};

struct DLevel {
    int64_t N = 0;
    int64_t nnz = 0;  // unpadded nnz(K_l)
    DCsr K, P, R;
    double *invd = nullptr;
    double *b = nullptr, *x = nullptr, *r = nullptr, *d[2] = {nullptr, nullptr};
};

struct DevState {
    int device = 0;
    int nsm = 148;
    int nlevels = 0;
    int m = 4;
    int sweeps = 30;
    DLevel lev[32];
    std::vector<DevBuf> bufs;
    // PCG vectors and scalars
    double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double *partials = nullptr;
    unsigned *counter = nullptr;
    dev::Scalars *S = nullptr;
    dev::Scalars *hS = nullptr;  // pinned host mirror
    double *stage = nullptr;  // device copies of F and u for amg_pcg_solve_host (2·N_0)
    int max_grid = 1184;
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev;
    size_t ev_used = 0;
    int64_t launches_total = 0;
    double bytes_dominant = 0.0;

    void *alloc(size_t bytes) {
        void *p = nullptr;
        if (bytes == 0) bytes = 16;
        if (g_alloc) {
            p = g_alloc(bytes, device, nullptr);
            if (!p) throw Error{AMG_ENOMEM, "device allocation (hook) failed"};
        } else {
            cudaError_t e = cudaMalloc(&p, bytes);
            if (e != cudaSuccess) throw Error{AMG_ENOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e)};
        }
        bufs.push_back({p, bytes});
        return p;
    }
    template <class T>
    T *alloc_n(int64_t n) { return static_cast<T *>(alloc(sizeof(T) * (size_t)std::max<int64_t>(n, 1))); }

    ~DevState() {
        for (auto &b : bufs) {
            if (g_free) g_free(b.p, b.bytes, device, nullptr);
            else cudaFree(b.p);
        }
        for (auto e : ev) cudaEventDestroy(e);
        if (hS) cudaFreeHost(hS);
    }
};

namespace {

int choose_G(int64_t nrows) {
    // enough row groups to give every SM ~64 warps of work, coalesced epilogues where possible
    int64_t target = nrows / (148 * 64);
    int G = 1;
    while (G < 32 && 2 * G <= target) G *= 2;
    return G;
}

// Pad column of row i: the diagonal for square operators, else the row's first column.
inline int32_t pad_col(const HCsr &A, int64_t i, bool square) {
    if (square) return (int32_t)i;
    return A.rp[i + 1] > A.rp[i] ? A.ci[A.rp[i]] : 0;
}

// Upload a host CSR as CSR2 (rows padded to even length with (pad column, 0.0)).
void upload_csr2(DevState &D, const HCsr &A, DCsr &out, bool square) {
    const int64_t n = A.nrows;
    Buf<int64_t> rp(n + 1);
    rp[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t len = A.rp[i + 1] - A.rp[i];
        rp[i + 1] = rp[i] + len + (len & 1);
    }
    const int64_t nnz2 = rp[n];
    Buf<int32_t> ci(nnz2);
    Buf<double> v(nnz2);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        int64_t o = rp[i];
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++, o++) {
            ci[o] = A.ci[k];
            v[o] = A.v[k];
        }
        if (o < rp[i + 1]) {
            ci[o] = pad_col(A, i, square);
            v[o] = 0.0;
        }
    }
    out.fmt = 0;
    out.stored = nnz2;
    out.rp = D.alloc_n<int64_t>(n + 1);
    out.ci = D.alloc_n<int32_t>(nnz2);
    out.v = D.alloc_n<double>(nnz2);
    out.G = choose_G(n);
    CUDA_OK(cudaMemcpy(out.rp, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.ci, ci.data(), sizeof(int32_t) * nnz2, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.v, v.data(), sizeof(double) * nnz2, cudaMemcpyHostToDevice));
}

// Slice offsets (in pairs) of the SELL2 layout; returns the stored entry count.
int64_t sell2_offsets(const HCsr &A, Buf<int64_t> &soff) {
    const int64_t n = A.nrows, nsl = (n + 31) / 32;
    soff.alloc(nsl + 1);
    soff[0] = 0;
    for (int64_t s = 0; s < nsl; s++) {
        int64_t W = 0;
        for (int64_t i = s * 32; i < std::min(n, s * 32 + 32); i++) W = std::max(W, (A.rp[i + 1] - A.rp[i] + 1) / 2);
        soff[s + 1] = soff[s] + 32 * W;
    }
    return 2 * soff[nsl];
}

void upload_sell2(DevState &D, const HCsr &A, DCsr &out, bool square) {
    const int64_t n = A.nrows, nsl = (n + 31) / 32;
    Buf<int64_t> soff;
    const int64_t stored = sell2_offsets(A, soff);
    Buf<int32_t> ci(stored);
    Buf<double> v(stored);
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t s = 0; s < nsl; s++) {
        const int64_t W = (soff[s + 1] - soff[s]) / 32;
        for (int l = 0; l < 32; l++) {
            const int64_t i = s * 32 + l;
            const int64_t b = i < n ? A.rp[i] : 0, len = i < n ? A.rp[i + 1] - A.rp[i] : 0;
            const int32_t pc = i < n ? pad_col(A, i, square) : 0;
            for (int64_t k = 0; k < W; k++)
                for (int h = 0; h < 2; h++) {
                    const int64_t e = 2 * k + h;
                    const int64_t dst = 2 * (soff[s] + 32 * k + l) + h;
                    ci[dst] = e < len ? A.ci[b + e] : pc;
                    v[dst] = e < len ? A.v[b + e] : 0.0;
                }
        }
    }
    out.fmt = 1;
    out.stored = stored;
    out.soff = D.alloc_n<int64_t>(nsl + 1);
    out.ci = D.alloc_n<int32_t>(stored);
    out.v = D.alloc_n<double>(stored);
    CUDA_OK(cudaMemcpy(out.soff, soff.data(), sizeof(int64_t) * (nsl + 1), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.ci, ci.data(), sizeof(int32_t) * stored, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.v, v.data(), sizeof(double) * stored, cudaMemcpyHostToDevice));
}

// Format choice (amg_params.format): 1 = CSR2 everywhere; 2 = SELL2 wherever allowed; 0 = auto:
// SELL2 when there are enough 32-row slices to fill the GPU (>= 4 per SM) and padding <= 10 %.
void upload_op(DevState &D, const HCsr &A, DCsr &out, bool square, int format, bool force_csr) {
    out.nrows = A.nrows;
    out.ncols = A.ncols;
    out.nnz = A.nnz();
    bool sell = false;
    if (!force_csr && format != 1) {
        if (format == 2) {
            sell = true;
        } else {
            Buf<int64_t> soff;
            const int64_t stored = sell2_offsets(A, soff);
            const int64_t nsl = (A.nrows + 31) / 32;
            sell = nsl >= 4 * D.nsm && (double)stored <= 1.10 * (double)std::max<int64_t>(out.nnz, 1);
        }
    }
    if (sell) upload_sell2(D, A, out, square);
    else upload_csr2(D, A, out, square);
}

int grid_for(const DevState &D, int64_t n) {
    int64_t g = (n + dev::kBlock - 1) / dev::kBlock;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, D.max_grid));
}

dev::DotCtx dotctx(DevState &D, int kind) { return dev::DotCtx{D.partials, D.counter, D.S, kind}; }

template <class Epi>
void launch_csr(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind = dev::DOT_NONE) {
    const int2 *ci2 = reinterpret_cast<const int2 *>(A.ci);
    const double2 *v2 = reinterpret_cast<const double2 *>(A.v);
    if (A.fmt == 1) {
        const int64_t nsl = (A.nrows + 31) / 32;
        const int64_t wpb = dev::kBlock / 32;
        int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nsl + wpb - 1) / wpb, D.max_grid));
        dev::k_sell2<Epi><<<grid, dev::kBlock, 0, st>>>(A.soff, ci2, v2, g, A.nrows, epi, dotctx(D, dotkind));
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
        return;
    }
    const int64_t ngroups = (A.nrows + A.G - 1) / A.G;
    const int64_t warps_per_block = dev::kBlock / 32;
    int grid = (int)std::max<int64_t>(1, std::min<int64_t>((ngroups + warps_per_block - 1) / warps_per_block, D.max_grid));
    dev::DotCtx dc = dotctx(D, dotkind);
    switch (A.G) {
#define CASE(GG) \
    case GG: dev::k_csr2<GG, Epi><<<grid, dev::kBlock, 0, st>>>(A.rp, ci2, v2, g, A.nrows, epi, dc); break;
        CASE(1) CASE(2) CASE(4) CASE(8) CASE(16) CASE(32)
#undef CASE
        default: throw Error{AMG_EINVAL, "bad row-group size"};
    }
    D.launches_total++;
    CUDA_OK(cudaGetLastError());
}

// Profiling: events around the dominant kernel (level-0 fused Chebyshev step).
struct ProfScope {
    DevState &D;
    cudaStream_t st;
    bool on;
    ProfScope(DevState &D_, cudaStream_t s, bool dominant) : D(D_), st(s), on(D_.prof && dominant) {
        if (!on) return;
        if (D.ev_used + 2 > D.ev.size()) {
            for (int k = 0; k < 256; k++) {
                cudaEvent_t e;
                CUDA_OK(cudaEventCreate(&e));
                D.ev.push_back(e);
            }
        }
        CUDA_OK(cudaEventRecord(D.ev[D.ev_used], st));
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecord(D.ev[D.ev_used + 1], st);
        D.ev_used += 2;
    }
};

const double kC0 = 4.0 / 3.0;

// c.16 pre-smoothing steps i = 1..m-1 and the residual (a4, a5), restriction (a6), recursion,
// prolongation (a8), post-smoothing (a9, a10).  b, x: this level's right-hand side and output.
void vcycle_level(DevState &D, int l, const double *b, double *x, cudaStream_t st, int final_dot) {
    DLevel &L = D.lev[l];
    const int m = D.m;
    if (l == D.nlevels - 1) {
        const int n = (int)L.N;
        const size_t smem = sizeof(double) * 2 * (size_t)n;
        dev::k_coarse_solve<<<1, 1024, smem, st>>>(n, L.K.rp, L.K.ci, L.K.v, L.invd, b, x, D.sweeps);
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
        return;
    }
    DLevel &C = D.lev[l + 1];
    const bool coarse_is_last = (l + 1 == D.nlevels - 1);
    // --- pre-smoothing from x = 0: d0 = c0·b·invd (level 0 here; coarse levels: restrict epilogue)
    if (l == 0) {
        dev::k_cheb_first<<<grid_for(D, L.N), dev::kBlock, 0, st>>>(L.N, b, L.invd, L.d[0], kC0);
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
    }
    int cur = 0;
    for (int i = 1; i < m; i++) {
        dev::EpiCheb<false> e{};
        e.rin = (i == 1) ? b : L.r;
        e.rout = L.r;
        e.dold = L.d[cur];
        e.dnew = L.d[cur ^ 1];
        e.invd = L.invd;
        e.xin = (i == 1) ? nullptr : x;
        e.dpend = (i == 1) ? L.d[cur] : nullptr;
        e.xout = x;
        e.a = (double)(2 * i - 1) / (double)(2 * i + 3);
        e.bc = (double)(8 * i + 4) / (double)(2 * i + 3);
        ProfScope ps(D, st, l == 0);
        launch_csr(D, L.K, L.d[cur], e, st);
        cur ^= 1;
    }
    // residual r = r − K d_{m−1}   (m == 1: r = b − K d0, x = d0)
    {
        dev::EpiResidualFrom e{};
        e.b = (m == 1) ? b : L.r;
        e.r = L.r;
        e.dpend = (m == 1) ? L.d[cur] : nullptr;
        e.x = x;
        launch_csr(D, L.K, L.d[cur], e, st);
    }
    // restriction b_c = R r, fused with the coarse level's first smoothing step d0_c = c0·b_c·invd_c
    {
        dev::EpiRestrict e{};
        e.bc = C.b;
        e.invd = coarse_is_last ? nullptr : C.invd;
        e.d0 = C.d[0];
        e.c0 = kC0;
        launch_csr(D, L.R, L.r, e, st);
    }
    vcycle_level(D, l + 1, C.b, C.x, st, dev::DOT_NONE);
    // prolongation x += P̄ x_c
    {
        dev::EpiProlong e{};
        e.x = x;
        launch_csr(D, L.P, C.x, e, st);
    }
    // post-smoothing: r = b − K x; d0 = c0·r·invd
    {
        dev::EpiPostFirst e{};
        e.b = b;
        e.r = L.r;
        e.invd = L.invd;
        e.d0 = L.d[0];
        e.c0 = kC0;
        launch_csr(D, L.K, x, e, st);
    }
    cur = 0;
    for (int i = 1; i < m; i++) {
        const bool last = (i == m - 1) && final_dot != dev::DOT_NONE;
        const double a = (double)(2 * i - 1) / (double)(2 * i + 3);
        const double bcf = (double)(8 * i + 4) / (double)(2 * i + 3);
        ProfScope ps(D, st, l == 0);
        if (last) {
            dev::EpiCheb<true> e{};
            e.rin = L.r; e.rout = L.r; e.dold = L.d[cur]; e.dnew = L.d[cur ^ 1]; e.invd = L.invd;
            e.xin = x; e.dpend = (i == 1) ? L.d[cur] : nullptr; e.xout = x; e.bdot = b; e.a = a; e.bc = bcf;
            launch_csr(D, L.K, L.d[cur], e, st, final_dot);
        } else {
            dev::EpiCheb<false> e{};
            e.rin = L.r; e.rout = L.r; e.dold = L.d[cur]; e.dnew = L.d[cur ^ 1]; e.invd = L.invd;
            e.xin = x; e.dpend = (i == 1) ? L.d[cur] : nullptr; e.xout = x; e.bdot = nullptr; e.a = a; e.bc = bcf;
            launch_csr(D, L.K, L.d[cur], e, st);
        }
        cur ^= 1;
    }
    if (m == 1) {
        dev::k_axpy1<<<grid_for(D, L.N), dev::kBlock, 0, st>>>(L.N, L.d[0], x);
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
    }
}

}  // namespace

// V-cycle with the rᵀz dot (kind) fused into the last level-0 post-smoothing step.
static void vcycle(DevState &D, const double *b, double *x, cudaStream_t st, int dotkind) {
    if (D.nlevels == 1) {
        vcycle_level(D, 0, b, x, st, dev::DOT_NONE);
        if (dotkind != dev::DOT_NONE) {
            dev::k_dot<<<grid_for(D, D.lev[0].N), dev::kBlock, 0, st>>>(D.lev[0].N, b, x, dotctx(D, dotkind));
            D.launches_total++;
        }
        return;
    }
    const bool fused = dotkind != dev::DOT_NONE && D.m > 1;
    vcycle_level(D, 0, b, x, st, fused ? dotkind : dev::DOT_NONE);
    if (dotkind != dev::DOT_NONE && !fused) {
        dev::k_dot<<<grid_for(D, D.lev[0].N), dev::kBlock, 0, st>>>(D.lev[0].N, b, x, dotctx(D, dotkind));
        D.launches_total++;
    }
}

DevState *dev_create(const HHierarchy &H, const amg_dist *dist) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw Error{AMG_ENODEV, "no CUDA device"};
    if (dist && dist->nranks > 1) throw Error{AMG_EINVAL, "multi-GPU hierarchies are not built by this version"};
    auto D = new DevState();
    try {
        int dev_id = 0;
        if (dist) {
            dev_id = dist->device;
            CUDA_OK(cudaSetDevice(dev_id));
        } else {
            CUDA_OK(cudaGetDevice(&dev_id));
        }
        D->device = dev_id;
        cudaDeviceProp prop;
        CUDA_OK(cudaGetDeviceProperties(&prop, dev_id));
        if (prop.major < 10) throw Error{AMG_ENODEV, "needs an sm_100a (Blackwell) device"};
        D->nsm = prop.multiProcessorCount;
        D->max_grid = D->nsm * 8;
        D->nlevels = H.nlevels;
        D->m = H.prm.cheb_degree;
        D->sweeps = H.prm.coarse_sweeps;
        for (int l = 0; l < H.nlevels; l++) {
            const HLevel &h = H.lev[l];
            DLevel &L = D->lev[l];
            L.N = h.N;
            L.nnz = h.K.nnz();
            const bool coarsest = (l + 1 == H.nlevels);
            upload_op(*D, h.K, L.K, true, H.prm.format, coarsest);
            if (!coarsest) {
                upload_op(*D, h.P, L.P, false, H.prm.format, false);
                upload_op(*D, h.R, L.R, false, H.prm.format, false);
            }
            Buf<double> invd(h.N);
            for (int64_t i = 0; i < h.N; i++) invd[i] = 1.0 / h.dhat[i];
            L.invd = D->alloc_n<double>(h.N);
            CUDA_OK(cudaMemcpy(L.invd, invd.data(), sizeof(double) * h.N, cudaMemcpyHostToDevice));
            L.b = D->alloc_n<double>(h.N);
            L.x = D->alloc_n<double>(h.N);
            L.r = D->alloc_n<double>(h.N);
            L.d[0] = D->alloc_n<double>(h.N);
            L.d[1] = D->alloc_n<double>(h.N);
        }
        const HLevel &hl = H.lev[H.nlevels - 1];
        if (hl.N > 3072) throw Error{AMG_EINVAL, "coarsest level larger than 3072 rows (raise max_levels)"};
        const int64_t N0 = H.lev[0].N;
        D->r = D->alloc_n<double>(N0);
        D->z = D->alloc_n<double>(N0);
        D->p = D->alloc_n<double>(N0);
        D->q = D->alloc_n<double>(N0);
        D->partials = D->alloc_n<double>(D->max_grid + 32);
        D->counter = D->alloc_n<unsigned>(4);
        D->S = D->alloc_n<dev::Scalars>(1);
        CUDA_OK(cudaMemset(D->counter, 0, 4 * sizeof(unsigned)));
        CUDA_OK(cudaMemset(D->S, 0, sizeof(dev::Scalars)));
        CUDA_OK(cudaMallocHost(&D->hS, sizeof(dev::Scalars)));
        D->bytes_dominant = 12.0 * (double)H.lev[0].K.nnz() + 64.0 * (double)N0;
        CUDA_OK(cudaDeviceSynchronize());
    } catch (...) {
        delete D;
        throw;
    }
    return D;
}

void dev_destroy(DevState *D) { delete D; }

// c.19 — PCG.  F, u: device pointers of length N_0.
static amg_status pcg(DevState &D, const double *F, double *u, double rtol, int maxit, cudaStream_t st, int *iters,
                      double *relres, double *hist) {
    DLevel &L0 = D.lev[0];
    const int64_t N = L0.N;
    *iters = 0;
    *relres = 0.0;
    CUDA_OK(cudaMemsetAsync(D.S, 0, sizeof(dev::Scalars), st));
    // ‖F‖²
    dev::k_dot<<<grid_for(D, N), dev::kBlock, 0, st>>>(N, F, F, dotctx(D, dev::DOT_FF));
    D.launches_total++;
    // r = F − K u ; ‖r‖²
    {
        dev::EpiResidualFrom e{F, D.r, nullptr, nullptr};
        launch_csr(D, L0.K, u, e, st);
    }
    dev::k_dot<<<grid_for(D, N), dev::kBlock, 0, st>>>(N, D.r, D.r, dotctx(D, dev::DOT_RR));
    D.launches_total++;
    CUDA_OK(cudaMemcpyAsync(D.hS, D.S, sizeof(dev::Scalars), cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    const double nF = std::sqrt(D.hS->ff);
    if (nF == 0.0) {
        CUDA_OK(cudaMemsetAsync(u, 0, sizeof(double) * N, st));
        CUDA_OK(cudaStreamSynchronize(st));
        if (hist) hist[0] = 0.0;
        return AMG_OK;
    }
    double rn = std::sqrt(D.hS->rr);
    if (hist) hist[0] = rn / nF;
    *relres = rn / nF;
    if (rn <= rtol * nF) return AMG_OK;
    // z = V(r); ρ = rᵀz; p = z
    vcycle(D, D.r, D.z, st, dev::DOT_RZ_INIT);
    dev::k_p_update<<<grid_for(D, N), dev::kBlock, 0, st>>>(N, D.z, D.p, D.S, 1);
    D.launches_total++;
    amg_status status = AMG_NOT_CONVERGED;
    for (int k = 1; k <= maxit; k++) {
        {
            dev::EpiSpmvDot e{D.p, D.q};
            launch_csr(D, L0.K, D.p, e, st, dev::DOT_PQ);
        }
        dev::k_pcg_update<<<grid_for(D, N), dev::kBlock, 0, st>>>(N, D.p, D.q, u, D.r, dotctx(D, dev::DOT_RR));
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
        CUDA_OK(cudaMemcpyAsync(D.hS, D.S, sizeof(dev::Scalars), cudaMemcpyDeviceToHost, st));
        CUDA_OK(cudaStreamSynchronize(st));
        if (D.hS->flags) {
            *iters = k;
            return AMG_ENOTSPD;
        }
        rn = std::sqrt(D.hS->rr);
        *iters = k;
        *relres = rn / nF;
        if (hist) hist[k] = rn / nF;
        if (rn <= rtol * nF) {
            status = AMG_OK;
            break;
        }
        vcycle(D, D.r, D.z, st, dev::DOT_RZ);
        dev::k_p_update<<<grid_for(D, N), dev::kBlock, 0, st>>>(N, D.z, D.p, D.S, 0);
        D.launches_total++;
    }
    CUDA_OK(cudaGetLastError());
    return status;
}

}  // namespace amgb

// =================================================================================================
// C ABI — device entry points
// =================================================================================================
using namespace amgb;

#define API_BEGIN try {
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

static DevState *need_dev(amg_hierarchy *H) {
    if (!H) throw Error{AMG_EINVAL, "NULL hierarchy"};
    if (!H->dev) throw Error{AMG_ENODEV, "hierarchy has no device part (host_only setup)"};
    CUDA_OK(cudaSetDevice(H->dev->device));
    return H->dev;
}

extern "C" amg_status amg_set_allocator(amg_alloc_fn alloc, amg_free_fn free_fn) {
    if ((alloc == nullptr) != (free_fn == nullptr)) {
        set_error("allocator hook needs both alloc and free (or neither)");
        return AMG_EINVAL;
    }
    set_allocator(alloc, free_fn);
    return AMG_OK;
}

extern "C" amg_status amg_pcg_solve(amg_hierarchy *H, const double *F, double *u, double rtol, int maxit,
                                    void *stream, int *iters, double *relres, double *hist) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!F || !u || !iters || !relres || maxit < 0 || !(rtol >= 0.0)) throw Error{AMG_EINVAL, "bad argument"};
    return pcg(*D, F, u, rtol, maxit, (cudaStream_t)stream, iters, relres, hist);
    API_END
}

extern "C" amg_status amg_pcg_solve_host(amg_hierarchy *H, const double *F, double *u, double rtol, int maxit,
                                         void *stream, int *iters, double *relres, double *hist) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!F || !u || !iters || !relres || maxit < 0 || !(rtol >= 0.0)) throw Error{AMG_EINVAL, "bad argument"};
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = D->lev[0].N;
    if (!D->stage) D->stage = D->alloc_n<double>(2 * N);
    double *dF = D->stage, *dU = D->stage + N;
    CUDA_OK(cudaMemcpyAsync(dF, F, sizeof(double) * N, cudaMemcpyHostToDevice, st));
    CUDA_OK(cudaMemcpyAsync(dU, u, sizeof(double) * N, cudaMemcpyHostToDevice, st));
    amg_status s = pcg(*D, dF, dU, rtol, maxit, st, iters, relres, hist);
    CUDA_OK(cudaMemcpyAsync(u, dU, sizeof(double) * N, cudaMemcpyDeviceToHost, st));
    CUDA_OK(cudaStreamSynchronize(st));
    return s;
    API_END
}

extern "C" amg_status amg_vcycle(amg_hierarchy *H, const double *r, double *z, void *stream) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!r || !z) throw Error{AMG_EINVAL, "bad argument"};
    vcycle(*D, r, z, (cudaStream_t)stream, dev::DOT_NONE);
    CUDA_OK(cudaGetLastError());
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_level_apply(amg_hierarchy *H, int level, int op, const double *x, double *y, void *stream) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (level < 0 || level >= D->nlevels || op < 0 || op > 2 || !x || !y) throw Error{AMG_EINVAL, "bad argument"};
    if (op > 0 && level == D->nlevels - 1) throw Error{AMG_EINVAL, "no transfer operator on the coarsest level"};
    DLevel &L = D->lev[level];
    const DCsr &A = op == 0 ? L.K : op == 1 ? L.P : L.R;
    dev::EpiStore e{y};
    launch_csr(*D, A, x, e, (cudaStream_t)stream);
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_set_profiling(amg_hierarchy *H, int enable) {
    API_BEGIN
    DevState *D = need_dev(H);
    CUDA_OK(cudaDeviceSynchronize());
    D->prof = enable != 0;
    D->ev_used = 0;
    D->launches_total = 0;
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_get_kernel_stats(amg_hierarchy *H, amg_kernel_stats *st) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!st) throw Error{AMG_EINVAL, "NULL stats"};
    CUDA_OK(cudaDeviceSynchronize());
    double total = 0.0;
    for (size_t k = 0; k + 1 < D->ev_used; k += 2) {
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, D->ev[k], D->ev[k + 1]));
        total += ms;
    }
    st->launches = (int64_t)(D->ev_used / 2);
    st->total_ms = total;
    st->bytes_per_launch = D->bytes_dominant;
    st->kernels_launched = D->launches_total;
    return AMG_OK;
    API_END
}
