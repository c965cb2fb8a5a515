// devstate.cuh — device-side state of a hierarchy (internal; not part of the C ABI): operators in
// their streaming layouts, per-level vectors, PCG scalars, graphs and profiling, plus the CSR launcher
// declarations.  The launchers are instantiated per epilogue in the inst_*.cu files so the kernel
// variants compile in parallel.
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <utility>
#include <string>
#include <vector>

#include "common.hpp"
#include "kernels.cuh"

namespace amgb {

#define CUDA_OK(call)                                                                              \
    do {                                                                                           \
        cudaError_t e_ = (call);                                                                   \
        if (e_ != cudaSuccess)                                                                     \
            throw Error{AMG_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_)};            \
    } while (0)

// Programmatic dependent launch of the solve-path kernels (kernels.cuh pdl_enter): each may be
// scheduled while its predecessor drains.  OFF by default (AMG_PDL=1 turns it on): measured on B200 it
// slows the solve — C3 7.26 vs 6.98 ms per iteration, C2 0.286 vs 0.257 ms (run r2n) — since the
// persistent one-wave grids leave no launch gap to hide and the early-resident successor CTAs only
// crowd the predecessor's tail.
inline bool pdl_enabled() {
    static const bool on = [] {
        const char *e = std::getenv("AMG_PDL");
        return e && std::atoi(e) != 0;
    }();
    return on;
}
template <class... KArgs, class... Args>
inline void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CUDA_OK(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
};

// A device operator in one of three streaming formats (kernels.cuh):
//   CSR2 (fmt 0): rows padded to even length; warp per group of G rows.
//   SELL2 (fmt 1): 32-row slices, one row per lane, pair-interleaved columns; soff = slice offsets.
//   SELL-VI (fmt 2): 32-row slices, one row per lane, one 32-bit word per entry (16-bit column offset
//     from rbase | 16-bit value index into vtab) in lane-interleaved quads; soff = slice offsets in
//     quads per lane; G = 32.
// SELL-VI value tables of up to kSellviSmemVals entries (64 KB) are staged in shared memory per CTA
// (C3's K₀: 1,054 values; C4's: 4,147).  At U = 4 the kernel's 80 registers allow 3 CTAs of 256 threads
// per SM, and 3 × 64 KB still fits the SM's shared memory, so staging never lowers the occupancy there.
constexpr int64_t kSellviSmemVals = 8192;
// windowed SELL-VI (k_sellviw): slices per block (= warps per CTA), the largest staged window (doubles;
// further bounded by kWinSmem with the table, device.cu; C3's windows are ≤ 5,950), and the column gap
// below which two runs of a window are merged rather than copied separately
constexpr int kWinSlices = dev::kBlock / 32;
constexpr int64_t kWinMax = 14336;
constexpr int64_t kWinSmem = 110 * 1024;  // window + value table of one CTA: 2 CTAs fit an SM
constexpr int64_t kWinGap = 8;

// Resident CTAs per SM of kernel `fn` at (block, dynamic smem) on the CURRENT device, after raising
// its max-dynamic-shared-memory attribute to `smem_attr` there (0: leave it).  Function attributes
// are per device/context, so both are cached per (kernel, device, smem, smem_attr), under a mutex
// (device.cu).
int resident_ctas(const void *fn, int block, int smem, int smem_attr = 0);

struct DCsr {
    int64_t nrows = 0, ncols = 0, nnz = 0, stored = 0;  // stored: entries incl. padding
    int fmt = 0;
    int mult = 2;  // CSR layouts: every row padded to a multiple of `mult` entries
    int pf = 0;    // register CSR core: L2 bulk prefetch of the next row (autotuned)
    bool l2keep = false;  // register CSR core: normal L2 priority for the streams (fits in L2)
    int64_t *rp = nullptr;    // CSR2 row pointers (entries)
    int64_t *soff = nullptr;  // SELL2 slice offsets (pairs)
    int32_t *ci = nullptr;
    double *v = nullptr;
    int G = 32;    // CSR cores: rows per warp group
    int U = 4;     // CSR cores: pairs per lane per round trip (CSR2) / chunk of 32·U pairs (CSR4T)
    // CSR layouts: kernel (bit 0: 0 register-batched k_csr2, 1 TMA-staged k_csr4t, needs 4-padding),
    // column source (bit 1: 0 int32 columns, 1 16-bit offsets from a per-row base, ColsD16) and value
    // source (bit 3: 0 streamed fp64 values, 1 value index into the distinct-value table; k_csr2 only)
    int kern = 0;
    // 16-bit column offsets (kern & 2): col − rbase[row] per stored entry, rbase = first column of the row
    uint16_t *off16 = nullptr;
    int32_t *rbase = nullptr;
    // value index (kern & 8, register core only; CSR-VI, kernels.cuh): vtab = the operator's distinct
    // values (by decreasing frequency, nvals of them), vidx = per stored entry its index in vtab; vpk =
    // per stored entry (16-bit column offset | value index << 16) when both fit 16 bits
    double *vtab = nullptr;
    int64_t nvals = 0;
    uint32_t *vidx = nullptr;
    uint32_t *vpk = nullptr;
    int obits = 16;  // SELL-VI: column-offset bits of a word (the value index takes the other 32 − obits)
    // windowed SELL-VI (k_sellviw, single GPU): words hold (window position | value index << pbits);
    // binfo per block of kWinSlices slices {first run, end run, window doubles, -}, wruns {first
    // column, doubles, window offset, -}; wmax = the largest window (doubles)
    bool win = false;
    int pbits = 0, wmax = 0;
    int64_t nruns = 0;
    int4 *binfo = nullptr;
    int4 *wruns = nullptr;
    int nbuf = 2;  // windows staged per CTA: 2 (double-buffered) or 1 (autotuned with U)
    int64_t wwhole = 0;  // blocks processed whole; the later ones are split into 2^wl items (k_sellviw)
    int wl = 0;
    // SELL-VI: the slices of the last (partial) round — slice positions >= nwhole — are split into
    // 2^lparts parts of consecutive quads, one warp each, so the tail round is short; partial = the
    // parts' two chains per row, sticket = per-slice arrival counters (zero between launches)
    int lparts = 0;
    int64_t nwhole = 0;
    double2 *partial = nullptr;
    unsigned *sticket = nullptr;
    // bytes one application must stream from HBM for this operator (values of the nnz stored entries
    // or their value indices + the value table, the column data of the chosen source, row pointers);
    // vectors are counted by the caller
    double alg_bytes() const {
        const double z = (double)nnz, rows = (double)nrows;
        if (fmt == 2 && win)  // windowed SELL-VI: 4 B word per entry, the table, slice offsets, block runs
            return 4.0 * z + 8.0 * (double)nvals + 8.0 * (double)((nrows + 31) / 32 + 1) +
                   16.0 * (double)(nruns + (nrows + 32 * kWinSlices - 1) / (32 * kWinSlices));
        if (fmt == 2)  // SELL-VI: 4 B word per entry, the value table, row bases, slice offsets
            return 4.0 * z + 8.0 * (double)nvals + 4.0 * rows + 8.0 * (double)((nrows + 31) / 32 + 1);  // padding excluded
        if (kern & 8) {
            if ((kern & 2) && vpk) return 4.0 * z + 4.0 * rows + 8.0 * (double)nvals + 8.0 * (rows + 1);
            const double cols = (kern & 2) ? 2.0 * z + 4.0 * rows : 4.0 * z;
            return cols + 4.0 * z + 8.0 * (double)nvals + 8.0 * (rows + 1);
        }
        const double idx = (kern & 2) ? 2.0 * z + 4.0 * rows : 4.0 * z;
        return 8.0 * z + idx + 8.0 * (rows + 1);
    }
    float tuned_us = 0.f;  // autotuned apply time (0 if not tuned)
    // halo plan (multi-GPU): ghost g (ascending global id) sits at slot lo_base + g of the gathered
    // vector if g < nlo (lower ranks, negative slots) and at hi_base + g − nlo otherwise.  K_l's ghosts
    // are adjacent to the owned block; P̄_{l−1}'s (the other gatherer of a coarse x) lie beyond them.
    bool halo = false;
    int64_t nown = 0, nghost = 0, nsend = 0, nlo = 0, lo_base = 0, hi_base = 0;
    int64_t slot(int64_t g) const { return g < nlo ? lo_base + g : hi_base + (g - nlo); }
    // P2P transport: part = this operator's kernels take part in the cross-GPU lock-step; push_ptr /
    // push_dst = where this rank's owned entries of the vector this operator GATHERS go on other ranks
    // (rank, slot), CSR over the owned index
    bool part = false;
    unsigned wmask = 0;  // ranks the kernels of this operator wait for (its level's neighbourhood)
    unsigned pmask = 0;  // ranks this operator's push plan sends to
    int *push_ptr = nullptr;
    int2 *push_dst = nullptr;
    std::vector<char> pushed;   // host: owned index i has a push destination
    std::vector<char> bnd;      // host: row i touches a ghost value or is pushed (P2P boundary row)
    std::vector<char> ghostrow; // host: row i reads a ghost column (computed at upload, before the host
                                // operators may be released)
    int *gorder = nullptr;      // device: row groups (of the current G) boundary-first
    int64_t nbnd = 0, gorder_G = 0, gorder_cap = 0;
    int *sidx = nullptr;     // device: local owned indices to send, by destination rank
    double *sbuf = nullptr;  // device: packed send buffer
    std::vector<int> hs_count, hs_off, hr_count, hr_off;  // halo send/recv counts and offsets per rank
};

struct DLevel {
    int64_t N = 0;    // global rows
    int64_t n = 0;    // rows held by this rank (N when replicated or on one GPU)
    int64_t nnz = 0;  // unpadded nnz(K_l)
    bool replicated = false;
    DCsr K, P, R;
    double *invd = nullptr;
    double *diag = nullptr;  // coarsest level: diag(K_L) (§5.1 coarse CG)
    double *b = nullptr, *x = nullptr, *r = nullptr, *d[2] = {nullptr, nullptr};
};

struct DevState {
    int device = 0;
    int nsm = 148;
    int nlevels = 0;
    int m = 4;
    int sweeps = 30;
    DLevel lev[32];
    // multi-GPU (one process per GPU; NCCL over NVLink/NVSwitch)
    int rank = 0, nranks = 1, last_dist = 0;
    ncclComm_t comm = nullptr;
    int64_t row_begin0 = 0, row_end0 = 0;  // this rank's rows of level 0 (global ids)
    // P2P transport (default when nranks > 1; AMG_TRANSPORT=nccl selects NCCL halos): own slab
    // (cudaMalloc, IPC-exported: flags, dot slots, every vector), the other ranks' slabs mapped
    bool p2p = false;
    dev::P2P pp{};
    char *slab = nullptr;
    size_t slab_bytes = 0, slab_used = 0;
    std::vector<char *> peer_slabs;  // opened IPC mappings (closed in the destructor)
    char **d_base = nullptr;         // device array [nranks] of slab bases
    int *ag_ptr = nullptr;           // all-gather push plan of the first replicated level's b
    int64_t ag_row0 = 0;             // this rank's first row of that level
    int2 *ag_dst = nullptr;
    double *ag_send = nullptr, *ag_recv = nullptr;  // all-gather into the first replicated level
    int64_t ag_stride = 0;
    int64_t *ag_bounds = nullptr;                   // device copy of that level's row partition
    std::vector<DevBuf> bufs;
    // PCG vectors and scalars
    double *r = nullptr, *z = nullptr, *p = nullptr, *q = nullptr;
    double *partials = nullptr;
    unsigned *counter = nullptr;
    dev::Scalars *S = nullptr;
    dev::Scalars *hS = nullptr;  // pinned host mirror
    double *stage = nullptr;  // device copies of F and u for amg_pcg_solve_host (2·N_0)
    int max_grid = 1184;
    // solver variants (amg_params): FCG outer iteration, §5.1 coarse CG
    int krylov = 0, coarse_solver = 0, coarse_maxit = 30;
    double coarse_tol = 1e-4;
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev;
    size_t ev_used = 0;
    int64_t launches_total = 0;
    double bytes_dominant = 0.0;
    double prof_ms = 0.0;
    int64_t prof_n = 0;
    // per-level time breakdown (env AMG_PROF_LEVELS=1 with AMG_GRAPHS=0): events at the entry / exit of
    // every level of the V-cycle and around its recursion; exclusive ms per level accumulated
    bool lvl_prof = false;
    std::vector<cudaEvent_t> lev_ev;
    size_t lev_ev_used = 0;
    std::vector<std::pair<int, int>> lev_marks;  // (level, kind) per event: 0 enter, 1 child start, 2 child end, 3 exit
    double lvl_ms[32] = {0};
    int64_t lvl_vcycles = 0;
    // CUDA graphs of the PCG iteration (kind 0: first iteration, 1: later iterations)
    bool graphs = true;
    cudaStream_t cap = nullptr;
    struct Seg {
        cudaGraphExec_t exec = nullptr;
        double *u = nullptr;
        bool prof = false;
        size_t ev0 = 0, ev1 = 0;
        int64_t nk = 0;
    } seg[2];
    // device-side loop (AMG_DEVICE_LOOP, default on with graphs, 1 GPU or the P2P transport): one
    // graph with a conditional WHILE node around one iteration + k_loop_ctl
    bool dev_loop = true;
    dev::LoopCtl *ctl = nullptr;   // device
    dev::LoopCtl *hctl = nullptr;  // pinned host mirror
    double *dhist = nullptr;       // device history, capacity hist_cap
    int hist_cap = 0;
    struct Loop {
        cudaGraphExec_t exec = nullptr;
        double *u = nullptr;
        int64_t nk = 0;  // kernels per iteration
    } loop;

    void *alloc(size_t bytes);  // through the allocator hook (device.cu)
    template <class T>
    T *alloc_n(int64_t n) { return static_cast<T *>(alloc(sizeof(T) * (size_t)std::max<int64_t>(n, 1))); }

    ~DevState();
};


// P2P lock-step descriptor for a kernel: participating kernels get the transport, others none
inline dev::P2P p2p_of(const DevState &D, bool part, unsigned mask = ~0u) {
    if (!(D.p2p && part)) return dev::P2P{};
    dev::P2P p = D.pp;
    p.wait_mask = mask;
    return p;
}
// A kernel working for operator A that waits at its start and publishes at its end (plain kernels).
inline dev::P2P p2p_of(const DevState &D, const DCsr &A) { return p2p_of(D, A.part, A.wmask); }
// The CSR cores on A: with A's boundary-first group order (mid-kernel publication).  ONLY for kernels
// that implement the group order — a plain kernel handed a group order would never publish.
// rows per unit of the boundary-first order: the row group (CSR), the slice (SELL-VI), the 8-slice
// block of the windowed SELL-VI core
inline int64_t order_granule(const DCsr &A) { return A.fmt == 2 && A.win ? 32 * kWinSlices : A.G; }
inline dev::P2P p2p_csr(const DevState &D, const DCsr &A) {
    dev::P2P p = p2p_of(D, A.part, A.wmask);
    if (p.nranks > 0 && (A.fmt == 0 || A.fmt == 2) && A.gorder && A.gorder_G == order_granule(A)) {
        p.gorder = A.gorder;
        p.nbnd = A.nbnd;
    }
    return p;
}
// dot products of the PCG are global: with P2P every rank deposits into every rank's slots
// dotkind = kind | (kind2 << 8): up to two fused dot products of one kernel
inline dev::DotCtx dotctx(DevState &D, int dotkind) {
    return dev::DotCtx{D.partials, D.counter, D.S, dotkind & 255,
                       (dotkind != dev::DOT_NONE) ? p2p_of(D, true) : dev::P2P{}, dotkind >> 8};
}
// push descriptor of `buf` (a vector in the own slab) along operator A's push plan
inline dev::Push push_of(const DevState &D, const DCsr &A, const double *buf) {
    if (!D.p2p || !A.push_ptr || !buf) return dev::Push{};
    return dev::Push{A.push_ptr, A.push_dst, D.d_base, (long long)((const char *)buf - D.slab), D.nranks};
}

// y-side epilogue applied to A·g for a CSR-layout (autotuned kernel / column source) or SELL2 operator.
template <class Epi>
void launch_csr(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind = dev::DOT_NONE);

#define AMGB_EPILOGUES(X) \
    X(dev::EpiStore) X(dev::EpiSpmvDot) X(dev::EpiSpmvDot2) X(dev::EpiResidualFrom) X(dev::EpiCheb<false>) X(dev::EpiCheb<true>) \
    X(dev::EpiPostFirst) X(dev::EpiRestrict) X(dev::EpiProlong)
#define AMGB_EXTERN_LAUNCH(E) \
    extern template void launch_csr<E>(DevState &, const DCsr &, const double *, E, cudaStream_t, int);
AMGB_EPILOGUES(AMGB_EXTERN_LAUNCH)
#undef AMGB_EXTERN_LAUNCH

}  // namespace amgb
