// kernels.cuh — hand-written sm_100a fp64 kernels of the solve phase.
//
// The whole solve phase is HBM-bandwidth bound (≈0.17 flop/B): every kernel below is a streaming
// kernel; no tensor cores (nothing here is a dense contraction).  Matrix streams (values + column
// indices) are ≈99% of the algorithmic bytes, so the design goal is full-rate, coalesced, 128-bit
// streaming of the CSR arrays with the x-gathers served from L1/L2, and every vector update fused
// into the epilogue of the SpMV that produces it.
//
// Matrix layout on the device ("CSR2"): each row padded to an even length with (col = a valid column,
// val = 0.0), so that every row starts 16-byte aligned and is read as double2 values + int2 columns.
// One warp owns a group of G consecutive rows: it reduces one row at a time across its 32 lanes
// (warp-shuffle tree) and parks row t's sum in lane t; the epilogue then runs on G lanes at once, so
// epilogue vector traffic is coalesced (G = 32 on the large levels).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace amgb {
namespace dev {

constexpr int kBlock = 256;

// Checked build (AMG_CHECKS; libamg_b200_checked.so, `python -m paper_2511_21268_b200.build --checked`):
// device-side invariants of the index structures — window positions and copies, value indices, split
// parts and their tickets, ghost-push destinations — print the failing condition and trap.  The
// product build compiles them out.  (compute-sanitizer is not available on the B200 pool: these
// checks and the oracle comparisons stand in for it.)
#ifdef AMG_CHECKS
#define AMG_DCHECK(c)                                                                                    \
    do {                                                                                                 \
        if (!(c)) {                                                                                      \
            printf("AMG_CHECKS: %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, (int)blockIdx.x, \
                   (int)threadIdx.x);                                                                    \
            __trap();                                                                                    \
        }                                                                                                \
    } while (0)
#else
#define AMG_DCHECK(c) ((void)0)
#endif

// Programmatic dependent launch (PDL, opt-in with AMG_PDL=1; devstate.cuh launch_k): a solve-path kernel
// launched with programmatic stream serialization may be scheduled while its predecessor drains.  It
// starts with griddepcontrol.wait — full completion and memory flush of the predecessor, before any
// global access — and then lets its own successor launch (launch_dependents after the wait: at most two
// grids overlap).  Without the launch attribute both instructions are no-ops.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Device scalar block.  Reductions only deposit sums (per rank; the multi-GPU path all-reduces the
// slot right after the kernel); consumers derive α = ρ/pᵀq and β = ρ/ρ_prev themselves, so the
// same kernels serve 1 and N GPUs.  The host reads the whole block once per iteration.
struct Scalars {
    double ff;       // F·F
    double rr;       // r·r (after the CG update)
    double pq;       // pᵀKp
    double rz;       // ρ = rᵀz of the current iteration
    double rz_prev;  // ρ of the previous iteration (set at the end of each iteration)
    double pr;       // FCG: pᵀr (α = pᵀr / pᵀq)
    double zq;       // FCG: zᵀq_prev (β = −zᵀq_prev / pᵀq_prev)
    double pad;
};

// Device-side Krylov loop (one CUDA graph per solve: a conditional WHILE node whose body is one
// iteration + k_loop_ctl, which takes the stopping decision on the device and sets the condition).
struct LoopCtl {
    int k;         // iterations completed
    int maxit;
    int status;    // amg_status of the loop: 0 converged, 1 maxit reached, -5 breakdown
    int first;     // 1 until the first iteration's p = z has run
    double nF;     // ‖F‖₂
    double thr;    // rtol·‖F‖₂
    double *hist;  // [maxit + 1] device: ‖r_k‖/‖F‖
};

enum DotKind { DOT_NONE = 0, DOT_FF, DOT_RR, DOT_PQ, DOT_RZ, DOT_PR, DOT_ZQ, DOT_NKINDS };

__device__ __forceinline__ double *scalar_slot(Scalars *S, int kind) {
    switch (kind) {
        case DOT_FF: return &S->ff;
        case DOT_RR: return &S->rr;
        case DOT_PQ: return &S->pq;
        case DOT_RZ: return &S->rz;
        case DOT_PR: return &S->pr;
        case DOT_ZQ: return &S->zq;
        default: return &S->pad;
    }
}

// accumulation of one (double) or two (double2) fused dot products
__device__ __forceinline__ void acc_add(double &a, double b) { a += b; }
__device__ __forceinline__ void acc_add(double2 &a, double2 b) {
    a.x += b.x;
    a.y += b.y;
}

// ------------------------------------------------------------------------------------------------
// P2P transport of the multi-GPU path (one process per GPU; every rank's "slab" of vectors, flags and
// dot slots is mapped into every other rank's address space over NVLink/NVSwitch).  There is no
// separate communication step: a kernel that produces values another rank gathers STORES them straight
// into that rank's ghost slots from its epilogue (Push), and the kernels run in a cross-GPU lock-step:
// every participating kernel waits at its start until every rank has completed the previous
// participating kernel (flags[q] >= my completed count) and, when its last CTA finishes, publishes its
// own completed count to every rank (release, system scope).  No kernel pushes into the buffer it
// gathers, so this ordering makes every ghost read see the values of the previous kernel and no push
// overwrite a value still being read.
// ------------------------------------------------------------------------------------------------
struct P2P {
    int nranks;                  // 0: no cross-GPU traffic (1 GPU, NCCL transport, or a local-only kernel)
    int rank;
    char *const *base;           // [nranks] slab base of every rank, mapped (base[rank] = own slab)
    unsigned long long *flags;   // own slab: flags[q] = participating kernels completed by rank q
    unsigned long long *epoch;   // own slab: participating kernels completed by this rank
    unsigned *ticket;            // own slab: CTA completion ticket (zero between launches)
    long long flags_off;         // byte offset of flags[] in every slab
    long long dslot_off;         // byte offset of the dot slots dslot[kind][rank] in every slab
    unsigned wait_mask;          // ranks this kernel reads from or writes to (bit q): the ones it waits for
    // CSR cores: row groups in the order BOUNDARY-FIRST.  Boundary groups (positions < nbnd) read ghost
    // values or push theirs: each warp waits before its first one.  When every warp of the grid is past
    // its boundary groups the kernel publishes its count (warp ticket `bticket`), EARLY: the interior
    // groups that follow read only owned values and push nothing, so the neighbours' next kernel does
    // not wait for them.  gorder == nullptr: wait at the kernel start, publish at its end.
    const int *gorder;
    long long nbnd;
    unsigned *bticket;           // own slab: warp ticket of the early publication (zero between launches)
    long long spin_max;          // polls (100 ns apart) before a wait traps: AMG_P2P_SPIN_MAX, default 2^26 ≈ 7 s
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Kernel prologue: wait until every rank in wait_mask has completed as many participating kernels as
// this one.  A kernel that gathers ghosts pushed by rank q, or pushes into rank q's ghost slots, has q in
// its mask (RAW and WAR across ranks); dot products and the all-gather wait for every rank.
// Bounded: a peer that never arrives (a dead rank) traps after pp.spin_max polls (AMG_P2P_SPIN_MAX;
// default ≈ 7 s) instead of hanging the GPU.  Callers enter a solve on every rank within that bound.
__device__ __forceinline__ void peer_wait(const P2P &pp) {
    if (pp.nranks == 0) return;
    if (threadIdx.x == 0) {
        const unsigned long long e = *(volatile unsigned long long *)pp.epoch;
        for (int q = 0; q < pp.nranks; q++) {
            if (!((pp.wait_mask >> q) & 1u)) continue;
            long long spins = 0;
            while (ld_acquire_sys(pp.flags + q) < e) {
                __nanosleep(100);
                if (++spins > pp.spin_max) __trap();
            }
        }
    }
    __syncthreads();
}

// Warp-level wait of the interior-first CSR cores (lane 0 polls; __syncwarp orders the warp's loads).
__device__ __forceinline__ void peer_wait_warp(const P2P &pp) {
    if (pp.nranks == 0) return;
    if ((threadIdx.x & 31) == 0) {
        const unsigned long long e = *(volatile unsigned long long *)pp.epoch;
        for (int q = 0; q < pp.nranks; q++) {
            if (!((pp.wait_mask >> q) & 1u)) continue;
            long long spins = 0;
            while (ld_acquire_sys(pp.flags + q) < e) {
                __nanosleep(100);
                if (++spins > pp.spin_max) __trap();
            }
        }
    }
    __syncwarp();
}

// Early publication of the boundary-first CSR cores: each warp calls it once, after its last boundary
// group (all its pushes issued); the last warp of the grid publishes the new count.
__device__ __forceinline__ void peer_signal_warp(const P2P &pp) {
    if (pp.nranks == 0) return;
    __syncwarp();
    if ((threadIdx.x & 31) == 0) {
        __threadfence_system();
        const unsigned total = gridDim.x * (blockDim.x >> 5);
        const unsigned t = atomicAdd(pp.bticket, 1u);
        if (t == total - 1) {
            __threadfence_system();
            const unsigned long long e = *(volatile unsigned long long *)pp.epoch + 1ull;
            *(volatile unsigned long long *)pp.epoch = e;
            *(volatile unsigned *)pp.bticket = 0u;
            for (int q = 0; q < pp.nranks; q++)
                st_release_sys(reinterpret_cast<unsigned long long *>(pp.base[q] + pp.flags_off) + pp.rank, e);
        }
    }
    __syncwarp();
}

// Early publication of the windowed SELL-VI core (block-granular boundary-first order): each CTA checks
// in once, after the barrier that ended its last boundary item (every thread's pushes issued); the
// last CTA of the grid publishes the new count.  Counts CTAs on the same bticket as the warp version.
__device__ __forceinline__ void peer_signal_cta(const P2P &pp) {
    if (pp.nranks == 0) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned t = atomicAdd(pp.bticket, 1u);
        if (t == gridDim.x - 1) {
            __threadfence_system();
            const unsigned long long e = *(volatile unsigned long long *)pp.epoch + 1ull;
            *(volatile unsigned long long *)pp.epoch = e;
            *(volatile unsigned *)pp.bticket = 0u;
            for (int q = 0; q < pp.nranks; q++)
                st_release_sys(reinterpret_cast<unsigned long long *>(pp.base[q] + pp.flags_off) + pp.rank, e);
        }
    }
    __syncthreads();
}

// Kernel epilogue (every CTA, after all its stores): the last CTA to finish publishes the new count.
__device__ __forceinline__ void peer_signal(const P2P &pp) {
    if (pp.nranks == 0 || pp.gorder) return;  // boundary-first kernels published early
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence_system();
        const unsigned t = atomicAdd(pp.ticket, 1u);
        if (t == gridDim.x - 1) {
            __threadfence_system();
            const unsigned long long e = *(volatile unsigned long long *)pp.epoch + 1ull;
            *(volatile unsigned long long *)pp.epoch = e;
            *(volatile unsigned *)pp.ticket = 0u;
            for (int q = 0; q < pp.nranks; q++)
                st_release_sys(reinterpret_cast<unsigned long long *>(pp.base[q] + pp.flags_off) + pp.rank, e);
        }
    }
}

// Ghost-value push list of one gathered vector: owned row i goes to (rank, slot) for
// t in [ptr[i], ptr[i+1]); the destination is base[rank] + voff + 8·slot (the gathering rank's ghost
// area of that vector).  ptr == nullptr: nothing to push.
struct Push {
    const int *ptr;
    const int2 *dst;
    char *const *base;
    long long voff;
    int nranks = 0;  // checked build: destination ranks are < nranks
    __device__ __forceinline__ void put(int64_t i, double v) const {
        if (!ptr) return;
        const int b = ptr[i], e = ptr[i + 1];
        AMG_DCHECK(b <= e);
        for (int t = b; t < e; t++) {
            const int2 d = dst[t];
            AMG_DCHECK(d.x >= 0 && (nranks == 0 || d.x < nranks));
            *reinterpret_cast<double *>(base[d.x] + voff + 8ll * d.y) = v;
        }
    }
};

struct DotCtx {
    double *partials;    // >= 2·gridDim.x
    unsigned *counter;   // zero between launches
    Scalars *S;
    int kind;
    P2P pp;              // nranks > 0: deposit the rank's sum in every rank's dslot[kind][rank] instead
    int kind2;           // second fused dot (double2 accumulators), DOT_NONE if none
};

__device__ __forceinline__ double warp_sum(double s) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    return s;
}

// Deterministic block reduction + "last block finalises" (fixed partial order ⇒ run-to-run
// identical scalars; no atomics on values).  NV values (1 or 2 fused dots) per launch.
template <int BS, int NV>
__device__ __forceinline__ void block_dot_finalize_v(const double *v, const DotCtx &dc) {
    __shared__ double red[NV][BS / 32];
    __shared__ bool last;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; k++) {
        const double t = warp_sum(v[k]);
        if (lane == 0) red[k][wid] = t;
    }
    __syncthreads();
    if (wid == 0) {
#pragma unroll
        for (int k = 0; k < NV; k++) {
            double t = lane < BS / 32 ? red[k][lane] : 0.0;
            t = warp_sum(t);
            if (lane == 0) dc.partials[(size_t)k * gridDim.x + blockIdx.x] = t;
        }
        if (lane == 0) {
            __threadfence();
            unsigned ticket = atomicAdd(dc.counter, 1u);
            last = (ticket == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    double tot[NV];
#pragma unroll
    for (int k = 0; k < NV; k++) {
        double t = 0.0;
        for (unsigned i = threadIdx.x; i < gridDim.x; i += BS) t += __ldcg(dc.partials + (size_t)k * gridDim.x + i);
        t = warp_sum(t);
        __syncthreads();
        if (lane == 0) red[k][wid] = t;
        __syncthreads();
        double s = 0.0;
        for (int w = 0; w < BS / 32; w++) s += red[k][w];
        tot[k] = s;
    }
    if (threadIdx.x == 0) {
        const int kinds[2] = {dc.kind, dc.kind2};
        for (int k = 0; k < NV; k++) {
            if (dc.pp.nranks > 0) {  // P2P: every rank sums the slots in rank order (k_dot_collect)
                for (int q = 0; q < dc.pp.nranks; q++)
                    *reinterpret_cast<double *>(dc.pp.base[q] + dc.pp.dslot_off +
                                                8ll * (kinds[k] * dc.pp.nranks + dc.pp.rank)) = tot[k];
            } else {
                *scalar_slot(dc.S, kinds[k]) = tot[k];
            }
        }
        *dc.counter = 0u;
    }
}

template <int BS>
__device__ __forceinline__ void block_dot_finalize_n(double v, const DotCtx &dc) {
    block_dot_finalize_v<BS, 1>(&v, dc);
}
template <int BS>
__device__ __forceinline__ void block_dot_finalize_n(double2 v, const DotCtx &dc) {
    const double a[2] = {v.x, v.y};
    block_dot_finalize_v<BS, 2>(a, dc);
}

template <class T>
__device__ __forceinline__ void block_dot_finalize(T v, const DotCtx &dc) { block_dot_finalize_n<kBlock>(v, dc); }

// ------------------------------------------------------------------------------------------------
// Epilogues.  load(row) fetches the row's vector inputs; the cores call it when a row group STARTS, so
// these loads are in flight together with the matrix stream instead of adding a dependent DRAM round
// trip after the row sum.  operator()(row, s, pre) consumes the row sum s = (A·g)_row and returns the
// row's contribution to the fused dot product (ignored unless kDot).
// ------------------------------------------------------------------------------------------------
struct NoPre {};

struct EpiStore {  // y = A x
    static constexpr bool kDot = false;
    using Acc = double;
    using Pre = NoPre;
    double *y;
    __device__ __forceinline__ Pre load(int64_t) const { return {}; }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &) const { y[i] = s; return 0.0; }
};

struct EpiSpmvDot {  // a1: q = K p, pᵀq
    static constexpr bool kDot = true;
    using Acc = double;
    struct Pre { double p; };
    const double *p;
    double *q;
    __device__ __forceinline__ Pre load(int64_t i) const { return {p[i]}; }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &pr) const {
        q[i] = s;
        return pr.p * s;
    }
};

// a1 for the flexible CG: q = K p with both pᵀq and pᵀr (α = pᵀr / pᵀq)
struct EpiSpmvDot2 {
    static constexpr bool kDot = true;
    using Acc = double2;
    struct Pre { double p, r; };
    const double *p;
    const double *r;
    double *q;
    __device__ __forceinline__ Pre load(int64_t i) const { return {p[i], r[i]}; }
    __device__ __forceinline__ double2 operator()(int64_t i, double s, const Pre &pr) const {
        q[i] = s;
        return make_double2(pr.p * s, pr.p * pr.r);
    }
};

struct EpiResidualFrom {  // r = b − K x  (also: r −= K d with b == r);  optionally x = dpend
    static constexpr bool kDot = false;
    using Acc = double;
    struct Pre { double b, dp; };
    const double *b;
    double *r;
    const double *dpend;  // nullable: x = dpend (degree-1 pre-smoothing)
    double *x;
    Push pushR;           // r to the ranks whose restriction gathers it
    __device__ __forceinline__ Pre load(int64_t i) const { return {b[i], dpend ? dpend[i] : 0.0}; }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &pr) const {
        const double rr = pr.b - s;
        r[i] = rr;
        if (dpend) x[i] = pr.dp;
        pushR.put(i, rr);
        return 0.0;
    }
};

// a4/a10: fused Chebyshev step (Lottes 4th kind, ρ = 1; SURVEY c.16):
//   r = rin − K d_old;  d_new = a·d_old + bc·(r·invd);  x = ((xin or 0) + dpend) + d_new.
template <bool kDotRZ>
struct EpiCheb {
    static constexpr bool kDot = kDotRZ;
    using Acc = double;
    struct Pre { double rin, dold, invd, xin, dp, bd; };  // raw loads only: no arithmetic until the row sum
    const double *rin;
    double *rout;
    const double *dold;
    double *dnew;
    const double *invd;
    const double *xin;    // nullable (x = 0 on entry)
    const double *dpend;  // nullable (pending d_0 not yet added to x)
    double *xout;
    const double *bdot;   // kDotRZ: returns bdot[i]·x_new[i]
    double a, bc;
    Push pushD, pushX;    // d_new (gathered by the next step) / x (gathered by the coarse-to-fine P̄)
    __device__ __forceinline__ Pre load(int64_t i) const {
        Pre p;
        p.rin = rin[i];
        p.dold = dold[i];
        p.invd = invd[i];
        p.xin = xin ? xin[i] : 0.0;
        p.dp = dpend ? dpend[i] : 0.0;
        p.bd = kDotRZ ? bdot[i] : 0.0;
        return p;
    }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &p) const {
        const double r = p.rin - s;
        const double dn = a * p.dold + bc * (r * p.invd);
        double x = p.xin;
        if (dpend) x = x + p.dp;
        x = x + dn;
        rout[i] = r;
        dnew[i] = dn;
        xout[i] = x;
        pushD.put(i, dn);
        pushX.put(i, x);
        return kDotRZ ? p.bd * x : 0.0;
    }
};

struct EpiPostFirst {  // a9: r = b − K x;  d0 = c0·(r·invd)  (x += d0 is folded into the next step)
    static constexpr bool kDot = false;
    using Acc = double;
    struct Pre { double b, invd; };
    const double *b;
    double *r;
    const double *invd;
    double *d0;
    double c0;
    Push pushD;
    __device__ __forceinline__ Pre load(int64_t i) const { return {b[i], invd[i]}; }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &p) const {
        const double rr = p.b - s;
        const double d = c0 * (rr * p.invd);
        r[i] = rr;
        d0[i] = d;
        pushD.put(i, d);
        return 0.0;
    }
};

struct EpiRestrict {  // a6 (+a3 of the coarse level): b_c = R r;  d0_c = c0·(b_c·invd_c)
    static constexpr bool kDot = false;
    using Acc = double;
    struct Pre { double invd; };
    double *bc;
    const double *invd;  // nullable (coarsest level: no smoother)
    double *d0;
    double c0;
    Push pushB, pushD;  // b_c to every rank (replicated coarse level) / d0_c to the coarse halo
    __device__ __forceinline__ Pre load(int64_t i) const { return {invd ? invd[i] : 0.0}; }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &p) const {
        bc[i] = s;
        pushB.put(i, s);
        if (invd) {
            const double d = c0 * (s * p.invd);
            d0[i] = d;
            pushD.put(i, d);
        }
        return 0.0;
    }
};

struct EpiProlong {  // a8: x += P̄ e
    static constexpr bool kDot = false;
    using Acc = double;
    struct Pre { double x; };
    double *x;
    Push pushX;
    __device__ __forceinline__ Pre load(int64_t i) const { return {x[i]}; }
    __device__ __forceinline__ double operator()(int64_t i, double s, const Pre &p) const {
        const double xn = p.x + s;
        x[i] = xn;
        pushX.put(i, xn);
        return 0.0;
    }
};

// ------------------------------------------------------------------------------------------------
// The streaming CSR2 core: warp per group of G rows, 128-bit loads, 2 row chunks in flight per lane.
// ------------------------------------------------------------------------------------------------
// Matrix streams: read once, keep them out of L1 (L1 holds the gathered vector).  `volatile` keeps
// ptxas from interleaving a stalled gather between the batched stream loads (SASS-checked: without it
// only ~2 stream loads were in flight per lane).
// L2 policy of the matrix streams: evict-first, so the 3.7 GB fine-level stream does not push the
// gathered vector and the epilogue vectors (≈ 8 MB each at C3) out of the 126 MB L2.
__device__ __forceinline__ uint64_t stream_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
// Normal L2 priority for operators small enough to stay L2-resident across their repeated
// applications in a V-cycle (DCsr::l2keep): their lines survive the evict-first streams of the large
// levels.
__device__ __forceinline__ uint64_t keep_policy() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ double2 ld_stream(const double2 *p, uint64_t pol) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int2 ld_stream(const int2 *p, uint64_t pol) {
    int2 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;"
                 : "=r"(r.x), "=r"(r.y)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ double ld_stream(const double *p, uint64_t pol) {
    double r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ int ld_stream(const int *p, uint64_t pol) {
    int r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ unsigned ld_stream(const unsigned short *p, uint64_t pol) {
    unsigned short r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ unsigned ld_stream(const unsigned *p, uint64_t pol) {
    unsigned r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
    return r;
}
// L2 prefetch of a contiguous byte range by one thread (bulk async copy engine; no registers held).
// Address and size must be multiples of 16.
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
// Gather of the multiplied vector through the read-only path (L1-allocating).
__device__ __forceinline__ double ld_gather(const double *p) {
    double r;
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
}

// Entry sources of the CSR cores (the column and the value of stored entry k).  row(i) returns the
// per-row state; the register core loads word(k) — the entry's streamed index data — for a whole batch
// of entries first, then val(v, k, w) for the batch, then gathers x[col(w, row state)].  Every source
// yields the same columns and bitwise the same values, so the choice changes bytes and speed, never
// results.  kVals: the values are streamed from v (else val() looks them up in a value table).  The TMA
// core stages the column stream (stream(k), kIdxBytes per entry) with the values into shared memory.
//
// ColsI32: plain int32 columns (4 B per entry), streamed like the values.
struct ColsI32 {
    static constexpr int kIdxBytes = 4;  // bytes per entry of the staged column stream
    static constexpr bool kVals = true;
    using W = int;
    const int *ci;
    __device__ __forceinline__ int row(int64_t) const { return 0; }
    __device__ __forceinline__ W word(int64_t k, uint64_t pol) const { return ld_stream(ci + k, pol); }
    __device__ __forceinline__ int col(W w, int) const { return w; }
    __device__ __forceinline__ double val(const double *v, int64_t k, W, uint64_t pol) const { return ld_stream(v + k, pol); }
    __device__ __forceinline__ void prefetch(int64_t b, int64_t e) const { prefetch_l2(ci + b, (uint32_t)((e - b) * 4)); }
    __device__ __forceinline__ const void *stream(int64_t k) const { return ci + k; }
    __device__ __forceinline__ int staged(const unsigned char *sidx, int j, int) const {
        return reinterpret_cast<const int *>(sidx)[j];
    }
};

// ColsD16: 16-bit column offsets ("CSR-D16").  base[i] = the first (smallest) column of row i and every
// stored entry holds col − base[i] in 16 bits.  Any operator whose rows each span < 65536 columns
// qualifies — the C3 levels span ≤ 57,624 (fine) and ≤ 33,325 (coarse) columns per row — and its column
// stream shrinks from 4 to 2 B per entry (12 → 10 B per non-zero with the value).
struct ColsD16 {
    static constexpr int kIdxBytes = 2;
    static constexpr bool kVals = true;
    using W = unsigned;
    const unsigned short *off;
    const int *base;  // per row
    __device__ __forceinline__ int row(int64_t i) const { return __ldg(base + i); }
    __device__ __forceinline__ W word(int64_t k, uint64_t pol) const { return ld_stream(off + k, pol); }
    __device__ __forceinline__ int col(W w, int b) const { return b + (int)w; }
    __device__ __forceinline__ double val(const double *v, int64_t k, W, uint64_t pol) const { return ld_stream(v + k, pol); }
    __device__ __forceinline__ void prefetch(int64_t b, int64_t e) const { prefetch_l2(off + b, (uint32_t)((e - b) * 2)); }
    __device__ __forceinline__ const void *stream(int64_t k) const { return off + k; }
    __device__ __forceinline__ int staged(const unsigned char *sidx, int j, int b) const {
        return b + (int)reinterpret_cast<const unsigned short *>(sidx)[j];
    }
};

// Value-indexed sources ("CSR-VI": Kourtis, Goumas, Koziris, "Optimizing sparse matrix-vector
// multiplication using index and value compression", CF 2008).  An operator with few distinct values
// stores each entry's value as an index into a table of its distinct values (most frequent first,
// built on the host); the value read is an L1-resident table lookup instead of 8 streamed bytes.  The
// IgA operators are full of repeated values (C3: K_0 has 306 M entries but 1,053 distinct values, K_1
// 190 K) because every interior row is the same stencil.  Values are bitwise the stored ones (a
// lossless format), so row sums are bitwise those of the streamed-value sources.  Tail entries beyond a
// row's end (k >= e) are never looked up.
//
// ColsD16V16: one 32-bit word per entry: low half the 16-bit column offset (as ColsD16), high half the
// value index (< 65536 distinct values): 4 B per entry instead of 10.
struct ColsD16V16 {
    static constexpr int kIdxBytes = 4;
    static constexpr bool kVals = false;
    using W = unsigned;
    const unsigned *w;
    const int *base;      // per row
    const double *table;  // distinct values
    __device__ __forceinline__ int row(int64_t i) const { return __ldg(base + i); }
    __device__ __forceinline__ W word(int64_t k, uint64_t pol) const { return ld_stream(w + k, pol); }
    __device__ __forceinline__ int col(W x, int b) const { return b + (int)(x & 0xffffu); }
    __device__ __forceinline__ double val(const double *, int64_t, W x, uint64_t) const { return ld_gather(table + (x >> 16)); }
    __device__ __forceinline__ void prefetch(int64_t b, int64_t e) const { prefetch_l2(w + b, (uint32_t)((e - b) * 4)); }
};

// ColsD16V32: 16-bit column offsets + a 32-bit value index per entry (6 B per entry instead of 10).
struct ColsD16V32 {
    static constexpr int kIdxBytes = 6;
    static constexpr bool kVals = false;
    using W = uint2;
    const unsigned short *off;
    const unsigned *vi;
    const int *base;
    const double *table;
    __device__ __forceinline__ int row(int64_t i) const { return __ldg(base + i); }
    __device__ __forceinline__ W word(int64_t k, uint64_t pol) const {
        return make_uint2(ld_stream(off + k, pol), ld_stream(vi + k, pol));
    }
    __device__ __forceinline__ int col(W x, int b) const { return b + (int)x.x; }
    __device__ __forceinline__ double val(const double *, int64_t, W x, uint64_t) const { return ld_gather(table + x.y); }
    __device__ __forceinline__ void prefetch(int64_t b, int64_t e) const {
        prefetch_l2(off + b, (uint32_t)((e - b) * 2));
        prefetch_l2(vi + b, (uint32_t)((e - b) * 4));
    }
};

// ColsI32V32: int32 columns + a 32-bit value index (8 B per entry instead of 12).
struct ColsI32V32 {
    static constexpr int kIdxBytes = 8;
    static constexpr bool kVals = false;
    using W = uint2;
    const int *ci;
    const unsigned *vi;
    const double *table;
    __device__ __forceinline__ int row(int64_t) const { return 0; }
    __device__ __forceinline__ W word(int64_t k, uint64_t pol) const {
        return make_uint2((unsigned)ld_stream(ci + k, pol), ld_stream(vi + k, pol));
    }
    __device__ __forceinline__ int col(W x, int) const { return (int)x.x; }
    __device__ __forceinline__ double val(const double *, int64_t, W x, uint64_t) const { return ld_gather(table + x.y); }
    __device__ __forceinline__ void prefetch(int64_t b, int64_t e) const {
        prefetch_l2(ci + b, (uint32_t)((e - b) * 4));
        prefetch_l2(vi + b, (uint32_t)((e - b) * 4));
    }
};

// The streaming CSR core: one warp owns a group of G consecutive rows and reduces one row at a time.
// Rows are padded to a multiple of 8 entries (64-byte aligned).  A row is walked in windows of 64
// entries; lane l multiplies entries l and l+32 of each window (two 256-byte value loads per warp
// instruction, and the x-gathers of one instruction hit ≈ 6 cache lines instead of ≈ 11 for an
// (2l, 2l+1) pairing, measured on the C3 levels), accumulating them in two separate chains.  U windows
// are loaded back to back before any is consumed.  The row sum is a fixed xor-shuffle tree of the
// 32 lanes' (chain0 + chain1); all CSR kernel variants use exactly this order (bitwise-equal results).
// pf bit 0: while reducing row t of a group, lane 0 has the bulk-copy engine prefetch row t+1's values
// and column data into L2, so the next row's loads hit L2 instead of DRAM (more bytes in flight per
// warp without holding registers).  pf bit 1: the matrix streams use the normal L2 priority instead of
// evict-first (operators that fit in L2; DCsr::l2keep).
template <int G, int U, class Epi, class Cols>
__global__ void __launch_bounds__(kBlock) k_csr2(const int64_t *__restrict__ rp, Cols cols,
                                                 const double *__restrict__ v, const double *__restrict__ g,
                                                 int64_t nrows, Epi epi, DotCtx dc, P2P pp, int pf) {
    pdl_enter();
    if (!pp.gorder) peer_wait(pp);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t ngroups = (nrows + G - 1) / G;
    const uint64_t pol = (pf & 2) ? keep_policy() : stream_policy();
    typename Epi::Acc dacc{};
    bool signalled = pp.gorder == nullptr || pp.nranks == 0;
    if (!signalled && warp < pp.nbnd) peer_wait_warp(pp);  // this warp has boundary groups
    for (int64_t pos = warp; pos < ngroups; pos += nwarps) {
        if (!signalled && pos >= pp.nbnd) {  // past this warp's boundary groups
            peer_signal_warp(pp);
            signalled = true;
        }
        const int64_t grp = pp.gorder ? (int64_t)__ldg(pp.gorder + pos) : pos;
        const int64_t r0 = grp * G;
        const int nr = (int)(nrows - r0 < (int64_t)G ? nrows - r0 : (int64_t)G);
        // group prologue, one round trip for the whole group: lane t fetches row r0+t's pointers and
        // column-source state (broadcast by shuffles below) and its epilogue inputs
        typename Epi::Pre pre{};
        int64_t gb = 0, ge = 0;
        int grs = 0;
        if (lane < nr) {
            gb = __ldg(rp + r0 + lane);
            ge = __ldg(rp + r0 + lane + 1);
            grs = cols.row(r0 + lane);
            pre = epi.load(r0 + lane);
        }
        double mine = 0.0;
        for (int t = 0; t < nr; t++) {
            const int64_t b = __shfl_sync(0xffffffffu, gb, t), e = __shfl_sync(0xffffffffu, ge, t);
            const int rs = __shfl_sync(0xffffffffu, grs, t);
            if ((pf & 1) && t + 1 < nr) {
                const int64_t nb = __shfl_sync(0xffffffffu, gb, t + 1), ne = __shfl_sync(0xffffffffu, ge, t + 1);
                // rows are padded to 8 entries: every stream's range is 16-byte aligned
                if (lane == 0 && ne > nb && (nb & 7) == 0 && ((ne - nb) & 7) == 0) {
                    if constexpr (Cols::kVals) prefetch_l2(v + nb, (uint32_t)((ne - nb) * 8));
                    cols.prefetch(nb, ne);
                }
            }
            double s0 = 0.0, s1 = 0.0;
            for (int64_t k0 = b + lane; k0 < e; k0 += 64 * U) {
                double va[U], vb[U];
                typename Cols::W wa[U], wb[U];
                // past the row end: column 0 (always a valid index) with value 0.0 — no sentinel, since
                // distributed operators have negative (lower-ghost) columns
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t ka = k0 + 64 * u, kb = ka + 32;
                    if (ka < e) wa[u] = cols.word(ka, pol);
                    if (kb < e) wb[u] = cols.word(kb, pol);
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t ka = k0 + 64 * u, kb = ka + 32;
                    va[u] = ka < e ? cols.val(v, ka, wa[u], pol) : 0.0;
                    vb[u] = kb < e ? cols.val(v, kb, wb[u], pol) : 0.0;
                }
                double xa[U], xb[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const int64_t ka = k0 + 64 * u, kb = ka + 32;
                    xa[u] = ld_gather(g + (ka < e ? cols.col(wa[u], rs) : 0));
                    xb[u] = ld_gather(g + (kb < e ? cols.col(wb[u], rs) : 0));
                }
#pragma unroll
                for (int u = 0; u < U; u++) {
                    s0 = fma(va[u], xa[u], s0);
                    s1 = fma(vb[u], xb[u], s1);
                }
            }
            const double s = warp_sum(s0 + s1);
            if (lane == t) mine = s;
        }
        if (lane < nr) acc_add(dacc, epi(r0 + lane, mine, pre));
    }
    if (!signalled) peer_signal_warp(pp);  // only boundary groups (or none) for this warp
    if constexpr (Epi::kDot) block_dot_finalize(dacc, dc);
    peer_signal(pp);
}

// ------------------------------------------------------------------------------------------------
// TMA-staged CSR core ("CSR4T"): rows padded to a multiple of 8 entries, so every row's value and
// column-stream ranges are 16-byte aligned multiples of 16 bytes.  Each warp walks its rows in chunks of
// 64·U entries; one elected lane keeps the next NS−1 chunks' values and column data (int32 or 16-bit
// offsets) in flight into an NS-stage shared-memory ring with cp.async.bulk (TMA, completion on an
// mbarrier per stage) while the warp reduces the current chunk from shared memory and gathers x through
// L1/L2: the HBM stream never waits for the gathers or for registers.  Lane l takes entries l and l+32
// of every 64-entry window, in the same two chains as k_csr2 (bitwise-equal row sums).
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

constexpr int kBlockT = 128;  // 4 warps per CTA for the TMA-staged core

constexpr int kTmaStages = 3;

template <int U, int kIdxBytes>
struct TmaCfg {
    static constexpr int NS = kTmaStages;
    static constexpr int CH = 64 * U;                         // entries per chunk
    static constexpr int IDX = CH * 8;                        // offset of the column data in a stage
    static constexpr int STAGE = CH * (8 + kIdxBytes);        // bytes per stage
    static constexpr int WARP = (NS * STAGE + 8 * NS + 127) / 128 * 128;  // NS stages + NS mbarriers, 128-B aligned
    static constexpr int SMEM = (kBlockT / 32) * WARP;        // dynamic shared memory per CTA
};

template <int G, int U, class Epi, class Cols>
__global__ void __launch_bounds__(kBlockT) k_csr4t(const int64_t *__restrict__ rp, Cols cols,
                                                   const double *__restrict__ v, const double *__restrict__ g,
                                                   int64_t nrows, Epi epi, DotCtx dc, P2P pp) {
    pdl_enter();
    if (!pp.gorder) peer_wait(pp);
    using C = TmaCfg<U, Cols::kIdxBytes>;
    constexpr int NS = C::NS;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    unsigned char *wb = smem + wib * C::WARP;
    uint64_t *bar = reinterpret_cast<uint64_t *>(wb + NS * C::STAGE);
    if (lane == 0) {
        for (int k = 0; k < NS; k++) mbar_init(&bar[k], 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t warp = ((int64_t)blockIdx.x * kBlockT + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlockT) >> 5;
    const int64_t ngroups = (nrows + G - 1) / G;
    const uint64_t pol = stream_policy();

    // chunk cursor: position in the group order, group, row-in-group, entry range [k0, min(k0+CH, e))
    struct Cur {
        int64_t pos, grp, k0, e;
        int t, nr;
        bool valid, gfirst;  // gfirst: first chunk of the group's first row
    };
    auto group_of = [&](int64_t pos) -> int64_t { return pp.gorder ? (int64_t)__ldg(pp.gorder + pos) : pos; };
    auto row_start = [&](Cur &c) {
        const int64_t row = c.grp * G + c.t;
        c.k0 = __ldg(rp + row);
        c.e = __ldg(rp + row + 1);
        c.gfirst = (c.t == 0);
    };
    auto advance = [&](Cur &c) {
        if (!c.valid) return;
        if (c.k0 + C::CH < c.e) {
            c.k0 += C::CH;
            c.gfirst = false;
            return;
        }
        if (++c.t >= c.nr) {
            c.pos += nwarps;
            c.t = 0;
            if (c.pos >= ngroups) {
                c.valid = false;
                return;
            }
            c.grp = group_of(c.pos);
            c.nr = (int)(nrows - c.grp * G < (int64_t)G ? nrows - c.grp * G : (int64_t)G);
        }
        row_start(c);
    };
    auto issue = [&](const Cur &c, int s) {
        if (lane == 0 && c.valid) {
            const int64_t ne = (c.e - c.k0 < (int64_t)C::CH ? c.e - c.k0 : (int64_t)C::CH);
            unsigned char *st = wb + s * C::STAGE;
            fence_proxy_async();
            mbar_arrive_expect_tx(&bar[s], (uint32_t)(ne * (8 + Cols::kIdxBytes)));
            if (ne > 0) {
                bulk_g2s(st, v + c.k0, (uint32_t)(ne * 8), &bar[s], pol);
                bulk_g2s(st + C::IDX, cols.stream(c.k0), (uint32_t)(ne * Cols::kIdxBytes), &bar[s], pol);
            }
        }
    };

    double acc = 0.0, acc1 = 0.0, mine = 0.0;
    typename Epi::Acc dacc{};
    typename Epi::Pre pre{};
    uint32_t phase = 0;  // bit s = parity of stage s
    // cur = chunk being reduced; ahead = the last chunk issued (NS−1 chunks in flight ahead of cur)
    Cur cur;
    cur.pos = warp;
    cur.t = 0;
    cur.valid = cur.pos < ngroups;
    if (cur.valid) {
        cur.grp = group_of(cur.pos);
        cur.nr = (int)(nrows - cur.grp * G < (int64_t)G ? nrows - cur.grp * G : (int64_t)G);
        row_start(cur);
    }
    Cur ahead = cur;
    issue(ahead, 0);
    for (int k = 1; k < NS - 1; k++) {
        advance(ahead);
        issue(ahead, k);
    }
    int s = 0;
    bool signalled = pp.gorder == nullptr || pp.nranks == 0;
    if (!signalled && warp < pp.nbnd) peer_wait_warp(pp);  // this warp has boundary groups
    while (cur.valid) {
        advance(ahead);
        issue(ahead, (s + NS - 1) % NS);
        if (!signalled && cur.pos >= pp.nbnd) {  // past this warp's boundary groups
            peer_signal_warp(pp);
            signalled = true;
        }
        if (cur.gfirst && lane < cur.nr) pre = epi.load(cur.grp * G + lane);
        const int rs = cols.row(cur.grp * G + cur.t);
        mbar_wait(&bar[s], (phase >> s) & 1u);
        phase ^= 1u << s;
        const int ne = (int)(cur.e - cur.k0 < (int64_t)C::CH ? cur.e - cur.k0 : (int64_t)C::CH);
        const double *sv = reinterpret_cast<const double *>(wb + s * C::STAGE);
        const unsigned char *sidx = wb + s * C::STAGE + C::IDX;
        double xa[U], xb[U], va[U], vb[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const int ja = lane + 64 * u, jb = ja + 32;
            va[u] = vb[u] = xa[u] = xb[u] = 0.0;
            if (ja < ne) {
                va[u] = sv[ja];
                xa[u] = __ldg(g + cols.staged(sidx, ja, rs));
            }
            if (jb < ne) {
                vb[u] = sv[jb];
                xb[u] = __ldg(g + cols.staged(sidx, jb, rs));
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            acc = fma(va[u], xa[u], acc);
            acc1 = fma(vb[u], xb[u], acc1);
        }
        if (cur.k0 + C::CH >= cur.e) {  // last chunk of the row
            const double sum = warp_sum(acc + acc1);
            acc = 0.0;
            acc1 = 0.0;
            if (lane == cur.t) mine = sum;
            if (cur.t == cur.nr - 1) {  // last row of the group: coalesced epilogue
                if (lane < cur.nr) acc_add(dacc, epi(cur.grp * G + lane, mine, pre));
                mine = 0.0;
            }
        }
        __syncwarp();
        advance(cur);
        s = (s + 1) % NS;
    }
    if (!signalled) peer_signal_warp(pp);
    if constexpr (Epi::kDot) block_dot_finalize_n<kBlockT>(dacc, dc);
    peer_signal(pp);
}

// ------------------------------------------------------------------------------------------------
// The streaming SELL-32 core ("SELL2"): slices of 32 consecutive rows, one row per lane.  Within a
// slice, pair-column k of lane l lives at pair index soff[s] + 32·k + l, so each warp-wide load is a
// contiguous 512-byte value segment + 256-byte column segment.  No shuffles; the epilogue is one
// row per lane (coalesced).  U independent pair loads per lane are in flight per iteration.
// ------------------------------------------------------------------------------------------------
template <class Epi>
__global__ void __launch_bounds__(kBlock) k_sell2(const int64_t *__restrict__ soff, const int2 *__restrict__ ci2,
                                                  const double2 *__restrict__ v2, const double *__restrict__ g,
                                                  int64_t nrows, Epi epi, DotCtx dc, P2P pp) {
    pdl_enter();
    peer_wait(pp);
    constexpr int U = 4;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nslices = (nrows + 31) >> 5;
    const uint64_t pol = stream_policy();
    typename Epi::Acc dacc{};
    for (int64_t sl = warp; sl < nslices; sl += nwarps) {
        const int64_t off = __ldg(soff + sl);
        const int W = (int)((__ldg(soff + sl + 1) - off) >> 5);
        const int64_t row = (sl << 5) + lane;
        typename Epi::Pre pre{};
        if (row < nrows) pre = epi.load(row);
        const double2 *vp = v2 + off + lane;
        const int2 *cp = ci2 + off + lane;
        double acc[U];
#pragma unroll
        for (int u = 0; u < U; u++) acc[u] = 0.0;
        int k = 0;
        for (; k + U <= W; k += U) {
            double2 va[U];
            int2 ca[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                va[u] = ld_stream(vp + (int64_t)(k + u) * 32, pol);
                ca[u] = ld_stream(cp + (int64_t)(k + u) * 32, pol);
            }
#pragma unroll
            for (int u = 0; u < U; u++) {
                acc[u] = fma(va[u].x, __ldg(g + ca[u].x), acc[u]);
                acc[u] = fma(va[u].y, __ldg(g + ca[u].y), acc[u]);
            }
        }
        for (; k < W; k++) {
            const double2 va = ld_stream(vp + (int64_t)k * 32, pol);
            const int2 ca = ld_stream(cp + (int64_t)k * 32, pol);
            acc[0] = fma(va.x, __ldg(g + ca.x), acc[0]);
            acc[0] = fma(va.y, __ldg(g + ca.y), acc[0]);
        }
        if (row < nrows) acc_add(dacc, epi(row, (acc[0] + acc[1]) + (acc[2] + acc[3]), pre));
    }
    if constexpr (Epi::kDot) block_dot_finalize(dacc, dc);
    peer_signal(pp);
}

// ------------------------------------------------------------------------------------------------
// SELL-VI core (layout 2): 32-row slices, ONE ROW PER LANE, one 32-bit word per stored entry = column
// offset from the row's smallest column (low `obits` bits) | index into the operator's distinct-value
// table (CSR-VI above; the high 32 − obits bits).  obits is the operator's: 16 at C3, 18 for the wider
// rows of C4/C5.  Slice s stores W4_s = ⌈(its longest row)/4⌉ columns of 32 quads: quad q of lane t
// holds entries 4q..4q+3 of row 32s+t (padding: offset 0, the index of 0.0), so one 128-bit load per
// lane fetches 4 entries and a warp load is 512 contiguous bytes.
//
// Why row per lane on the IgA operators: lane t and lane t+1 hold rows i and i+1, x-neighbours, so
// entry k of the 32 rows is one stencil position at 32 consecutive columns — the x-gather of one warp
// instruction is 256 contiguous bytes (2–3 L1 wavefronts instead of ≈ 6 for a row per warp), and the
// 32 rows of an interior slice have the SAME value at entry k — the table lookup is one broadcast.
// Together with the 4 B streamed per entry this moves the fine-level operator from 10 B/entry at ≈ 9
// L1 wavefronts per 32 entries (CSR-D16) to 4 B at ≈ 4–5.
//
// Summation order: entry k of a row goes to chain k & 1, each chain accumulates in increasing k, the
// row sum is chain0 + chain1 — independent of U (quads in flight per lane), so every U gives
// bitwise-equal results.  (Not the CSR cores' order: the layout is chosen per operator by a fixed rule at
// setup, never by timing, so results do not depend on the autotuner.)  Slices are visited in the
// boundary-first order of 32-row groups on P2P runs, with the same early publication as k_csr2.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream(const uint4 *p, uint64_t pol) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p), "l"(pol));
    return r;
}
__device__ __forceinline__ unsigned quad_at(const uint4 &q, int j) { return j == 0 ? q.x : j == 1 ? q.y : j == 2 ? q.z : q.w; }
extern __shared__ double sellvi_table[];  // dynamic shared memory of k_sellvi<.., kSmem = true>
template <bool kSmem>
__device__ __forceinline__ double tab_at(const double *t, unsigned i) {
    if constexpr (kSmem) return sellvi_table[i];
    else return ld_gather(t + i);
}

// kSmem: the value table (nvals entries) is first copied into shared memory, where the lookups of one
// warp instruction — a few distinct values, mostly one — take one wavefront instead of ≈ 3 L1 lines.
template <int U, class Epi, bool kSmem>
__global__ void __launch_bounds__(kBlock) k_sellvi(const int64_t *__restrict__ soff, const uint4 *__restrict__ w,
                                                   const int *__restrict__ rbase, const double *__restrict__ gtable,
                                                   int nvals, int obits, const double *__restrict__ g, int64_t nrows,
                                                   Epi epi, DotCtx dc, P2P pp, int64_t nwhole, int lparts,
                                                   double2 *partial, unsigned *sticket) {
    pdl_enter();
    const unsigned omask = (1u << obits) - 1u;
    const double *table = gtable;
    if constexpr (kSmem) {
        for (int i = threadIdx.x; i < nvals; i += blockDim.x) sellvi_table[i] = __ldg(gtable + i);
        __syncthreads();
    }
    if (!pp.gorder) peer_wait(pp);
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * kBlock) >> 5;
    const int64_t nslices = (nrows + 31) >> 5;
    const uint64_t pol = stream_policy();
    typename Epi::Acc dacc{};
    bool signalled = pp.gorder == nullptr || pp.nranks == 0;
    // work items: slice positions [0, nwhole) whole, then every later position split into 2^lparts parts
    const int64_t nitems = nwhole + ((nslices - nwhole) << lparts);
    const int64_t nbnd_items = pp.nbnd <= nwhole ? pp.nbnd : nwhole + ((pp.nbnd - nwhole) << lparts);
    // a warp with boundary ITEMS waits for the neighbours (with split slices there are more boundary
    // items than boundary slice positions: waiting on `warp < nbnd` let the warps in between read
    // ghost values before the neighbours had published them)
    if (!signalled && warp < nbnd_items) peer_wait_warp(pp);
    for (int64_t it = warp; it < nitems; it += nwarps) {
        if (!signalled && it >= nbnd_items) {
            peer_signal_warp(pp);
            signalled = true;
        }
        int64_t pos = it;
        int part = 0, lp = 0;
        if (it >= nwhole) {
            pos = nwhole + ((it - nwhole) >> lparts);
            part = (int)((it - nwhole) & ((1 << lparts) - 1));
            lp = lparts;
        }
        const int parts = 1 << lp;
        const int64_t sl = pp.gorder ? (int64_t)__ldg(pp.gorder + pos) : pos;
        const int64_t off = __ldg(soff + sl);
        const int W4s = (int)(__ldg(soff + sl + 1) - off);
        // this item's quads [q0, q0 + W4) of the slice (the whole slice when parts == 1)
        const int q0 = (int)(((int64_t)W4s * part) >> lp);
        const int W4 = (int)(((int64_t)W4s * (part + 1)) >> lp) - q0;
        const int64_t row = (sl << 5) + lane;
        typename Epi::Pre pre{};
        int b = 0;
        if (row < nrows) {
            b = __ldg(rbase + row);
            if (parts == 1) pre = epi.load(row);
        }
        const uint4 *wp = w + ((off + q0) << 5) + lane;
        double s0 = 0.0, s1 = 0.0;
        int q = 0;
        // software pipeline: the next batch's words are requested before this batch's gathers, so the
        // HBM stream never waits behind the (L1/L2) gathers
        uint4 wa[U], wn[U];
        if (U <= W4) {
#pragma unroll
            for (int u = 0; u < U; u++) wa[u] = ld_stream(wp + (int64_t)u * 32, pol);
        }
        for (; q + U <= W4; q += U) {
            const bool more = q + 2 * U <= W4;
            if (more) {
#pragma unroll
                for (int u = 0; u < U; u++) wn[u] = ld_stream(wp + (int64_t)(q + U + u) * 32, pol);
            }
            double va[4 * U], xa[4 * U];
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    AMG_DCHECK((int)(quad_at(wa[u], j) >> obits) < nvals);
                    va[4 * u + j] = tab_at<kSmem>(table, quad_at(wa[u], j) >> obits);
                }
#pragma unroll
            for (int u = 0; u < U; u++)
#pragma unroll
                for (int j = 0; j < 4; j++) xa[4 * u + j] = ld_gather(g + (b + (int)(quad_at(wa[u], j) & omask)));
#pragma unroll
            for (int u = 0; u < 4 * U; u += 2) {
                s0 = fma(va[u], xa[u], s0);
                s1 = fma(va[u + 1], xa[u + 1], s1);
            }
            if (more) {
#pragma unroll
                for (int u = 0; u < U; u++) wa[u] = wn[u];
            }
        }
        for (; q < W4; q++) {
            const uint4 wq = ld_stream(wp + (int64_t)q * 32, pol);
            double va[4], xa[4];
#pragma unroll
            for (int j = 0; j < 4; j++) va[j] = tab_at<kSmem>(table, quad_at(wq, j) >> obits);
#pragma unroll
            for (int j = 0; j < 4; j++) xa[j] = ld_gather(g + (b + (int)(quad_at(wq, j) & omask)));
            s0 = fma(va[0], xa[0], s0);
            s1 = fma(va[1], xa[1], s1);
            s0 = fma(va[2], xa[2], s0);
            s1 = fma(va[3], xa[3], s1);
        }
        if (parts == 1) {
            if (row < nrows) acc_add(dacc, epi(row, s0 + s1, pre));
            continue;
        }
        // split slice: deposit this part's two chains; the warp completing the slice's last part sums
        // the parts' chains in part order (fixed, whichever warp arrives last) and runs the epilogue
        const int64_t npad = nslices << 5;
        AMG_DCHECK(part >= 0 && part < parts && q0 + W4 <= W4s);
        __stcg(partial + (int64_t)part * npad + row, make_double2(s0, s1));
        __threadfence();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) {
            const unsigned tk = atomicAdd(sticket + sl, 1u);
            AMG_DCHECK(tk < (unsigned)parts);  // a ticket left over from an earlier launch would show here
            last = tk == (unsigned)(parts - 1);
        }
        last = __shfl_sync(0xffffffffu, last, 0);
        if (!last) continue;
        __threadfence();
        double c0 = 0.0, c1 = 0.0;
        for (int j = 0; j < parts; j++) {
            const double2 v = __ldcg(partial + (int64_t)j * npad + row);
            c0 += v.x;
            c1 += v.y;
        }
        if (lane == 0) sticket[sl] = 0u;  // every part has arrived: reset for the next launch
        if (row < nrows) {
            pre = epi.load(row);
            acc_add(dacc, epi(row, c0 + c1, pre));
        }
    }
    if (!signalled) peer_signal_warp(pp);
    if constexpr (Epi::kDot) block_dot_finalize(dacc, dc);
    peer_signal(pp);
}

// ------------------------------------------------------------------------------------------------
// The windowed SELL-VI core k_sellviw: the gathered vector staged in shared memory by TMA.
// ------------------------------------------------------------------------------------------------
// k_sellvi is bound by the L1 data pipe, not by HBM (ncu, C3 level 0: 78-82 % of the LSU wavefronts,
// 64 % of DRAM): a warp's x-gather of 32 consecutive doubles at an arbitrary offset costs ≈ 2.9 L1
// wavefronts (3 lines) plus tag work, the table lookup ≈ 1.6 and the word stream 1 per 32 entries.
// Here a CTA's 8 warps take 8 CONSECUTIVE slices (a block of 256 rows) and the union of the columns
// those rows touch — a few contiguous runs: for the 3-D stencil one run per z-offset, (rows + 2·p·m_x·
// (m_y+1)) doubles — is copied into shared memory with cp.async.bulk (one bulk copy per run, completion
// on an mbarrier) before the warps need it.  Each entry's word holds the POSITION of its column in the
// staged window (pbits bits) instead of an offset from a row base, so the gather is one ld.shared of
// 32 consecutive doubles: 2 wavefronts, conflict-free, no tag lookups, no L2 round trip on the
// critical path.  NBUF = 2 stages block b+1's window while block b is computed (the copies of the
// next block are issued at the top of the iteration, after the barrier that retired its buffer);
// NBUF = 1 issues them after that barrier and relies on the other resident CTAs to cover the latency.
// Block layout (host, device.cu upload_sellvi): binfo[b] = {first run, end run, window doubles, -};
// runs[r] = {first column, doubles (even), window offset (even), -}; columns and lengths are even so
// every copy is 16-B aligned (the vector must be 16-B aligned: single-GPU layout).  Summation order
// is k_sellvi's (chain k & 1 per entry k of a row), so results are bitwise those of k_sellvi on
// whole (unsplit) slices.
// Tail: the blocks of the last round (positions >= nwhole, counted against the nominal 3·n_SM CTAs so
// the choice depends on the operator alone) are split into 2^wl work items of 8 >> wl consecutive
// slices each; the item's CTA stages the block's whole window and its first 8 >> wl warps take one
// slice each.  Slices stay whole, so the split changes timing, never results.
template <int U, class Epi, int NBUF, bool kSmem>
__global__ void __launch_bounds__(kBlock) k_sellviw(const int64_t *__restrict__ soff, const uint4 *__restrict__ w,
                                                    const int4 *__restrict__ binfo, const int4 *__restrict__ runs,
                                                    const double *__restrict__ gtable, int nvals, int pbits, int wmax,
                                                    const double *__restrict__ g, int64_t nrows, Epi epi, DotCtx dc,
                                                    int64_t nwhole, int wl, P2P pp) {
    pdl_enter();
    constexpr int WPB = kBlock / 32;  // warps per CTA = slices per block
    extern __shared__ __align__(16) double wsm[];
    __shared__ __align__(8) uint64_t bar[NBUF];
    const int tabn = kSmem ? ((nvals + 1) & ~1) : 0;
    double *tab = wsm;
    double *xw = wsm + tabn;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t nslices = (nrows + 31) >> 5;
    const int64_t nblk = (nslices + WPB - 1) / WPB;
    const unsigned pmask = (1u << pbits) - 1u;
    const uint64_t pol = stream_policy();
    if (threadIdx.x == 0) {
        for (int k = 0; k < NBUF; k++) mbar_init(&bar[k], 1);
        fence_mbar_init();
    }
    if constexpr (kSmem) {
        for (int i = threadIdx.x; i < nvals; i += blockDim.x) tab[i] = __ldg(gtable + i);
    }
    __syncthreads();
    const double *table = kSmem ? tab : gtable;
    // P2P (multi-GPU shares): without a block order every CTA waits for the neighbours at its start
    // and the kernel publishes at its end; with one (pp.gorder: the block positions of BOUNDARY blocks
    // — a row reads a ghost value or pushes one — first, pp.nbnd of them) warp 0 waits only before
    // staging a boundary block's window, and each CTA checks in once it is past its boundary items;
    // the last CTA to check in publishes the new count while the interior items still run
    if (!pp.gorder) peer_wait(pp);
    bool signalled = pp.gorder == nullptr || pp.nranks == 0;
    const int64_t nbnd_pos = pp.gorder ? pp.nbnd : 0;  // boundary block POSITIONS
    auto blk_at = [&](int64_t pos) { return pp.gorder ? (int64_t)__ldg(pp.gorder + pos) : pos; };
    bool waited = signalled, cwaited = signalled;
    // warp 0 stages the block at position `pos` into buffer `buf`: lane 0 arms the barrier with the
    // window's bytes, then the lanes issue one bulk copy per run
    auto stage = [&](int64_t pos, int buf) {
        if (!waited && pos < nbnd_pos) {  // ghost values are read by the copies below
            peer_wait_warp(pp);
            waited = true;
        }
        const int4 bi = __ldg(binfo + blk_at(pos));
        if (lane == 0) mbar_arrive_expect_tx(&bar[buf], (uint32_t)bi.z * 8u);
        __syncwarp();
        AMG_DCHECK(bi.x <= bi.y && bi.z >= 0 && bi.z <= wmax);
        for (int r = bi.x + lane; r < bi.y; r += 32) {
            const int4 ru = __ldg(runs + r);
            AMG_DCHECK(ru.y > 0 && (ru.x & 1) == 0 && (ru.y & 1) == 0 && (ru.z & 1) == 0 && ru.z + ru.y <= bi.z);
            bulk_g2s(xw + (int64_t)buf * wmax + ru.z, g + ru.x, (uint32_t)ru.y * 8u, &bar[buf], keep_policy());
        }
    };
    typename Epi::Acc dacc{};
    const int64_t nitems = nwhole + ((nblk - nwhole) << wl);
    auto block_of = [&](int64_t item) { return item < nwhole ? item : nwhole + ((item - nwhole) >> wl); };
    int64_t item = blockIdx.x;
    if (wib == 0 && item < nitems) stage(block_of(item), 0);
    const int64_t nbnd_items = nbnd_pos <= nwhole ? nbnd_pos : nwhole + ((nbnd_pos - nwhole) << wl);
    for (int it = 0; item < nitems; item += gridDim.x, it++) {
        if (!signalled && item >= nbnd_items) {  // past this CTA's boundary items (all their pushes issued)
            peer_signal_cta(pp);
            signalled = true;
        }
        const int buf = NBUF == 2 ? (it & 1) : 0;
        if (NBUF == 2 && wib == 0 && item + gridDim.x < nitems) stage(block_of(item + gridDim.x), buf ^ 1);
        const int64_t blk = blk_at(block_of(item));
        // this item's slices: the whole block, or part (item − nwhole) mod 2^wl of WPB >> wl slices
        const int per = item < nwhole ? WPB : WPB >> wl;
        const int first = item < nwhole ? 0 : (int)((item - nwhole) & ((1 << wl) - 1)) * per;
        const int64_t sl = wib < per ? blk * WPB + first + wib : nslices;  // warps beyond `per` idle
        const int64_t row = (sl << 5) + lane;
        typename Epi::Pre pre{};
        if (sl < nslices && row < nrows) pre = epi.load(row);  // epilogue inputs in flight with the stream
        mbar_wait(&bar[buf], (uint32_t)((it / NBUF) & 1));
        if (!cwaited && item < nbnd_items) {  // every warp acquires the neighbours' flags itself before
            peer_wait_warp(pp);               // its first boundary item (its pushes overwrite ghost slots)
            cwaited = true;
        }
        if (sl < nslices) {
            const double *xb = xw + (int64_t)buf * wmax;
#ifdef AMG_CHECKS
            const int wlen = __ldg(binfo + blk).z;  // the staged window of this block
#endif
            const int64_t off = __ldg(soff + sl);
            const int W4 = (int)(__ldg(soff + sl + 1) - off);
            const uint4 *wp = w + (off << 5) + lane;
            double s0 = 0.0, s1 = 0.0;
            int q = 0;
            uint4 wa[U], wn[U];
            if (U <= W4) {
#pragma unroll
                for (int u = 0; u < U; u++) wa[u] = ld_stream(wp + (int64_t)u * 32, pol);
            }
            for (; q + U <= W4; q += U) {
                const bool more = q + 2 * U <= W4;
                if (more) {
#pragma unroll
                    for (int u = 0; u < U; u++) wn[u] = ld_stream(wp + (int64_t)(q + U + u) * 32, pol);
                }
                double va[4 * U], xa[4 * U];
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int j = 0; j < 4; j++) {
                        AMG_DCHECK((int)(quad_at(wa[u], j) >> pbits) < nvals && (int)(quad_at(wa[u], j) & pmask) < wlen);
                        va[4 * u + j] = tab_at<kSmem>(table, quad_at(wa[u], j) >> pbits);
                    }
#pragma unroll
                for (int u = 0; u < U; u++)
#pragma unroll
                    for (int j = 0; j < 4; j++) xa[4 * u + j] = xb[quad_at(wa[u], j) & pmask];
#pragma unroll
                for (int u = 0; u < 4 * U; u += 2) {
                    s0 = fma(va[u], xa[u], s0);
                    s1 = fma(va[u + 1], xa[u + 1], s1);
                }
                if (more) {
#pragma unroll
                    for (int u = 0; u < U; u++) wa[u] = wn[u];
                }
            }
            for (; q < W4; q++) {
                const uint4 wq = ld_stream(wp + (int64_t)q * 32, pol);
                double va[4], xa[4];
#pragma unroll
                for (int j = 0; j < 4; j++) {
                    AMG_DCHECK((int)(quad_at(wq, j) >> pbits) < nvals && (int)(quad_at(wq, j) & pmask) < wlen);
                    va[j] = tab_at<kSmem>(table, quad_at(wq, j) >> pbits);
                }
#pragma unroll
                for (int j = 0; j < 4; j++) xa[j] = xb[quad_at(wq, j) & pmask];
                s0 = fma(va[0], xa[0], s0);
                s1 = fma(va[1], xa[1], s1);
                s0 = fma(va[2], xa[2], s0);
                s1 = fma(va[3], xa[3], s1);
            }
            if (row < nrows) acc_add(dacc, epi(row, s0 + s1, pre));
        }
        __syncthreads();  // every warp is done with `buf`: it may be refilled
        if (NBUF == 1 && wib == 0 && item + gridDim.x < nitems) {
            fence_proxy_async();
            stage(block_of(item + gridDim.x), 0);
        }
    }
    if (!signalled) peer_signal_cta(pp);
    if constexpr (Epi::kDot) block_dot_finalize(dacc, dc);
    peer_signal(pp);
}

// Non-template kernels are defined in device.cu only (AMGB_PLAIN_KERNELS); the inst_*.cu units see
// just the templated streaming cores above.
#ifdef AMGB_PLAIN_KERNELS
// ------------------------------------------------------------------------------------------------
// Elementwise / reduction kernels (grid-stride, fused)
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kBlock) k_cheb_first(int64_t n, const double *__restrict__ b,
                                                        const double *__restrict__ invd, double *__restrict__ d0,
                                                        double c0, Push push, P2P pp) {
    pdl_enter();
    peer_wait(pp);
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double d = c0 * (b[i] * invd[i]);
        d0[i] = d;
        push.put(i, d);
    }
    peer_signal(pp);
}

// y = x (owned rows) and the ghost push of y (P2P: the initial residual's copy of u)
__global__ void __launch_bounds__(kBlock) k_copy_push(int64_t n, const double *__restrict__ x, double *__restrict__ y,
                                                       Push push, P2P pp) {
    pdl_enter();
    peer_wait(pp);
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double v = x[i];
        y[i] = v;
        push.put(i, v);
    }
    peer_signal(pp);
}

// P2P all-reduce of one dot product: every rank deposited its sum in dslot[kind][q] of every rank
// (block_dot_finalize); each rank adds them in rank order (identical on every rank).
__global__ void k_dot_collect(int kind, int kind2, Scalars *S, P2P pp) {
    pdl_enter();
    peer_wait(pp);
    if (threadIdx.x == 0) {
        const int kinds[2] = {kind, kind2};
        for (int k = 0; k < 2; k++) {
            if (kinds[k] == DOT_NONE) continue;
            const double *slot = reinterpret_cast<const double *>(pp.base[pp.rank] + pp.dslot_off) + kinds[k] * pp.nranks;
            double s = 0.0;
            for (int q = 0; q < pp.nranks; q++) s += *(volatile const double *)(slot + q);
            *scalar_slot(S, kinds[k]) = s;
        }
    }
    peer_signal(pp);
}

// autotuning scratch: a smooth positive pattern
__global__ void __launch_bounds__(kBlock) k_fill_pattern(int64_t n, double *__restrict__ x) {
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        x[i] = 1.0 + 1e-3 * (double)(i % 97);
}

__global__ void __launch_bounds__(kBlock) k_axpy1(int64_t n, const double *__restrict__ d, double *__restrict__ x) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        x[i] = x[i] + d[i];
}

// dot(a, b) -> scalar of kind dc.kind
__global__ void __launch_bounds__(kBlock) k_dot(int64_t n, const double *__restrict__ a, const double *__restrict__ b,
                                                 DotCtx dc) {
    pdl_enter();
    peer_wait(dc.pp);
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        s += a[i] * b[i];
    block_dot_finalize(s, dc);
    peer_signal(dc.pp);
}

// a2: u += α p; r −= α q; ‖r‖² with α = ρ/pᵀq from the (all-reduced) device scalars
__global__ void __launch_bounds__(kBlock) k_pcg_update(int64_t n, const double *__restrict__ p,
                                                        const double *__restrict__ q, double *__restrict__ u,
                                                        double *__restrict__ r, DotCtx dc, int flex) {
    pdl_enter();
    peer_wait(dc.pp);
    const double alpha = (flex ? dc.S->pr : dc.S->rz) / dc.S->pq;  // FCG: pᵀr / pᵀq; CG: ρ / pᵀq
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        u[i] = u[i] + alpha * p[i];
        const double ri = r[i] - alpha * q[i];
        r[i] = ri;
        s += ri * ri;
    }
    block_dot_finalize(s, dc);
    peer_signal(dc.pp);
}

// a11: p = z + β p  (first iteration: p = z)
__global__ void __launch_bounds__(kBlock) k_p_update(int64_t n, const double *__restrict__ z, double *__restrict__ p,
                                                      const Scalars *__restrict__ S, int first_, int flex, Push push,
                                                      P2P pp, const LoopCtl *__restrict__ ctl) {
    pdl_enter();
    peer_wait(pp);
    const int first = ctl ? ctl->first : first_;  // device loop: the first iteration is decided on the device
    // CG: β = ρ/ρ_prev; FCG(1): β = −zᵀq_prev / pᵀq_prev (S->pq still holds the previous iteration's)
    const double beta = first ? 0.0 : flex ? -S->zq / S->pq : S->rz / S->rz_prev;
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock) {
        const double v = first ? z[i] : z[i] + beta * p[i];
        p[i] = v;
        push.put(i, v);
    }
    peer_signal(pp);
}

// end of a PCG iteration: ρ_prev <- ρ (one thread; after every consumer of ρ in this iteration)
__global__ void k_roll_rho(Scalars *S) {
    pdl_enter();
    S->rz_prev = S->rz;
}

// Device loop control, after iteration k's ‖r‖² (c.19 stopping test, as the host loop takes it):
// breakdown (CG: rᵀz <= 0; pᵀKp <= 0), ‖r_k‖ <= rtol·‖F‖, or k == maxit end the WHILE loop.  Every
// rank holds the same all-reduced scalars, so every rank takes the same decision.
__global__ void k_loop_ctl(const Scalars *__restrict__ S, LoopCtl *__restrict__ c, int flex,
                           cudaGraphConditionalHandle h) {
    pdl_enter();
    const int k = c->k + 1;
    c->k = k;
    c->first = 0;
    unsigned go = 1;
    if ((!flex && !(S->rz > 0.0)) || !(S->pq > 0.0)) {
        c->status = -5;
        go = 0;
    } else {
        const double rn = sqrt(S->rr);
        c->hist[k] = rn / c->nF;
        if (rn <= c->thr) {
            c->status = 0;
            go = 0;
        } else if (k >= c->maxit) {
            c->status = 1;
            go = 0;
        }
    }
    cudaGraphSetConditional(h, go);
}

// gather/scatter helpers of the multi-GPU path
__global__ void __launch_bounds__(kBlock) k_pack(int64_t n, const int *__restrict__ idx, const double *__restrict__ x,
                                                  double *__restrict__ buf) {
    pdl_enter();
    for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += (int64_t)gridDim.x * kBlock)
        buf[i] = x[idx[i]];
}
// recv (nranks x stride) -> full[bounds[q] + i] for i < bounds[q+1]-bounds[q]
__global__ void __launch_bounds__(kBlock) k_unpack_allgather(int nranks, int64_t stride,
                                                              const int64_t *__restrict__ bounds,
                                                              const double *__restrict__ recv,
                                                              double *__restrict__ full) {
    pdl_enter();
    for (int q = 0; q < nranks; q++) {
        const int64_t b = bounds[q], c = bounds[q + 1] - b;
        for (int64_t i = (int64_t)blockIdx.x * kBlock + threadIdx.x; i < c; i += (int64_t)gridDim.x * kBlock)
            full[b + i] = recv[q * stride + i];
    }
}

// a7: coarsest level, `sweeps` ℓ1-Jacobi sweeps from x = 0 in ONE CTA (the coarsest level has ≤ 50
// rows at the default coarse size): the operator (when it fits), b, invd and the double-buffered x live
// in shared memory; warp w reduces rows w, w+32, … with its lanes striding over the row (shuffle tree),
// and a __syncthreads separates the sweeps.
__global__ void __launch_bounds__(1024) k_coarse_solve(int n, const int64_t *__restrict__ rp,
                                                        const int *__restrict__ ci, const double *__restrict__ v,
                                                        const double *__restrict__ invd, const double *__restrict__ b,
                                                        double *__restrict__ x, int sweeps, int staged, P2P pp) {
    pdl_enter();
    peer_wait(pp);
    extern __shared__ double sm[];
    double *xa = sm, *xb = sm + n, *sb = sm + 2 * n, *sd = sm + 3 * n;
    const int nnz = (int)rp[n];
    double *sv = sm + 4 * n;
    int *sc = reinterpret_cast<int *>(sv + (staged ? nnz : 0));
    int *srp = sc + (staged ? nnz : 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        xa[i] = 0.0;
        sb[i] = b[i];
        sd[i] = invd[i];
    }
    if (staged) {
        for (int k = threadIdx.x; k < nnz; k += blockDim.x) {
            sv[k] = v[k];
            sc[k] = ci[k];
        }
        for (int i = threadIdx.x; i <= n; i += blockDim.x) srp[i] = (int)rp[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int s = 0; s < sweeps; s++) {
        for (int i = wid; i < n; i += nw) {
            double t = 0.0;
            if (staged) {
                for (int k = srp[i] + lane; k < srp[i + 1]; k += 32) t = fma(sv[k], xa[sc[k]], t);
            } else {
                for (int64_t k = rp[i] + lane; k < rp[i + 1]; k += 32) t = fma(v[k], xa[ci[k]], t);
            }
            t = warp_sum(t);
            if (lane == 0) xb[i] = xa[i] + (sb[i] - t) * sd[i];
        }
        __syncthreads();
        double *tmp = xa;
        xa = xb;
        xb = tmp;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = xa[i];
    peer_signal(pp);
}

// Deterministic CTA-wide sum (fixed shuffle tree + fixed warp order); every thread gets the result.
__device__ __forceinline__ double cta_sum(double v, double *red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();  // red is reused
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; w++) s += red[w];
    return s;
}

// a7, §5.1 variant: the coarsest level solved by CG preconditioned by one weighted-Jacobi
// sweep (z = D⁻¹ r with D = diag(K_L); the weight does not change CG) from x = 0 until
// ‖r‖₂ <= tol·‖b‖₂ or maxit iterations, in ONE CTA: the operator (when it fits), x, r, z, p, q and
// D in shared memory, warp-per-row products, deterministic CTA reductions.
__global__ void __launch_bounds__(1024) k_coarse_cg(int n, const int64_t *__restrict__ rp, const int *__restrict__ ci,
                                                     const double *__restrict__ v, const double *__restrict__ diag,
                                                     const double *__restrict__ b, double *__restrict__ x, double tol,
                                                     int maxit, int staged, P2P pp) {
    pdl_enter();
    peer_wait(pp);
    extern __shared__ double sm[];
    __shared__ double red[32];
    double *sx = sm, *sr = sm + n, *sz = sm + 2 * n, *sp = sm + 3 * n, *sq = sm + 4 * n, *sd = sm + 5 * n;
    const int nnz = (int)rp[n];
    double *sv = sm + 6 * n;
    int *sc = reinterpret_cast<int *>(sv + (staged ? nnz : 0));
    int *srp = sc + (staged ? nnz : 0);
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        sx[i] = 0.0;
        sr[i] = b[i];
        sd[i] = diag[i];
    }
    if (staged) {
        for (int k = threadIdx.x; k < nnz; k += blockDim.x) {
            sv[k] = v[k];
            sc[k] = ci[k];
        }
        for (int i = threadIdx.x; i <= n; i += blockDim.x) srp[i] = (int)rp[i];
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double loc = 0.0;
    for (int i = threadIdx.x; i < n; i += blockDim.x) loc += sr[i] * sr[i];
    const double bn = sqrt(cta_sum(loc, red));
    if (bn > 0.0) {
        loc = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            sz[i] = sr[i] / sd[i];
            sp[i] = sz[i];
            loc += sr[i] * sz[i];
        }
        double rz = cta_sum(loc, red);
        for (int it = 0; it < maxit; it++) {
            for (int i = wid; i < n; i += nw) {  // q = K p
                double t = 0.0;
                if (staged) {
                    for (int k = srp[i] + lane; k < srp[i + 1]; k += 32) t = fma(sv[k], sp[sc[k]], t);
                } else {
                    for (int64_t k = rp[i] + lane; k < rp[i + 1]; k += 32) t = fma(v[k], sp[ci[k]], t);
                }
                t = warp_sum(t);
                if (lane == 0) sq[i] = t;
            }
            __syncthreads();
            loc = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) loc += sp[i] * sq[i];
            const double pq = cta_sum(loc, red);
            if (!(pq > 0.0)) break;
            const double alpha = rz / pq;
            loc = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                sx[i] = sx[i] + alpha * sp[i];
                sr[i] = sr[i] - alpha * sq[i];
                loc += sr[i] * sr[i];
            }
            if (sqrt(cta_sum(loc, red)) <= tol * bn) break;
            loc = 0.0;
            for (int i = threadIdx.x; i < n; i += blockDim.x) {
                sz[i] = sr[i] / sd[i];
                loc += sr[i] * sz[i];
            }
            const double rz_new = cta_sum(loc, red);
            const double beta = rz_new / rz;
            for (int i = threadIdx.x; i < n; i += blockDim.x) sp[i] = sz[i] + beta * sp[i];
            rz = rz_new;
            __syncthreads();
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = sx[i];
    peer_signal(pp);
}

#endif  // AMGB_PLAIN_KERNELS

}  // namespace dev
}  // namespace amgb
