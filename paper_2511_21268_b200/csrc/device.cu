// device.cu — device runtime of the solve phase: level storage in HBM, the V-cycle (c.18) and PCG
// (c.19) as a fixed sequence of fused streaming kernels (kernels.cuh), and the C-ABI entry points
// that need the GPU.
//
// Everything is device-resident after amg_setup: per iteration the host only enqueues kernels and
// reads back one 64-byte scalar block (‖r‖² and breakdown flags) for the convergence test.
#include <cuda_runtime.h>
#include <nccl.h>

#include <omp.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <cmath>
#include <string>
#include <vector>

#define AMGB_PLAIN_KERNELS
#include "devstate.cuh"

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

void *DevState::alloc(size_t bytes) {
    void *p = nullptr;
    // 256-B units: vectors may be read (never written) up to the next 16-B boundary past their end
    // by the window copies of k_sellviw
    bytes = (std::max<size_t>(bytes, 16) + 255) & ~(size_t)255;
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

DevState::~DevState() {
    for (auto &b : bufs) {
        if (g_free) g_free(b.p, b.bytes, device, nullptr);
        else cudaFree(b.p);
    }
    for (auto e : ev) cudaEventDestroy(e);
    if (hS) cudaFreeHost(hS);
    for (auto &s : seg)
        if (s.exec) cudaGraphExecDestroy(s.exec);
    if (loop.exec) cudaGraphExecDestroy(loop.exec);
    if (hctl) cudaFreeHost(hctl);
    if (cap) cudaStreamDestroy(cap);
    for (char *p : peer_slabs) cudaIpcCloseMemHandle(p);
    if (slab) {
        // no rank may still store into this slab: barrier over the communicator before freeing it
        if (comm) {
            int64_t *one = nullptr;
            if (cudaMalloc(&one, sizeof(int64_t)) == cudaSuccess) {
                if (ncclAllReduce(one, one, 1, ncclInt64, ncclSum, comm, nullptr) == ncclSuccess)
                    cudaStreamSynchronize(nullptr);
                cudaFree(one);
            }
        }
        cudaFree(slab);
    }
    if (comm) ncclCommDestroy(comm);
}

namespace {

// Rows per warp group: enough groups to give every SM ~64 warps of work, coalesced epilogues where
// possible.  Instantiated: 1, 4, 8, 32.  Env AMG_CSR_G overrides (experiments).
int choose_G(int64_t nrows) {
    if (const char *e = std::getenv("AMG_CSR_G")) return std::atoi(e);
    const int64_t target = nrows / (148 * 64);
    return target >= 32 ? 32 : target >= 8 ? 8 : target >= 4 ? 4 : 1;
}

// Pair loads per lane in flight: enough to cover the longest row in one round trip (max 8).
// Instantiated: 2, 4, 6, 8.  Env AMG_CSR_U overrides (experiments).
int choose_U(const HCsr &A) {
    if (const char *e = std::getenv("AMG_CSR_U")) return std::atoi(e);
    int64_t maxlen = 0;
    for (int64_t i = 0; i < A.nrows; i++) maxlen = std::max(maxlen, A.rp[i + 1] - A.rp[i]);
    const int64_t pairs_per_lane = ((maxlen + 1) / 2 + 31) / 32;
    return pairs_per_lane <= 2 ? 2 : pairs_per_lane <= 4 ? 4 : pairs_per_lane <= 6 ? 6 : 8;
}

// Pad column of row i: the diagonal for square operators, else the row's first column.
inline int32_t pad_col(const HCsr &A, int64_t i, bool square) {
    if (square) return (int32_t)i;
    return A.rp[i + 1] > A.rp[i] ? A.ci[A.rp[i]] : 0;
}

bool encode_d16(DevState &D, const int64_t *rp, const int32_t *ci, int64_t nrows, DCsr &out, Buf<uint16_t> *keep);
void encode_values(DevState &D, const double *v, int64_t stored, const uint16_t *off, DCsr &out);

// Upload a host CSR as CSR2 (rows padded to a multiple of `mult` entries with (pad column, 0.0);
// mult = 2 for format 1, 8 for the autotuned layouts: the TMA-staged core's bulk copies need 16-byte
// aligned value, int32 and 16-bit column ranges).
void upload_csr2(DevState &D, const HCsr &A, DCsr &out, bool square, int mult = 2) {
    const int64_t n = A.nrows;
    Buf<int64_t> rp(n + 1);
    rp[0] = 0;
    for (int64_t i = 0; i < n; i++) {
        int64_t len = A.rp[i + 1] - A.rp[i];
        rp[i + 1] = rp[i] + (len + mult - 1) / mult * mult;
    }
    const int64_t nnz2 = rp[n];
    Buf<int32_t> ci(nnz2);
    Buf<double> v(nnz2);
    int32_t maxc = 0;
    for (int64_t k = 0; k < A.nnz(); k++) maxc = std::max(maxc, A.ci[k]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        int64_t o = rp[i];
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; k++, o++) {
            ci[o] = A.ci[k];
            v[o] = A.v[k];
        }
        // padding continues the row's last run of columns where possible (stays inside the row's
        // column window and below the largest column present, so inside every gathered vector's
        // owned + ghost extent); the padded products are 0.0·x[col] for a valid column
        const bool has = A.rp[i + 1] > A.rp[i];
        const int32_t last = has ? A.ci[A.rp[i + 1] - 1] : 0;
        for (int32_t t = 1; o < rp[i + 1]; o++, t++) {
            const int64_t c = (int64_t)last + t;
            ci[o] = (has && c <= maxc) ? (int32_t)c : pad_col(A, i, square);
            v[o] = 0.0;
        }
    }
    out.fmt = 0;
    out.mult = mult;
    out.stored = nnz2;
    out.rp = D.alloc_n<int64_t>(n + 1);
    out.ci = D.alloc_n<int32_t>(nnz2);
    out.v = D.alloc_n<double>(nnz2);
    out.G = choose_G(n);
    out.U = choose_U(A);
    CUDA_OK(cudaMemcpy(out.rp, rp.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.ci, ci.data(), sizeof(int32_t) * nnz2, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.v, v.data(), sizeof(double) * nnz2, cudaMemcpyHostToDevice));
    if (mult >= 4) {
        Buf<uint16_t> off;
        const bool d16 = encode_d16(D, rp.data(), ci.data(), n, out, &off);
        if (mult >= 8) encode_values(D, v.data(), nnz2, d16 ? off.data() : nullptr, out);
    }
}

// Open-addressing map of fp64 bit patterns -> uint64 (value dictionary of encode_values).
struct BitsTable {
    static constexpr uint64_t kEmpty = ~0ull;  // a NaN pattern: never a stored value (checked)
    std::vector<uint64_t> key, val;
    uint64_t mask = 0;
    int64_t count = 0;
    explicit BitsTable(int64_t cap) {
        uint64_t sz = 16;
        while (sz < (uint64_t)cap * 2) sz <<= 1;
        key.assign(sz, kEmpty);
        val.assign(sz, 0);
        mask = sz - 1;
    }
    static uint64_t hash(uint64_t x) {
        x ^= x >> 31;
        x *= 0x7fb5d329728ea185ull;
        x ^= x >> 27;
        x *= 0x81dadef4bc2dd44dull;
        return x ^ (x >> 33);
    }
    // slot of x, inserted (value 0) if absent; the table must keep a free slot
    uint64_t insert(uint64_t x) {
        uint64_t h = hash(x) & mask;
        while (key[h] != kEmpty && key[h] != x) h = (h + 1) & mask;
        if (key[h] == kEmpty) {
            key[h] = x;
            count++;
        }
        return h;
    }
    uint64_t find(uint64_t x) const {
        uint64_t h = hash(x) & mask;
        while (key[h] != x) h = (h + 1) & mask;
        return h;
    }
};

// Distinct-value dictionary of n fp64 values (plus +0.0 when with_zero: the padding value): the
// distinct bit patterns ordered by decreasing frequency (ties: ascending bit pattern) into `tab`, and
// each value's index into idx[0..n).  Frequency order puts the values of the interior stencil — most
// of the entries — at the head of the table, so one warp's lookups touch few L1 lines.  Returns false
// (nothing built) if there are more than `cap` distinct values.  Parallel: per-thread count maps, merged.
bool value_dictionary(const double *v, int64_t n, bool with_zero, int64_t cap, std::vector<double> &tab,
                      Buf<uint32_t> &idx) {
    const int nt = omp_get_max_threads();
    std::vector<std::vector<std::pair<uint64_t, uint64_t>>> loc(nt);
    bool ok = true;
#pragma omp parallel num_threads(nt) reduction(&& : ok)
    {
        const int t = omp_get_thread_num(), T = omp_get_num_threads();
        const int64_t k0 = n * t / T, k1 = n * (t + 1) / T;
        BitsTable m(std::min<int64_t>(cap, 1 << 12));
        for (int64_t k = k0; k < k1; k++) {
            uint64_t x;
            std::memcpy(&x, v + k, 8);
            if (x == BitsTable::kEmpty || m.count > cap) { ok = false; break; }
            m.val[m.insert(x)]++;
            if (m.count * 2 > (int64_t)m.key.size()) {  // grow: load factor <= 1/2
                BitsTable big(m.count * 2);
                for (size_t h = 0; h < m.key.size(); h++)
                    if (m.key[h] != BitsTable::kEmpty) big.val[big.insert(m.key[h])] = m.val[h];
                m = std::move(big);
            }
        }
        if (ok)
            for (size_t h = 0; h < m.key.size(); h++)
                if (m.key[h] != BitsTable::kEmpty) loc[t].push_back({m.key[h], m.val[h]});
    }
    if (!ok) return false;
    std::vector<std::pair<uint64_t, uint64_t>> all;  // (bits, count)
    if (with_zero) all.push_back({0ull, 0ull});
    for (auto &l : loc) all.insert(all.end(), l.begin(), l.end());
    std::sort(all.begin(), all.end());
    size_t w = 0;
    for (size_t i = 0; i < all.size(); i++) {
        if (w > 0 && all[w - 1].first == all[i].first) all[w - 1].second += all[i].second;
        else all[w++] = all[i];
    }
    all.resize(w);
    const int64_t nv = (int64_t)all.size();
    if (nv > cap) return false;
    std::stable_sort(all.begin(), all.end(), [](const auto &a, const auto &b) { return a.second > b.second; });
    BitsTable map(nv);
    for (int64_t i = 0; i < nv; i++) map.val[map.insert(all[i].first)] = (uint64_t)i;
    idx.alloc(n);
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; k++) {
        uint64_t x;
        std::memcpy(&x, v + k, 8);
        idx[k] = (uint32_t)map.val[map.find(x)];
    }
    tab.resize(nv);
    for (int64_t i = 0; i < nv; i++) std::memcpy(&tab[i], &all[i].first, 8);
    return true;
}

// Value index (CSR-VI, kernels.cuh ColsD16V16 / ColsD16V32 / ColsI32V32) of an autotuned CSR operator:
// the value dictionary of its stored entries (padding 0.0 included) and every stored entry's index;
// plus the packed (16-bit offset | 16-bit value index) words when the operator has the 16-bit column
// encoding and at most 65536 distinct values.  Built only where it can pay — at least 4 entries per
// distinct value and at most 2^21 distinct values (a 16 MB table, L2 resident) — so the autotuner can
// choose it; env AMG_VALUE_INDEX=0 disables it.  Lossless: the kernels read bitwise the stored values.
void encode_values(DevState &D, const double *v, int64_t stored, const uint16_t *off, DCsr &out) {
    if (stored < 2000000) return;  // below the autotuning threshold: never chosen
    if (const char *e = std::getenv("AMG_VALUE_INDEX"))
        if (std::atoi(e) == 0) return;
    std::vector<double> tab;
    Buf<uint32_t> idx;
    if (!value_dictionary(v, stored, false, std::min<int64_t>(1 << 21, stored / 4), tab, idx)) return;
    const int64_t nv = (int64_t)tab.size();
    out.nvals = nv;
    out.vtab = D.alloc_n<double>(nv);
    out.vidx = D.alloc_n<uint32_t>(stored);
    CUDA_OK(cudaMemcpy(out.vtab, tab.data(), 8 * (size_t)nv, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.vidx, idx.data(), 4 * (size_t)stored, cudaMemcpyHostToDevice));
    if (off && nv <= 65536) {
#pragma omp parallel for schedule(static)
        for (int64_t k = 0; k < stored; k++) idx[k] = (uint32_t)off[k] | (idx[k] << 16);
        out.vpk = D.alloc_n<uint32_t>(stored);
        CUDA_OK(cudaMemcpy(out.vpk, idx.data(), 4 * (size_t)stored, cudaMemcpyHostToDevice));
    }
}

// SELL-VI layout (fmt 2; kernels.cuh k_sellvi) of a host CSR: 32-row slices of one 32-bit word per
// entry (16-bit offset from the row's smallest column | 16-bit value index), quads of 4 consecutive
// entries of a row per lane, lane-interleaved within the slice; soff counts quads per lane.  The
// offset takes obits = max(16, bits of the widest row's span) bits, the value index the other 32 −
// obits.  Returns false (caller keeps CSR) if obits > 24 or the operator has more than 2^(32 − obits)
// distinct values (+0.0 for the padding); `rule` additionally requires >= 2e6 non-zeros, at most 50 %
// padding and row-to-row locality (below) — the automatic choice of format 0, for K_l and P̄_l.
bool upload_sellvi(DevState &D, const HCsr &A, DCsr &out, bool rule) {
    const int64_t n = A.nrows, nsl = (n + 31) / 32, nnz = A.nnz();
    if (n == 0 || nnz == 0) return false;
    if (rule && nnz < 2000000) return false;
    if (const char *e = std::getenv("AMG_SELLVI"))
        if (std::atoi(e) == 0) return false;
    Buf<int32_t> base(n);
    int64_t span = 0;
#pragma omp parallel for schedule(static) reduction(max : span)
    for (int64_t i = 0; i < n; i++) {
        const bool has = A.rp[i + 1] > A.rp[i];
        const int32_t lo = has ? A.ci[A.rp[i]] : 0, hi = has ? A.ci[A.rp[i + 1] - 1] : 0;  // ascending columns
        base[i] = lo;
        span = std::max<int64_t>(span, (int64_t)hi - (int64_t)lo);
    }
    int obits = 16;  // offset bits: at least 16, enough for the widest row; the value index gets the rest
    while ((span >> obits) != 0) obits++;
    if (obits > 24) return false;
    Buf<int64_t> soff(nsl + 1);  // in quads (4 entries) per lane
    soff[0] = 0;
    for (int64_t s = 0; s < nsl; s++) {
        int64_t W = 0;
        for (int64_t i = s * 32; i < std::min(n, s * 32 + 32); i++) W = std::max(W, A.rp[i + 1] - A.rp[i]);
        soff[s + 1] = soff[s] + (W + 3) / 4;
    }
    const int64_t stored = soff[nsl] * 128;
    if (rule && (double)stored > 1.5 * (double)nnz) return false;
    std::vector<double> tab;
    Buf<uint32_t> idx;
    if (!value_dictionary(A.v.data(), nnz, true, (int64_t)1 << (32 - obits), tab, idx)) return false;
    if (rule) {
        // Locality test (sampled, deterministic): for an entry column k of a slice, the 32 rows' x-gather
        // lines (128 B) and distinct table values are what one warp instruction costs in L1.  The
        // row-per-lane layout pays only when rows i and i+1 are shifted copies of each other (the fine
        // stencil: ≈ 4.7 lines, ≈ 4 values at C3-like sizes; P̄₀: 5.1, 9.0); the coarse Galerkin
        // operators are not (K₁: 9.7 lines, 17 values), and stay CSR.
        double lines = 0.0, vals = 0.0;
        int64_t samples = 0;
        const int64_t sstep = std::max<int64_t>(1, nsl / 512);
        for (int64_t s = 0; s < nsl; s += sstep) {
            const int64_t W = (soff[s + 1] - soff[s]) * 4;
            for (int64_t k = 0; k < W; k += 4) {
                int64_t ln[32], vv[32];
                int nl = 0, nv2 = 0;
                for (int64_t i = s * 32; i < std::min(n, s * 32 + 32); i++) {
                    if (A.rp[i] + k >= A.rp[i + 1]) continue;
                    const int64_t c = A.ci[A.rp[i] + k] >> 4, v = idx[A.rp[i] + k];
                    bool seen = false;
                    for (int t = 0; t < nl && !seen; t++) seen = ln[t] == c;
                    if (!seen) ln[nl++] = c;
                    seen = false;
                    for (int t = 0; t < nv2 && !seen; t++) seen = vv[t] == v;
                    if (!seen) vv[nv2++] = v;
                }
                if (!nl) continue;
                lines += nl;
                vals += nv2;
                samples++;
            }
        }
        if (samples == 0 || (lines + 0.5 * vals) / (double)samples > 12.0) return false;
        // Long rows with a table too large for shared memory: every lookup is an L2 gather, and a K_ℓ
        // with ~700 entries per row then runs ≈ 3× slower than in CSR (a coarse K₁ share on an interior
        // rank of a 4-GPU C3 run passed the test above with < 65,536 values; level 1 took 3.0 instead of
        // 0.95 ms per V-cycle).  Short rows (P̄_ℓ, ≤ 64 entries) keep SELL-VI with a global table.
        if ((int64_t)tab.size() > kSellviSmemVals && nnz > 64 * n) return false;
    }
    uint32_t zero = 0;
    for (size_t t = 0; t < tab.size(); t++) {
        uint64_t b;
        std::memcpy(&b, &tab[t], 8);
        if (b == 0) zero = (uint32_t)t;
    }
    // Windowed variant (k_sellviw): blocks of kWinSlices consecutive slices; the union of a block's
    // columns as runs of even length starting at even columns (gaps of <= kWinGap columns are staged
    // rather than split), each entry's word = its column's position in the block's window.  Every
    // vector it may gather is 16-B aligned at column 0 (the lower ghost areas of the distributed
    // vectors have even length).  AMG_SELLVI_WIN=0 keeps the plain SELL-VI words.
    // only with the value table in shared memory: P̄₀ at C3 (17.9 K values, global table) ran 54.9 µs
    // windowed against 43.9 µs plain (run r2p)
    bool win = (int64_t)tab.size() <= kSellviSmemVals;
    if (const char *e = std::getenv("AMG_SELLVI_WIN"))
        if (std::atoi(e) == 0) win = false;
    const int64_t nblk = (nsl + kWinSlices - 1) / kWinSlices;
    // the largest window: one window and the value table within kWinSmem (two CTAs per SM).  Measured
    // (run r2k): L3's ≈ 10 K-double windows at 2 CTAs/SM beat the plain layout (22.7 vs 23.3 ms per
    // iteration); C4's p = 4 windows with its 4,147-value table would leave 1 CTA/SM (1.90 vs 1.33 ms
    // per level-0 step) and stay plain.  AMG_WIN_MAX overrides (experiments).
    int64_t win_max = std::min<int64_t>(kWinMax, kWinSmem / 8 - (((int64_t)tab.size() + 1) & ~1));
    if (const char *e = std::getenv("AMG_WIN_MAX")) win_max = std::max<int64_t>(256, std::min<int64_t>(20000, std::atoll(e)));
    std::vector<std::vector<int4>> bruns;
    int64_t wmax = 0;
    if (win) {
        bruns.resize(nblk);
        bool ok = true;
#pragma omp parallel for schedule(dynamic, 16) reduction(max : wmax) reduction(&& : ok)
        for (int64_t b = 0; b < nblk; b++) {
            const int64_t r0 = b * kWinSlices * 32, r1 = std::min(n, r0 + kWinSlices * 32);
            std::vector<int32_t> cols(A.ci.data() + A.rp[r0], A.ci.data() + A.rp[r1]);
            std::sort(cols.begin(), cols.end());
            cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
            std::vector<int4> &R = bruns[b];
            int64_t tot = 0;
            for (size_t k = 0; k < cols.size();) {
                int64_t lo = cols[k] & ~1, hi = cols[k];
                size_t j = k + 1;
                while (j < cols.size() && (int64_t)cols[j] <= hi + 1 + kWinGap) hi = cols[j++];
                // inclusive and odd: an even length from an even start.  With an odd column count the
                // last run may end one double past the vector: device vectors are allocated in 256-B
                // units (DevState::alloc), so that double is inside the allocation (its value meets only
                // padding entries' 0.0 weights — never: no entry references it)
                hi |= 1;
                if (!R.empty() && lo <= (int64_t)R.back().x + R.back().y - 1 + kWinGap) {  // adjoining after rounding
                    const int64_t nhi = std::max<int64_t>(hi, R.back().x + R.back().y - 1);
                    tot += nhi - (R.back().x + R.back().y - 1);
                    R.back().y = (int)(nhi - R.back().x + 1);
                } else {
                    R.push_back(int4{(int)lo, (int)(hi - lo + 1), (int)tot, 0});
                    tot += hi - lo + 1;
                }
                k = j;
            }
            wmax = std::max<int64_t>(wmax, tot);
            ok = ok && tot <= win_max;
        }
        if (!ok || wmax == 0) win = false;
    }
    int pbits = 1;
    while (((int64_t)1 << pbits) < wmax) pbits++;
    if (win && (int64_t)tab.size() > ((int64_t)1 << (32 - pbits))) win = false;
    Buf<uint32_t> w(stored);
#pragma omp parallel for schedule(static)
    for (int64_t s = 0; s < nsl; s++) {
        const int64_t W = (soff[s + 1] - soff[s]) * 4;
        const std::vector<int4> *R = win ? &bruns[s / kWinSlices] : nullptr;
        for (int t = 0; t < 32; t++) {
            const int64_t i = s * 32 + t;
            const int64_t b = i < n ? A.rp[i] : 0, len = i < n ? A.rp[i + 1] - A.rp[i] : 0;
            size_t r = 0;
            for (int64_t k = 0; k < W; k++) {  // entry k of lane t: quad k/4, component k%4
                const int64_t dst = ((soff[s] + k / 4) * 32 + t) * 4 + k % 4;
                if (!win) {
                    w[dst] = k < len ? (uint32_t)(A.ci[b + k] - base[i]) | (idx[b + k] << obits) : zero << obits;
                } else if (k < len) {
                    const int32_t c = A.ci[b + k];  // ascending within the row: the run index only grows
                    while ((int64_t)(*R)[r].x + (*R)[r].y <= c) r++;
                    w[dst] = (uint32_t)((*R)[r].z + (c - (*R)[r].x)) | (idx[b + k] << pbits);
                } else {
                    w[dst] = zero << pbits;  // position 0 (a staged value), value 0.0
                }
            }
        }
    }
    if (win) {
        std::vector<int4> binfo(nblk), runs;
        for (int64_t b = 0; b < nblk; b++) {
            const int64_t tot = bruns[b].empty() ? 0 : bruns[b].back().z + bruns[b].back().y;
            binfo[b] = int4{(int)runs.size(), (int)(runs.size() + bruns[b].size()), (int)tot, 0};
            runs.insert(runs.end(), bruns[b].begin(), bruns[b].end());
        }
        out.win = true;
        out.pbits = pbits;
        if (8 * ((tab.size() <= (size_t)kSellviSmemVals ? ((int64_t)tab.size() + 1) & ~1 : 0) + 2 * ((wmax + 1) & ~1)) > 227 * 1024)
            out.nbuf = 1;
        // tail split of the last round (k_sellviw): against the nominal 3 CTAs per SM (U = 4, one
        // window: the usual choice), the leftover blocks are split in 2 or 4 items so the last round
        // is short; AMG_SELLVIW_SPLIT=k forces 2^k items for every block (tests), 0 disables
        {
            // only where the tail is a large share (<= 4 full rounds: the multi-GPU shares); at C3 on one
            // GPU (8 rounds) the split items' duplicated window copies and idle warps cost more than the
            // shorter tail saves (228 vs 221 µs, run r2i)
            const int64_t cnom = 3 * (int64_t)D.nsm, tail = nblk % cnom;
            const bool few = nblk / cnom <= 4;
            int wl = 0;
            while (few && tail > 0 && wl < 2 && (tail << (wl + 1)) <= cnom) wl++;
            int64_t wwhole = nblk - tail;
            if (const char *e = std::getenv("AMG_SELLVIW_SPLIT")) {
                wl = std::max(0, std::min(3, std::atoi(e)));
                wwhole = 0;
            }
            out.wl = wl;
            out.wwhole = wl ? wwhole : nblk;
        }
        out.wmax = (int)((wmax + 1) & ~1);
        out.nruns = (int64_t)runs.size();
        out.binfo = D.alloc_n<int4>(nblk);
        out.wruns = D.alloc_n<int4>(std::max<int64_t>(1, (int64_t)runs.size()));
        CUDA_OK(cudaMemcpy(out.binfo, binfo.data(), sizeof(int4) * nblk, cudaMemcpyHostToDevice));
        if (!runs.empty()) CUDA_OK(cudaMemcpy(out.wruns, runs.data(), sizeof(int4) * runs.size(), cudaMemcpyHostToDevice));
    }
    out.fmt = 2;
    out.obits = obits;
    out.stored = stored;
    out.G = 32;
    out.U = 2;
    out.kern = 0;
    out.nvals = (int64_t)tab.size();
    out.soff = D.alloc_n<int64_t>(nsl + 1);
    out.vpk = D.alloc_n<uint32_t>(stored);
    out.rbase = D.alloc_n<int32_t>(n);
    out.vtab = D.alloc_n<double>(out.nvals);
    CUDA_OK(cudaMemcpy(out.soff, soff.data(), sizeof(int64_t) * (nsl + 1), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.vpk, w.data(), sizeof(uint32_t) * stored, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.rbase, base.data(), sizeof(int32_t) * n, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.vtab, tab.data(), sizeof(double) * out.nvals, cudaMemcpyHostToDevice));
    // Tail split (k_sellvi): a slice is one warp's work item, and with few slices per resident warp the
    // last round runs a handful of slices on an idle GPU — a 4-GPU share of C3's K₀ has 7,353 slices
    // for ≈ 3,552 resident warps (24 per SM at U = 4): 3 rounds for 2.07 rounds of work.  The slices of
    // that last round (counted against the nominal 24 · n_SM warps, not the tuned grid, so the split
    // is a function of the operator alone) are split into 2^lparts ranges of consecutive quads (≤ 4
    // parts of ≥ 8 quads, enough items to fill the round).  A split slice sums its parts' chains in
    // part order — fixed, never dependent on timing; dot epilogues keep whole slices.
    {
        const int64_t wnom = 24 * (int64_t)D.nsm, tail = nsl % wnom;
        const int64_t avgq = (stored / 128) / std::max<int64_t>(nsl, 1);
        int lp = 0;
        // only where the tail is a large share of the work (≤ 4 full rounds: the multi-GPU shares); at
        // C3 on 1 GPU (8 full rounds) the split items' fence, atomic and dependent epilogue load cost
        // as much as the shortened tail saves (232.7 vs 230.1 µs, run 48)
        const bool few = nsl / wnom <= 4;
        while (few && tail > 0 && lp < 2 && (tail << lp) < wnom && avgq >= 8 * (2 << lp)) lp++;
        int64_t nwhole = nsl - tail;
        if (const char *e = std::getenv("AMG_SELLVI_PARTS")) {  // experiments / tests: every slice split
            lp = std::max(0, std::min(3, std::atoi(e)));
            nwhole = 0;
        }
        if (out.win) lp = 0;  // the windowed core keeps whole slices (single GPU: 8+ full rounds at C3)
        out.lparts = lp;
        out.nwhole = lp ? nwhole : nsl;
        if (lp > 0) {
            out.partial = D.alloc_n<double2>((nsl * 32) << lp);
            out.sticket = D.alloc_n<unsigned>(nsl);
            CUDA_OK(cudaMemset(out.sticket, 0, sizeof(unsigned) * nsl));
        }
    }
    return true;
}

// 16-bit column offsets (ColsD16, kernels.cuh): base = the row's smallest stored column, offsets
// col − base.  Returns false (no encoding; int32 columns only) if a row spans more than 65535 columns.
bool encode_d16(DevState &D, const int64_t *rp, const int32_t *ci, int64_t nrows, DCsr &out, Buf<uint16_t> *keep) {
    Buf<int32_t> base(nrows);
    bool ok = true;
#pragma omp parallel for schedule(static) reduction(&& : ok)
    for (int64_t i = 0; i < nrows; i++) {
        int32_t lo = 0, hi = 0;
        if (rp[i + 1] > rp[i]) lo = hi = ci[rp[i]];
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) {
            lo = std::min(lo, ci[e]);
            hi = std::max(hi, ci[e]);
        }
        base[i] = lo;
        ok = ok && ((int64_t)hi - (int64_t)lo <= 65535);
    }
    if (!ok) return false;
    const int64_t stored = rp[nrows];
    Buf<uint16_t> off(stored);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < nrows; i++)
        for (int64_t e = rp[i]; e < rp[i + 1]; e++) off[e] = (uint16_t)(ci[e] - base[i]);
    out.off16 = D.alloc_n<uint16_t>(stored);
    out.rbase = D.alloc_n<int32_t>(nrows);
    CUDA_OK(cudaMemcpy(out.off16, off.data(), sizeof(uint16_t) * stored, cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(out.rbase, base.data(), sizeof(int32_t) * nrows, cudaMemcpyHostToDevice));
    if (keep) *keep = std::move(off);
    return true;
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

// Format choice (amg_params.format): 1 = CSR2 everywhere; 2 = SELL2 wherever allowed; 0 = auto.
// Auto = CSR2: measured on B200 at C3 level 0, CSR2 streams at 4.55 TB/s vs SELL2's 4.10 TB/s
// (profiles/r01), and SELL2 starves the GPU on the short coarse levels.
void upload_op(DevState &D, const HCsr &A, DCsr &out, bool square, int format, bool force_csr, int role) {
    out.nrows = A.nrows;
    out.ncols = A.ncols;
    out.nnz = A.nnz();
    // SELL-VI: format 0 by the fixed rule on the K_l and P̄_l, format 6 wherever admissible (never the
    // coarsest K)
    if (!force_csr && ((format == 0 && (role == 0 || role == 1)) || format == 6) && upload_sellvi(D, A, out, format == 0))
        return;
    if (format == 0 || format >= 3) {
        // rows padded to 8 entries (16-byte aligned value, int32 and 16-bit column ranges): runnable by
        // both the register-batched CSR2 core and the TMA-staged CSR4T core (format 0 autotunes)
        upload_csr2(D, A, out, square, 8);
        out.kern = (format == 3) ? 1 : (format == 4 && out.off16) ? 2 : (format == 5 && out.off16) ? 3 : 0;  // 6: CSR fallback
        return;
    }
    const bool sell = !force_csr && format == 2;
    if (sell) upload_sell2(D, A, out, square);
    else upload_csr2(D, A, out, square);
}

int grid_for(const DevState &D, int64_t n) {
    int64_t g = (n + dev::kBlock - 1) / dev::kBlock;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, D.max_grid));
}


// Setup-time autotuning of one CSR4-layout operator: time it with the epilogue it runs in the V-cycle
// (role 0: K_l with the fused Chebyshev step, 1: P̄_l with prolongation, 2: R_l with restriction) for
// every (kernel, G, U) candidate and keep the fastest.  All candidates sum each row in the same order,
// so the choice changes speed, never results.  Small operators (latency-bound) keep the heuristic.
template <class Epi>
float time_op(DevState &D, DCsr &A, const double *x, const Epi &e, cudaEvent_t e0, cudaEvent_t e1) {
    launch_csr(D, A, x, e, nullptr);
    float best = 1e30f;
    for (int round = 0; round < 2; round++) {  // best of 2 rounds of 3 back-to-back launches
        CUDA_OK(cudaEventRecord(e0, nullptr));
        for (int rep = 0; rep < 3; rep++) launch_csr(D, A, x, e, nullptr);
        CUDA_OK(cudaEventRecord(e1, nullptr));
        CUDA_OK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
    }
    return best;
}

// Tuning cache (env AMG_TUNE_CACHE = path): one line per tuned operator,
//   "<rank> <nranks> <level> <role> <nrows> <nnz> <kern> <G> <U> <pf> <us>".
// A hit (same rank, ranks, level, role and operator shape) reuses the stored choice, so separate runs
// (the bench, its ncu capture) execute the same kernel variants; misses are tuned and appended.
struct TuneKey {
    int rank, nranks, level, role;
    int64_t nrows, nnz;
};
bool tune_lookup(const TuneKey &k, DCsr &A) {
    const char *path = std::getenv("AMG_TUNE_CACHE");
    if (!path) return false;
    FILE *f = std::fopen(path, "r");
    if (!f) return false;
    int r, nr, l, ro, kern, G, U, pf;
    long long n, z;
    float us;
    bool hit = false;
    while (std::fscanf(f, "%d %d %d %d %lld %lld %d %d %d %d %f", &r, &nr, &l, &ro, &n, &z, &kern, &G, &U, &pf, &us) == 11) {
        if (r == k.rank && nr == k.nranks && l == k.level && ro == k.role && n == k.nrows && z == k.nnz) {
            // kern 16 marks a SELL-VI entry, 17 a windowed SELL-VI one (pf = windows staged per CTA);
            // skip entries of another layout or for encodings this operator lacks
            if ((kern == 16) != (A.fmt == 2 && !A.win) || (kern == 17) != (A.fmt == 2 && A.win) ||
                ((kern & 2) && kern < 16 && !A.off16) || ((kern & 8) && kern < 16 && !A.vtab))
                continue;
            if (kern == 17) {
                A.nbuf = pf == 1 ? 1 : 2;
                pf = 0;
            }
            if (kern >= 16) kern = 0;
            A.kern = kern;
            A.G = G;
            A.U = U;
            A.pf = pf;
            A.tuned_us = us;
            hit = true;
        }
    }
    std::fclose(f);
    return hit;
}
void tune_store(const TuneKey &k, const DCsr &A) {
    // appending is opt-in (AMG_TUNE_CACHE_WRITE=1): a committed cache read by the bench is never
    // modified by a run, and concurrent ranks never interleave lines in it
    const char *path = std::getenv("AMG_TUNE_CACHE");
    const char *wr = std::getenv("AMG_TUNE_CACHE_WRITE");
    if (!path || !wr || std::strcmp(wr, "1") != 0) return;
    if (FILE *f = std::fopen(path, "a")) {
        std::fprintf(f, "%d %d %d %d %lld %lld %d %d %d %d %.2f\n", k.rank, k.nranks, k.level, k.role,
                     (long long)k.nrows, (long long)k.nnz, A.fmt == 2 ? (A.win ? 17 : 16) : A.kern, A.G, A.U,
                     A.fmt == 2 && A.win ? A.nbuf : A.pf, A.tuned_us);
        std::fclose(f);
    }
}

}  // namespace

int resident_ctas(const void *fn, int block, int smem, int smem_attr) {
    static std::mutex mu;
    static std::map<std::tuple<const void *, int, int, int, int>, int> cache;
    static std::map<std::pair<const void *, int>, int> attr;  // the attribute only ever grows per (kernel, device)
    int dev = 0;
    CUDA_OK(cudaGetDevice(&dev));
    const auto key = std::make_tuple(fn, dev, block, smem, smem_attr);
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    int &cur = attr[std::make_pair(fn, dev)];
    if (smem_attr > cur) {
        CUDA_OK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_attr));
        cur = smem_attr;
    }
    int per_sm = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, block, smem));
    per_sm = std::max(per_sm, 1);
    cache.emplace(key, per_sm);
    return per_sm;
}

namespace {

float time_role(DevState &D, DCsr &A, int role, double *x, double *y1, double *y2, double *y3, cudaEvent_t e0,
                cudaEvent_t e1) {
    if (role == 0) {
        dev::EpiCheb<false> e{};
        e.rin = y1; e.rout = y1; e.dold = x; e.dnew = y2; e.invd = y3;
        e.xin = y3; e.dpend = nullptr; e.xout = y3; e.bdot = nullptr; e.a = 0.5; e.bc = 0.5;
        return time_op(D, A, x, e, e0, e1);
    } else if (role == 1) {
        dev::EpiProlong e{y1};
        return time_op(D, A, x, e, e0, e1);
    }
    dev::EpiRestrict e{y1, y3, y2, 1.0};
    return time_op(D, A, x, e, e0, e1);
}

void autotune_op(DevState &D, DCsr &A, int level, int role, double *x, double *y1, double *y2, double *y3) {
    if ((A.fmt != 0 && A.fmt != 2) || A.nnz < 2000000) return;
    if (std::getenv("AMG_CSR_G") || std::getenv("AMG_CSR_U")) return;
    if (const char *e = std::getenv("AMG_AUTOTUNE"))
        if (std::atoi(e) == 0) return;
    const TuneKey key{D.rank, D.nranks, level, role, A.nrows, A.nnz};
    if (tune_lookup(key, A)) return;
    cudaEvent_t e0, e1;
    CUDA_OK(cudaEventCreate(&e0));
    CUDA_OK(cudaEventCreate(&e1));
    if (A.fmt == 2) {  // SELL-VI: entries in flight per lane (bitwise-equal results for every U) and,
                       // windowed, the windows staged per CTA
        float best = 1e30f;
        int bu = A.U, bb = A.nbuf;
        for (int nb : {2, 1}) {
            if (nb == 1 && !A.win) continue;
            // two windows must fit the 227 KB of shared memory a CTA may have (next to the table)
            const int64_t tabn = A.nvals <= kSellviSmemVals ? (A.nvals + 1) & ~1 : 0;
            if (nb == 2 && A.win && 8 * (tabn + 2 * (int64_t)A.wmax) > 227 * 1024) continue;
            for (int U : {1, 2, 4}) {
                A.U = U;
                A.nbuf = nb;
                const float ms = time_role(D, A, role, x, y1, y2, y3, e0, e1);
                if (ms < best) {
                    best = ms;
                    bu = U;
                    bb = nb;
                }
            }
        }
        A.U = bu;
        A.nbuf = bb;
        A.tuned_us = best / 3.f * 1000.f;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        D.launches_total = 0;
        tune_store(key, A);
        return;
    }
    const int Gs[] = {1, 2, 4, 8, 32};  // G = 2: long rows, few of them (C3's K2: 7,383 pairs for 3,552 warps)
    const int Us[] = {2, 4, 6, 8};
    float best = 1e30f;
    int bk = A.kern, bg = A.G, bu = A.U, bp = A.pf;
    // kern bit 1 (16-bit column offsets) needs the encoding, bit 3 (value index) the value table
    std::vector<int> kerns = {0, 1};
    if (A.off16) kerns.insert(kerns.end(), {2, 3});
    if (A.vtab) {
        kerns.push_back(8);
        if (A.off16) kerns.push_back(10);
    }
    for (int kern : kerns)
        for (int G : Gs)
            for (int U : Us)
                for (int pf = 0; pf < 2; pf++) {
                if ((kern & 1) && U > 4) continue;
                if (pf && ((kern & 1) || G == 1)) continue;  // prefetch: register core, groups of > 1 row
                if ((A.nrows + G - 1) / G < 4 * D.nsm) continue;  // too few warp groups to fill the GPU
                A.kern = kern;
                A.G = G;
                A.U = U;
                A.pf = pf;
                const float ms = time_role(D, A, role, x, y1, y2, y3, e0, e1);
                if (ms < best) {
                    best = ms;
                    bk = kern;
                    bg = G;
                    bu = U;
                    bp = pf;
                }
            }
    A.kern = bk;
    A.G = bg;
    A.U = bu;
    A.pf = bp;
    A.tuned_us = best / 3.f * 1000.f;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    D.launches_total = 0;
    tune_store(key, A);
}

// Per-level breakdown mark (no-op unless D.lvl_prof).
void level_mark(DevState &D, int l, int kind, cudaStream_t st) {
    if (!D.lvl_prof) return;
    if (D.lev_ev_used >= D.lev_ev.size()) {
        for (int k = 0; k < 256; k++) {
            cudaEvent_t e;
            CUDA_OK(cudaEventCreate(&e));
            D.lev_ev.push_back(e);
        }
    }
    CUDA_OK(cudaEventRecord(D.lev_ev[D.lev_ev_used++], st));
    D.lev_marks.push_back({l, kind});
}

// Fold the recorded marks into exclusive per-level times (after the stream has completed).
void level_collect(DevState &D) {
    if (!D.lvl_prof || D.lev_ev_used == 0) return;
    // exclusive(l) = (exit − enter) − (child end − child start)
    std::vector<size_t> enter(32), cstart(32);
    for (size_t k = 0; k < D.lev_ev_used; k++) {
        const int l = D.lev_marks[k].first, kind = D.lev_marks[k].second;
        float ms = 0.f;
        if (kind == 0) enter[l] = k;
        else if (kind == 1) cstart[l] = k;
        else if (kind == 2) {
            CUDA_OK(cudaEventElapsedTime(&ms, D.lev_ev[cstart[l]], D.lev_ev[k]));
            D.lvl_ms[l] -= ms;
        } else {
            CUDA_OK(cudaEventElapsedTime(&ms, D.lev_ev[enter[l]], D.lev_ev[k]));
            D.lvl_ms[l] += ms;
            if (l == 0) D.lvl_vcycles++;
        }
    }
    D.lev_ev_used = 0;
    D.lev_marks.clear();
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
        // External: inside stream capture this becomes a real event-record node of the graph, so
        // the pair can be timed after every graph launch (the flag is only valid while capturing)
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_OK(cudaStreamIsCapturing(st, &cs));
        flags = (cs == cudaStreamCaptureStatusActive) ? cudaEventRecordExternal : cudaEventRecordDefault;
        CUDA_OK(cudaEventRecordWithFlags(D.ev[D.ev_used], st, flags));
    }
    ~ProfScope() {
        if (!on) return;
        cudaEventRecordWithFlags(D.ev[D.ev_used + 1], st, flags);
        D.ev_used += 2;
    }
    unsigned flags = 0;
};

#define NCCL_OK(call)                                                                              \
    do {                                                                                           \
        ncclResult_t r_ = (call);                                                                  \
        if (r_ != ncclSuccess)                                                                     \
            throw Error{AMG_ENCCL, std::string(#call) + ": " + ncclGetErrorString(r_)};            \
    } while (0)

// a12 (NCCL transport): fill the ghost slots of x (the vector A gathers) from their owning ranks —
// pack the owned entries others need, then one grouped NCCL send/recv per neighbour straight into the
// ghost area.  With the P2P transport the producers already pushed the ghosts: nothing to do.
void halo(DevState &D, const DCsr &A, double *x, cudaStream_t st) {
    if (!A.halo || D.p2p) return;
    if (A.nsend > 0) {
        launch_k(dev::k_pack, grid_for(D, A.nsend), dev::kBlock, 0, st, A.nsend, A.sidx, x, A.sbuf);
        D.launches_total++;
    }
    NCCL_OK(ncclGroupStart());
    for (int q = 0; q < D.nranks; q++) {
        if (A.hs_count[q]) NCCL_OK(ncclSend(A.sbuf + A.hs_off[q], (size_t)A.hs_count[q], ncclFloat64, q, D.comm, st));
        if (A.hr_count[q]) NCCL_OK(ncclRecv(x + A.slot(A.hr_off[q]), (size_t)A.hr_count[q], ncclFloat64, q, D.comm, st));
    }
    NCCL_OK(ncclGroupEnd());
}

// a12: sum a per-rank dot product across ranks into the device scalar block: NCCL all-reduce, or (P2P)
// a one-thread kernel adding the ranks' deposited sums in rank order.
void allreduce_dot(DevState &D, int dotkind, cudaStream_t st) {
    if (D.nranks == 1) return;
    const int kind = dotkind & 255, kind2 = dotkind >> 8;
    if (D.p2p) {
        launch_k(dev::k_dot_collect, 1, 32, 0, st, kind, kind2, D.S, p2p_of(D, true));
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
        return;
    }
    for (int k : {kind, kind2}) {
        if (k == dev::DOT_NONE) continue;
        double *slot = k == dev::DOT_FF ? &D.S->ff : k == dev::DOT_RR ? &D.S->rr : k == dev::DOT_PQ ? &D.S->pq
                     : k == dev::DOT_RZ ? &D.S->rz : k == dev::DOT_PR ? &D.S->pr : &D.S->zq;
        NCCL_OK(ncclAllReduce(slot, slot, 1, ncclFloat64, ncclSum, D.comm, st));
    }
}

const double kC0 = 4.0 / 3.0;

// c.16 pre-smoothing steps i = 1..m-1 and the residual (a4, a5), restriction (a6), recursion,
// prolongation (a8), post-smoothing (a9, a10).  b, x: this level's right-hand side and output
// (this rank's rows).  Ghost values reach the gathering kernels either by halo() (NCCL) right before
// them, or (P2P) by the producing epilogues' pushes (push_of: d_new/d0 along K_l's plan, r along R_l's,
// x after prolongation along K_l's, the final x of a coarse level along P̄_{l-1}'s).
void vcycle_level_body(DevState &D, int l, const double *b, double *x, cudaStream_t st, int final_dot,
                       const double *final_bdot);
void vcycle_level(DevState &D, int l, const double *b, double *x, cudaStream_t st, int final_dot,
                  const double *final_bdot = nullptr) {
    level_mark(D, l, 0, st);
    vcycle_level_body(D, l, b, x, st, final_dot, final_bdot);
    level_mark(D, l, 3, st);
}
void vcycle_level_body(DevState &D, int l, const double *b, double *x, cudaStream_t st, int final_dot,
                       const double *final_bdot) {
    DLevel &L = D.lev[l];
    const int m = D.m;
    // the first replicated level waits (P2P) for every rank's share of its right-hand side
    const bool first_rep = D.nranks > 1 && L.replicated && !D.lev[l - 1].replicated;
    if (l == D.nlevels - 1) {
        const int n = (int)L.N;
        // stage the operator in shared memory when it fits (the coarsest level is tiny by design)
        const size_t base = sizeof(double) * 4 * (size_t)n;
        const size_t full = base + (size_t)L.K.stored * 12 + sizeof(int) * (size_t)(n + 1);
        const int staged = full <= 200 * 1024 ? 1 : 0;
        const size_t smem = staged ? full : base;
        if (D.coarse_solver == 1) {  // §5.1: CG preconditioned by one weighted-Jacobi sweep
            const size_t base2 = sizeof(double) * 6 * (size_t)n;
            const size_t full2 = base2 + (size_t)L.K.stored * 12 + sizeof(int) * (size_t)(n + 1);
            const int staged2 = full2 <= 200 * 1024 ? 1 : 0;
            const size_t smem2 = staged2 ? full2 : base2;
            if (smem2 > 48 * 1024) (void)resident_ctas((const void *)dev::k_coarse_cg, 1024, (int)smem2, (int)smem2);
            launch_k(dev::k_coarse_cg, 1, 1024, smem2, st, n, L.K.rp, L.K.ci, L.K.v, L.diag, b, x, D.coarse_tol,
                                                    D.coarse_maxit, staged2, p2p_of(D, first_rep));
            D.launches_total++;
            CUDA_OK(cudaGetLastError());
            return;
        }
        if (smem > 48 * 1024) (void)resident_ctas((const void *)dev::k_coarse_solve, 1024, (int)smem, (int)smem);
        launch_k(dev::k_coarse_solve, 1, 1024, smem, st, n, L.K.rp, L.K.ci, L.K.v, L.invd, b, x, D.sweeps, staged,
                                                  p2p_of(D, first_rep));
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
        return;
    }
    DLevel &C = D.lev[l + 1];
    const bool coarse_is_last = (l + 1 == D.nlevels - 1);
    const DCsr *Pabove = l > 0 ? &D.lev[l - 1].P : nullptr;  // gathers this level's final x
    // --- pre-smoothing from x = 0: d0 = c0·b·invd (level 0 and the first replicated level; other
    //     coarse levels: restriction epilogue)
    if (l == 0 || first_rep) {
        launch_k(dev::k_cheb_first, grid_for(D, L.n), dev::kBlock, 0, st, L.n, b, L.invd, L.d[0], kC0,
                                                                   push_of(D, L.K, L.d[0]),
                                                                   p2p_of(D, l == 0 || first_rep,
                                                                          first_rep ? ~0u : L.K.wmask));
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
    }
    int cur = 0;
    for (int i = 1; i < m; i++) {
        halo(D, L.K, L.d[cur], st);
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
        e.pushD = push_of(D, L.K, L.d[cur ^ 1]);
        ProfScope ps(D, st, l == 0);
        launch_csr(D, L.K, L.d[cur], e, st);
        cur ^= 1;
    }
    // residual r = r − K d_{m−1}   (m == 1: r = b − K d0, x = d0)
    {
        halo(D, L.K, L.d[cur], st);
        dev::EpiResidualFrom e{};
        e.b = (m == 1) ? b : L.r;
        e.r = L.r;
        e.dpend = (m == 1) ? L.d[cur] : nullptr;
        e.x = x;
        e.pushR = push_of(D, L.R, L.r);
        launch_csr(D, L.K, L.d[cur], e, st);
    }
    // restriction b_c = R r, fused with the coarse level's first smoothing step d0_c = c0·b_c·invd_c
    halo(D, L.R, L.r, st);
    if (C.replicated && !L.replicated && D.p2p) {
        // last distributed level (P2P): each rank restricts its share of the coarse rows straight into
        // every rank's whole coarse right-hand side (an all-gather by pushes)
        dev::EpiRestrict e{};
        e.bc = C.b + D.ag_row0;
        e.invd = nullptr;
        e.d0 = nullptr;
        e.c0 = kC0;
        e.pushB = dev::Push{D.ag_ptr, D.ag_dst, D.d_base, (long long)((const char *)C.b - D.slab)};
        launch_csr(D, L.R, L.r, e, st);
    } else if (C.replicated && !L.replicated) {
        // last distributed level (NCCL): each rank restricts its share of the coarse rows, then an
        // all-gather assembles the whole coarse right-hand side on every rank
        dev::EpiRestrict e{};
        e.bc = D.ag_send;
        e.invd = nullptr;
        e.d0 = nullptr;
        e.c0 = kC0;
        launch_csr(D, L.R, L.r, e, st);
        NCCL_OK(ncclAllGather(D.ag_send, D.ag_recv, (size_t)D.ag_stride, ncclFloat64, D.comm, st));
        launch_k(dev::k_unpack_allgather, grid_for(D, D.ag_stride), dev::kBlock, 0, st, D.nranks, D.ag_stride,
                                                                                D.ag_bounds, D.ag_recv, C.b);
        D.launches_total++;
        if (!coarse_is_last) {
            launch_k(dev::k_cheb_first, grid_for(D, C.n), dev::kBlock, 0, st, C.n, C.b, C.invd, C.d[0], kC0, dev::Push{},
                                                                       dev::P2P{});
            D.launches_total++;
        }
        CUDA_OK(cudaGetLastError());
    } else {
        dev::EpiRestrict e{};
        e.bc = C.b;
        e.invd = coarse_is_last ? nullptr : C.invd;
        e.d0 = C.d[0];
        e.c0 = kC0;
        e.pushD = push_of(D, C.K, C.d[0]);
        launch_csr(D, L.R, L.r, e, st);
    }
    level_mark(D, l, 1, st);
    vcycle_level(D, l + 1, C.b, C.x, st, dev::DOT_NONE);
    level_mark(D, l, 2, st);
    // prolongation x += P̄ x_c
    {
        halo(D, L.P, C.x, st);
        dev::EpiProlong e{};
        e.x = x;
        e.pushX = push_of(D, L.K, x);
        launch_csr(D, L.P, C.x, e, st);
    }
    // post-smoothing: r = b − K x; d0 = c0·r·invd
    {
        halo(D, L.K, x, st);
        dev::EpiPostFirst e{};
        e.b = b;
        e.r = L.r;
        e.invd = L.invd;
        e.d0 = L.d[0];
        e.c0 = kC0;
        e.pushD = push_of(D, L.K, L.d[0]);
        launch_csr(D, L.K, x, e, st);
    }
    cur = 0;
    for (int i = 1; i < m; i++) {
        const bool lastd = (i == m - 1) && final_dot != dev::DOT_NONE;
        const double a = (double)(2 * i - 1) / (double)(2 * i + 3);
        const double bcf = (double)(8 * i + 4) / (double)(2 * i + 3);
        const dev::Push pd = (i < m - 1) ? push_of(D, L.K, L.d[cur ^ 1]) : dev::Push{};
        const dev::Push px = (i == m - 1 && Pabove) ? push_of(D, *Pabove, x) : dev::Push{};
        halo(D, L.K, L.d[cur], st);
        ProfScope ps(D, st, l == 0);
        if (lastd) {
            dev::EpiCheb<true> e{};
            e.rin = L.r; e.rout = L.r; e.dold = L.d[cur]; e.dnew = L.d[cur ^ 1]; e.invd = L.invd;
            e.xin = x; e.dpend = (i == 1) ? L.d[cur] : nullptr; e.xout = x; e.bdot = final_bdot ? final_bdot : b;
            e.a = a; e.bc = bcf;
            e.pushD = pd; e.pushX = px;
            launch_csr(D, L.K, L.d[cur], e, st, final_dot);
        } else {
            dev::EpiCheb<false> e{};
            e.rin = L.r; e.rout = L.r; e.dold = L.d[cur]; e.dnew = L.d[cur ^ 1]; e.invd = L.invd;
            e.xin = x; e.dpend = (i == 1) ? L.d[cur] : nullptr; e.xout = x; e.bdot = nullptr; e.a = a; e.bc = bcf;
            e.pushD = pd; e.pushX = px;
            launch_csr(D, L.K, L.d[cur], e, st);
        }
        cur ^= 1;
    }
    if (m == 1) {
        launch_k(dev::k_axpy1, grid_for(D, L.n), dev::kBlock, 0, st, L.n, L.d[0], x);
        D.launches_total++;
        CUDA_OK(cudaGetLastError());
    }
}

}  // namespace

// V-cycle with the rᵀz dot (kind) fused into the last level-0 post-smoothing step (then summed
// across ranks).
// bdot: the vector dotted with the V-cycle output (nullptr: b, giving rᵀz; FCG passes q_prev → zᵀq_prev).
static void vcycle(DevState &D, const double *b, double *x, cudaStream_t st, int dotkind, const double *bdot = nullptr) {
    const int64_t n0 = D.lev[0].n;
    const bool fused = dotkind != dev::DOT_NONE && D.m > 1 && D.nlevels > 1;
    vcycle_level(D, 0, b, x, st, fused ? dotkind : dev::DOT_NONE, bdot);
    if (dotkind != dev::DOT_NONE && !fused) {
        launch_k(dev::k_dot, grid_for(D, n0), dev::kBlock, 0, st, n0, bdot ? bdot : b, x, dotctx(D, dotkind));
        D.launches_total++;
    }
    if (dotkind != dev::DOT_NONE) allreduce_dot(D, dotkind, st);
}

namespace {
// Upload one rank's share of a distributed operator (local columns + halo plan).  Local columns keep
// the global order (lower ghosts negative, dist.cpp); lo_shift / hi_shift move the lower / upper ghost
// columns further out, past another gatherer's ghosts of the same vector (P̄_l's beyond K_{l+1}'s).
void upload_local(DevState &D, const LocalOp &op, DCsr &out, int format, int role, int64_t lo_shift = 0,
                  int64_t hi_shift = 0) {
    const int64_t nown = op.col_end - op.col_begin;
    if ((lo_shift > 0 || hi_shift > 0) && !op.full_cols && !op.ghost.empty()) {
        HCsr A;
        A.nrows = op.A.nrows;
        A.ncols = op.A.ncols + lo_shift + hi_shift;
        A.rp.alloc(A.nrows + 1);
        std::memcpy(A.rp.data(), op.A.rp.data(), sizeof(int64_t) * (A.nrows + 1));
        const int64_t nnz = op.A.nnz();
        A.ci.alloc(nnz);
        A.v.alloc(nnz);
        std::memcpy(A.v.data(), op.A.v.data(), sizeof(double) * nnz);
        for (int64_t k = 0; k < nnz; k++) {
            const int32_t c = op.A.ci[k];
            A.ci[k] = c < 0 ? (int32_t)(c - lo_shift) : c >= nown ? (int32_t)(c + hi_shift) : c;
        }
        upload_op(D, A, out, false, format, false, role);
    } else {
        upload_op(D, op.A, out, false, format, false, role);
    }
    if (op.full_cols || D.nranks == 1) return;
    out.halo = true;
    out.nown = nown;
    out.nghost = (int64_t)op.ghost.size();
    out.nlo = op.nlo;
    out.lo_base = -op.nlo - lo_shift;
    out.hi_base = nown + hi_shift;
    out.hs_count.assign(op.send_count.begin(), op.send_count.end());
    out.hs_off.assign(op.send_off.begin(), op.send_off.end());
    out.hr_count.assign(op.recv_count.begin(), op.recv_count.end());
    out.hr_off.assign(op.recv_off.begin(), op.recv_off.end());
    out.nsend = (int64_t)op.send_idx.size();
    if (out.nsend > 0) {
        out.sidx = D.alloc_n<int>(out.nsend);
        out.sbuf = D.alloc_n<double>(out.nsend);
        CUDA_OK(cudaMemcpy(out.sidx, op.send_idx.data(), sizeof(int) * out.nsend, cudaMemcpyHostToDevice));
    }
}

// All-gather of int64 host arrays (one per rank, equal length) over the NCCL communicator.
std::vector<int64_t> nccl_allgather_i64(DevState &D, const std::vector<int64_t> &mine) {
    const size_t n = mine.size();
    int64_t *dbuf = nullptr;
    CUDA_OK(cudaMalloc(&dbuf, sizeof(int64_t) * n * (D.nranks + 1)));
    std::vector<int64_t> all(n * D.nranks);
    CUDA_OK(cudaMemcpy(dbuf, mine.data(), sizeof(int64_t) * n, cudaMemcpyHostToDevice));
    NCCL_OK(ncclAllGather(dbuf, dbuf + n, n, ncclInt64, D.comm, nullptr));
    CUDA_OK(cudaStreamSynchronize(nullptr));
    CUDA_OK(cudaMemcpy(all.data(), dbuf + n, sizeof(int64_t) * n * D.nranks, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    return all;
}

// Slab layout (identical on every rank): flags, epoch, ticket, dot slots, then the vectors.
constexpr size_t kFlagsOff = 0, kEpochOff = 512, kTicketOff = 576, kBTicketOff = 640, kDslotOff = 1024,
                 kVecOff = 4096;

// Push plan of operator A's gathered vector: for each owned index j, the (rank, slot) pairs of the
// other ranks' ghost copies.  meta_of(q) = {lo_base, hi_base, nlo, recv_off[0..nranks)} of rank q's
// copy of A: my t-th value for q lands in q's ghost position recv_off[me] + t.
void build_push(DevState &D, const LocalOp &op, DCsr &A, const std::vector<int64_t> &meta, size_t meta_stride,
                size_t meta_pos) {
    const int nr = D.nranks, me = D.rank;
    const int64_t nown = op.col_end - op.col_begin;
    std::vector<int> cnt(nown + 1, 0);
    for (int q = 0; q < nr; q++)
        for (int t = 0; t < op.send_count[q]; t++) cnt[op.send_idx[op.send_off[q] + t] + 1]++;
    for (int64_t j = 0; j < nown; j++) cnt[j + 1] += cnt[j];
    if (cnt[nown] == 0) return;
    std::vector<int2> dst(cnt[nown]);
    std::vector<int> fill(cnt.begin(), cnt.end() - 1);
    for (int q = 0; q < nr; q++) {
        if (q == me || op.send_count[q] == 0) continue;
        const int64_t *mq = meta.data() + (size_t)q * meta_stride + meta_pos;
        const int64_t lo_base = mq[0], hi_base = mq[1], nlo = mq[2], g0 = mq[3 + me];
        for (int t = 0; t < op.send_count[q]; t++) {
            const int j = op.send_idx[op.send_off[q] + t];
            const int64_t g = g0 + t;
            dst[fill[j]++] = make_int2(q, (int)(g < nlo ? lo_base + g : hi_base + (g - nlo)));
        }
        A.pmask |= 1u << q;
    }
    A.pushed.assign(nown, 0);
    for (int64_t j = 0; j < nown; j++) A.pushed[j] = cnt[j + 1] > cnt[j];
    A.push_ptr = D.alloc_n<int>(nown + 1);
    A.push_dst = D.alloc_n<int2>((int64_t)dst.size());
    CUDA_OK(cudaMemcpy(A.push_ptr, cnt.data(), sizeof(int) * (nown + 1), cudaMemcpyHostToDevice));
    CUDA_OK(cudaMemcpy(A.push_dst, dst.data(), sizeof(int2) * dst.size(), cudaMemcpyHostToDevice));
}

// Row-group order of a CSR operator for its current G: boundary groups (any row reading a ghost value
// or pushed somewhere) first, then the interior ones.
void build_gorder(DevState &D, DCsr &A) {
    if (A.bnd.empty() || (A.fmt != 0 && A.fmt != 2)) return;
    if (const char *e = std::getenv("AMG_P2P_INTERIOR"))  // 0: every kernel waits at its start (debug)
        if (std::atoi(e) == 0) return;
    const int64_t G = order_granule(A), ng = (A.nrows + G - 1) / G;
    std::vector<int> order, tail;
    order.reserve(ng);
    for (int64_t g = 0; g < ng; g++) {
        bool b = false;
        for (int64_t i = g * G; i < std::min(A.nrows, (g + 1) * G) && !b; i++) b = A.bnd[i] != 0;
        (b ? order : tail).push_back((int)g);
    }
    A.nbnd = (int64_t)order.size();
    order.insert(order.end(), tail.begin(), tail.end());
    if (!A.gorder || A.gorder_cap < ng) {
        A.gorder = D.alloc_n<int>(ng);
        A.gorder_cap = ng;
    }
    CUDA_OK(cudaMemcpy(A.gorder, order.data(), sizeof(int) * ng, cudaMemcpyHostToDevice));
    A.gorder_G = G;
}

// P2P transport setup: IPC-export the slab, map every other rank's, build the push plans of every
// distributed operator and of the all-gather into the first replicated level, mark the participating
// operators.  Runs after autotuning (autotuning launches are local).
void p2p_setup(DevState &D, const DistPlan &plan) {
    const int nr = D.nranks, me = D.rank, ld = D.last_dist;
    // 1. slab handles
    {
        cudaIpcMemHandle_t h;
        CUDA_OK(cudaIpcGetMemHandle(&h, D.slab));
        std::vector<int64_t> mine((sizeof(h) + 7) / 8, 0);
        std::memcpy(mine.data(), &h, sizeof(h));
        const std::vector<int64_t> all = nccl_allgather_i64(D, mine);
        std::vector<char *> bases(nr, nullptr);
        for (int q = 0; q < nr; q++) {
            if (q == me) {
                bases[q] = D.slab;
                continue;
            }
            cudaIpcMemHandle_t hq;
            std::memcpy(&hq, all.data() + (size_t)q * mine.size(), sizeof(hq));
            void *ptr = nullptr;
            CUDA_OK(cudaIpcOpenMemHandle(&ptr, hq, cudaIpcMemLazyEnablePeerAccess));
            bases[q] = static_cast<char *>(ptr);
            D.peer_slabs.push_back(bases[q]);
        }
        D.d_base = D.alloc_n<char *>(nr);
        CUDA_OK(cudaMemcpy(D.d_base, bases.data(), sizeof(char *) * nr, cudaMemcpyHostToDevice));
    }
    // 2. every rank's ghost layout of every distributed operator: {lo_base, hi_base, nlo, recv_off[0..nr)}
    const size_t per = (size_t)nr + 3, stride = per * 3 * (size_t)(ld + 1);
    std::vector<int64_t> mine(stride, 0);
    for (int l = 0; l <= ld; l++) {
        const DCsr *ops[3] = {&D.lev[l].K, &D.lev[l].R, &D.lev[l].P};
        const LocalOp *lops[3] = {&plan.lev[l].K, &plan.lev[l].R, &plan.lev[l].P};
        for (int k = 0; k < 3; k++) {
            int64_t *m = mine.data() + ((size_t)l * 3 + k) * per;
            if (!ops[k]->halo) continue;
            m[0] = ops[k]->lo_base;
            m[1] = ops[k]->hi_base;
            m[2] = ops[k]->nlo;
            for (int q = 0; q < nr; q++) m[3 + q] = lops[k]->recv_off[q];
        }
    }
    const std::vector<int64_t> meta = nccl_allgather_i64(D, mine);
    for (int l = 0; l <= ld; l++) {
        DCsr *ops[3] = {&D.lev[l].K, &D.lev[l].R, &D.lev[l].P};
        const LocalOp *lops[3] = {&plan.lev[l].K, &plan.lev[l].R, &plan.lev[l].P};
        for (int k = 0; k < 3; k++) {
            if (k > 0 && l + 1 >= D.nlevels) continue;
            ops[k]->part = true;
            if (ops[k]->halo) build_push(D, *lops[k], *ops[k], meta, stride, ((size_t)l * 3 + k) * per);
        }
    }
    // 3. wait masks: the kernels of level l gather from / push to the ranks of K_l, R_l, P̄_l, P̄_{l−1}
    //    and K_{l+1} (restriction pushes d0 of the coarse level); the last distributed level's
    //    restriction pushes to everyone
    auto recv_mask = [&](const DCsr &A) {
        unsigned m = 0;
        if (A.halo)
            for (int q = 0; q < nr; q++)
                if (A.hr_count[q] > 0) m |= 1u << q;
        return m;
    };
    for (int l = 0; l <= ld; l++) {
        unsigned m = 1u << me;
        const DCsr *ops[5] = {&D.lev[l].K, &D.lev[l].R, &D.lev[l].P, l > 0 ? &D.lev[l - 1].P : nullptr,
                              (l + 1 <= ld) ? &D.lev[l + 1].K : nullptr};
        for (const DCsr *A : ops)
            if (A) m |= recv_mask(*A) | A->pmask;
        if (const char *e = std::getenv("AMG_P2P_MASK"))  // 0: wait for every rank (debug)
            if (std::atoi(e) == 0) m = ~0u;
        D.lev[l].K.wmask = D.lev[l].P.wmask = m;
        D.lev[l].R.wmask = (l == ld) ? ~0u : m;
    }
    // boundary rows (touch a ghost value or are pushed somewhere) of every distributed operator; the
    // CSR cores run the other row groups before waiting for any peer.  The ghost-reading rows were
    // marked at upload (DCsr::ghostrow; the host operators may be gone by now)
    auto ghost_rows = [&](const LocalOp &, std::vector<char> &b, const DCsr &A) { b = A.ghostrow; };
    auto add_pushed = [](std::vector<char> &b, const DCsr *A) {
        if (!A) return;
        for (size_t i = 0; i < A->pushed.size() && i < b.size(); i++) b[i] |= A->pushed[i];
    };
    for (int l = 0; l <= ld; l++) {
        DLevel &L = D.lev[l];
        const DCsr *Pab = l > 0 ? &D.lev[l - 1].P : nullptr;
        ghost_rows(plan.lev[l].K, L.K.bnd, L.K);
        add_pushed(L.K.bnd, &L.K);
        add_pushed(L.K.bnd, &L.R);
        add_pushed(L.K.bnd, Pab);
        build_gorder(D, L.K);
        if (l + 1 < D.nlevels) {
            ghost_rows(plan.lev[l].P, L.P.bnd, L.P);
            add_pushed(L.P.bnd, &L.K);
            build_gorder(D, L.P);
            ghost_rows(plan.lev[l].R, L.R.bnd, L.R);
            if (l == ld) std::fill(L.R.bnd.begin(), L.R.bnd.end(), 1);  // all-gather: every row pushed
            else add_pushed(L.R.bnd, &D.lev[l + 1].K);
            build_gorder(D, L.R);
        }
    }
    // 4. all-gather push of the first replicated level's right-hand side: my coarse rows to every rank
    if (ld + 1 < D.nlevels) {
        const std::vector<int64_t> &bd = plan.lev[ld + 1].bounds;
        const int64_t n = bd[me + 1] - bd[me];
        D.ag_row0 = bd[me];
        std::vector<int> ptr(n + 1);
        std::vector<int2> dst;
        for (int64_t i = 0; i < n; i++) {
            ptr[i] = (int)dst.size();
            for (int q = 0; q < nr; q++)
                if (q != me) dst.push_back(make_int2(q, (int)(bd[me] + i)));
        }
        ptr[n] = (int)dst.size();
        D.ag_ptr = D.alloc_n<int>(n + 1);
        D.ag_dst = D.alloc_n<int2>((int64_t)dst.size());
        CUDA_OK(cudaMemcpy(D.ag_ptr, ptr.data(), sizeof(int) * (n + 1), cudaMemcpyHostToDevice));
        if (!dst.empty()) CUDA_OK(cudaMemcpy(D.ag_dst, dst.data(), sizeof(int2) * dst.size(), cudaMemcpyHostToDevice));
    }
    // 5. the transport descriptor
    D.pp.nranks = nr;
    D.pp.rank = me;
    D.pp.base = D.d_base;
    D.pp.flags = reinterpret_cast<unsigned long long *>(D.slab + kFlagsOff);
    D.pp.epoch = reinterpret_cast<unsigned long long *>(D.slab + kEpochOff);
    D.pp.ticket = reinterpret_cast<unsigned *>(D.slab + kTicketOff);
    D.pp.bticket = reinterpret_cast<unsigned *>(D.slab + kBTicketOff);
    D.pp.flags_off = (long long)kFlagsOff;
    D.pp.dslot_off = (long long)kDslotOff;
    D.pp.wait_mask = ~0u;
    D.pp.spin_max = 1ll << 26;
    if (const char *sm = std::getenv("AMG_P2P_SPIN_MAX")) {
        const long long v = std::atoll(sm);
        if (v > 0) D.pp.spin_max = v;
    }
    // every rank has mapped every slab before any kernel may store into one
    std::vector<int64_t> one(1, 1);
    (void)nccl_allgather_i64(D, one);
    D.p2p = true;
}
}  // namespace

DevState *dev_create(const HHierarchy &H, const amg_dist *dist, const DistPlan *planp,
                     const std::function<void()> &release) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw Error{AMG_ENODEV, "no CUDA device"};
    if (dist && (dist->nranks < 1 || dist->rank < 0 || dist->rank >= dist->nranks))
        throw Error{AMG_EINVAL, "bad amg_dist (rank/nranks)"};
    auto D = new DevState();
    // env AMG_VERBOSE=1: setup phase times on stderr
    const bool verbose = std::getenv("AMG_VERBOSE") && std::atoi(std::getenv("AMG_VERBOSE")) != 0;
    auto t_start = std::chrono::steady_clock::now();
    auto lap = [&](const char *what) {
        if (!verbose) return;
        const auto t = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[amg rank %d] %s %.3f s\n", dist ? dist->rank : 0, what,
                     std::chrono::duration<double>(t - t_start).count());
        t_start = t;
    };
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
        D->krylov = H.prm.krylov;
        D->coarse_solver = H.prm.coarse_solver;
        D->coarse_tol = H.prm.coarse_tol;
        D->coarse_maxit = H.prm.coarse_maxit;
        if (const char *e = std::getenv("AMG_GRAPHS")) D->graphs = std::atoi(e) != 0;
        if (const char *e = std::getenv("AMG_DEVICE_LOOP")) D->dev_loop = std::atoi(e) != 0;
        if (const char *e = std::getenv("AMG_PROF_LEVELS")) D->lvl_prof = std::atoi(e) != 0 && !D->graphs;
        const int nr = dist ? dist->nranks : 1;
        D->rank = dist ? dist->rank : 0;
        D->nranks = nr;
        if (nr > 1 && (!planp || planp->nranks != nr)) throw Error{AMG_EINVAL, "missing distribution plan"};
        const DistPlan &plan = *planp;
        D->last_dist = nr > 1 ? plan.last_dist : H.nlevels - 1;
        const int fmt = H.prm.format;
        std::vector<int64_t> vlo(H.nlevels, 0), vhi(H.nlevels, 0);  // ghost extents of the level vectors
        for (int l = 0; l < H.nlevels; l++) {
            const HLevel &h = H.lev[l];
            DLevel &L = D->lev[l];
            L.N = h.N;
            L.nnz = level_nnz_K(H, l);
            const bool coarsest = (l + 1 == H.nlevels);
            L.replicated = nr > 1 && l > D->last_dist;
            int64_t r0 = 0;
            if (nr > 1 && !L.replicated) {
                const DistLevel &P = plan.lev[l];
                r0 = P.K.row_begin;
                L.n = P.K.row_end - P.K.row_begin;
                // rows that read a ghost column (the P2P boundary rows, p2p_setup), taken from the host
                // operators now: they may be released before p2p_setup runs
                auto ghost_rows = [](const LocalOp &op, std::vector<char> &b) {
                    const int64_t nown = op.col_end - op.col_begin;
                    b.assign(op.A.nrows, 0);
                    if (op.full_cols) return;
                    for (int64_t i = 0; i < op.A.nrows; i++)
                        for (int64_t k = op.A.rp[i]; k < op.A.rp[i + 1] && !b[i]; k++)
                            b[i] = op.A.ci[k] < 0 || op.A.ci[k] >= nown;
                };
                upload_local(*D, P.K, L.K, fmt, 0);
                ghost_rows(P.K, L.K.ghostrow);
                if (!coarsest) {
                    // P̄_l's ghosts of the coarse x lie beyond K_{l+1}'s on both sides
                    const LocalOp &Kc = plan.lev[l + 1].K;
                    const bool next_dist = !plan.lev[l + 1].replicated;
                    const int64_t klo = next_dist ? Kc.nlo : 0, khi = next_dist ? (int64_t)Kc.ghost.size() - Kc.nlo : 0;
                    upload_local(*D, P.P, L.P, fmt, 1, klo, khi);
                    upload_local(*D, P.R, L.R, fmt, 2);
                    ghost_rows(P.P, L.P.ghostrow);
                    ghost_rows(P.R, L.R.ghostrow);
                }
            } else {
                L.n = h.N;
                upload_op(*D, h.K, L.K, true, fmt, coarsest, 0);
                if (!coarsest) {
                    upload_op(*D, h.P, L.P, false, fmt, false, 1);
                    upload_op(*D, h.R, L.R, false, fmt, false, 2);
                }
            }
            if (coarsest) {  // diag(K_L) for the §5.1 coarse CG (the coarsest level is whole on every rank)
                Buf<double> dg(h.N);
                for (int64_t i = 0; i < h.N; i++) {
                    dg[i] = 0.0;
                    for (int64_t k = h.K.rp[i]; k < h.K.rp[i + 1]; k++)
                        if (h.K.ci[k] == i) dg[i] = h.K.v[k];
                }
                L.diag = D->alloc_n<double>(h.N);
                CUDA_OK(cudaMemcpy(L.diag, dg.data(), sizeof(double) * h.N, cudaMemcpyHostToDevice));
            }
            Buf<double> invd(L.n);
            for (int64_t i = 0; i < L.n; i++) invd[i] = 1.0 / h.dhat[r0 + i];
            L.invd = D->alloc_n<double>(L.n);
            CUDA_OK(cudaMemcpy(L.invd, invd.data(), sizeof(double) * L.n, cudaMemcpyHostToDevice));
            // ghost extents below / above the owned block over the gatherers of the level's vectors:
            // K_l (d, x), P̄_{l-1} (x, beyond K_l's ghosts) and R_l (r)
            const DCsr *gathers[3] = {&L.K, &L.R, l > 0 ? &D->lev[l - 1].P : nullptr};
            for (const DCsr *A : gathers) {
                if (!A || !A->halo) continue;
                vlo[l] = std::max(vlo[l], -A->lo_base);
                vhi[l] = std::max(vhi[l], A->hi_base - A->nown + (A->nghost - A->nlo));
            }
        }
        // every operator is on the device: the host copies may go (share-built hierarchies), then the
        // collectives — NCCL init and the transport decision — with nothing large held while waiting
        if (release) release();
        if (nr > 1) {
            ncclUniqueId id;
            static_assert(sizeof(id) == sizeof(dist->nccl_id), "ncclUniqueId size");
            std::memcpy(&id, dist->nccl_id, sizeof(id));
            NCCL_OK(ncclCommInitRank(&D->comm, nr, id, D->rank));
        }
        // transport: P2P peer memory (default) unless AMG_TRANSPORT=nccl, a degree-1 smoother, or a rank
        // that cannot map its peers — decided collectively so every rank uses the same one
        bool want_p2p = false;
        if (nr > 1) {
            int ok = 1;
            if (const char *e = std::getenv("AMG_TRANSPORT")) ok = std::strcmp(e, "nccl") != 0;
            if (H.prm.cheb_degree < 2 || nr > 32) ok = 0;  // wait masks are 32-bit
            for (int q = 0; q < ndev && ok; q++) {
                if (q == dev_id) continue;
                int can = 0;
                if (cudaDeviceCanAccessPeer(&can, dev_id, q) != cudaSuccess || !can) ok = 0;
            }
            std::vector<int64_t> v(1, ok);
            const std::vector<int64_t> all = nccl_allgather_i64(*D, v);
            want_p2p = true;
            for (int q = 0; q < nr; q++) want_p2p = want_p2p && all[q] != 0;
        }
        const int64_t n00 = D->lev[0].n;
        // level vectors b, x, r, d0, d1 and the PCG r, z, p, q: in the P2P slab (same offsets on every
        // rank: capacities are maxima over ranks) or from the allocator
        {
            // (lower extent, owned + upper extent) per vector group: every level, then the PCG vectors
            // (r, q: no ghosts; z, p: gathered by K_0)
            std::vector<int64_t> want;
            for (int l = 0; l < H.nlevels; l++) {
                want.push_back(vlo[l]);
                want.push_back(D->lev[l].n + vhi[l]);
            }
            want.push_back(0);
            want.push_back(n00);
            const DCsr &K0 = D->lev[0].K;
            want.push_back(K0.halo ? -K0.lo_base : 0);
            want.push_back(n00 + (K0.halo ? K0.hi_base - K0.nown + (K0.nghost - K0.nlo) : 0));
            if (want_p2p) {  // identical offsets on every rank: maxima over ranks
                const std::vector<int64_t> all = nccl_allgather_i64(*D, want);
                for (size_t k = 0; k < want.size(); k++)
                    for (int q = 0; q < nr; q++) want[k] = std::max(want[k], all[(size_t)q * want.size() + k]);
                size_t bytes = kVecOff;
                auto add = [&](int64_t lo, int64_t rest) {
                    lo = (lo + 1) & ~(int64_t)1;  // as vec() below
                    bytes += ((size_t)std::max<int64_t>(lo + rest, 1) * 8 + 255) / 256 * 256;
                };
                for (int l = 0; l < H.nlevels; l++)
                    for (int k = 0; k < 5; k++) add(want[2 * l], want[2 * l + 1]);
                const size_t g = 2 * (size_t)H.nlevels;
                for (int k = 0; k < 2; k++) add(want[g], want[g + 1]);
                for (int k = 0; k < 2; k++) add(want[g + 2], want[g + 3]);
                CUDA_OK(cudaMalloc(&D->slab, bytes));
                CUDA_OK(cudaMemset(D->slab, 0, bytes));
                D->slab_bytes = bytes;
                D->slab_used = kVecOff;
            }
            // a vector with `lo` ghost slots below its owned block: the returned pointer is owned[0],
            // 16-B aligned (lo rounded up to even; the capacities are maxima over ranks, so the
            // rounding keeps the slab offsets identical on every rank)
            auto vec = [&](int64_t lo, int64_t rest) -> double * {
                lo = (lo + 1) & ~(int64_t)1;
                double *p;
                if (!want_p2p) {
                    p = D->alloc_n<double>(lo + rest);
                } else {
                    p = reinterpret_cast<double *>(D->slab + D->slab_used);
                    D->slab_used += ((size_t)std::max<int64_t>(lo + rest, 1) * 8 + 255) / 256 * 256;
                }
                return p + lo;
            };
            for (int l = 0; l < H.nlevels; l++) {
                DLevel &L = D->lev[l];
                const int64_t lo = want[2 * l], rest = want[2 * l + 1];
                L.b = vec(lo, rest);
                L.x = vec(lo, rest);
                L.r = vec(lo, rest);
                L.d[0] = vec(lo, rest);
                L.d[1] = vec(lo, rest);
            }
            const size_t g = 2 * (size_t)H.nlevels;
            D->r = vec(want[g], want[g + 1]);
            D->q = vec(want[g], want[g + 1]);
            D->z = vec(want[g + 2], want[g + 3]);
            D->p = vec(want[g + 2], want[g + 3]);
        }
        const HLevel &hl = H.lev[H.nlevels - 1];
        if (hl.N > 6144) throw Error{AMG_EINVAL, "coarsest level larger than 6144 rows (raise max_levels)"};
        if (nr > 1) {
            const int lr = D->last_dist + 1;  // first replicated level
            const std::vector<int64_t> &bd = plan.lev[lr].bounds;
            for (int q = 0; q < nr; q++) D->ag_stride = std::max(D->ag_stride, bd[q + 1] - bd[q]);
            D->ag_send = D->alloc_n<double>(D->ag_stride);
            D->ag_recv = D->alloc_n<double>(D->ag_stride * nr);
            D->ag_bounds = D->alloc_n<int64_t>(nr + 1);
            CUDA_OK(cudaMemcpy(D->ag_bounds, bd.data(), sizeof(int64_t) * (nr + 1), cudaMemcpyHostToDevice));
            D->row_begin0 = plan.lev[0].K.row_begin;
            D->row_end0 = plan.lev[0].K.row_end;
        } else {
            D->row_begin0 = 0;
            D->row_end0 = H.lev[0].N;
        }
        const int64_t n0 = D->lev[0].n;
        D->partials = D->alloc_n<double>(D->nsm * 64 + 64);  // 2 dots x any resident grid (<= 32 CTAs per SM)
        D->counter = D->alloc_n<unsigned>(4);
        D->S = D->alloc_n<dev::Scalars>(1);
        CUDA_OK(cudaMemset(D->counter, 0, 4 * sizeof(unsigned)));
        CUDA_OK(cudaMemset(D->S, 0, sizeof(dev::Scalars)));
        CUDA_OK(cudaMallocHost(&D->hS, sizeof(dev::Scalars)));
        // operators whose streams fit in L2 may keep the normal L2 priority (env AMG_L2_KEEP_MB MB,
        // default 0 = off), so that their 2m+1 applications per V-cycle read from L2
        {
            double keep_mb = 0.0;  // off: measured no gain at C3 level 2 (110 MB, run 41)
            if (const char *e = std::getenv("AMG_L2_KEEP_MB")) keep_mb = std::atof(e);
            for (int l = 0; l < D->nlevels; l++)
                for (DCsr *A : {&D->lev[l].K, &D->lev[l].P, &D->lev[l].R})
                    A->l2keep = A->fmt == 0 && A->nnz > 0 && 10.0 * (double)A->nnz <= keep_mb * 1e6;
        }
        lap("upload");
        if (fmt == 0) {  // autotune every large operator on scratch vectors
            int64_t big = 1, lomax = 0;
            for (int l = 0; l < D->nlevels; l++)
                for (const DCsr *A : {&D->lev[l].K, &D->lev[l].P, &D->lev[l].R}) {
                    big = std::max(big, std::max(A->nrows, A->ncols));
                    if (A->halo) lomax = std::max(lomax, -A->lo_base);
                }
            lomax = (lomax + 1) & ~(int64_t)1;  // keep sx 16-B aligned (the windowed SELL-VI copies)
            double *scr = nullptr;  // x (with room for negative ghost columns), y1, y2, y3 scratch vectors
            CUDA_OK(cudaMalloc(&scr, sizeof(double) * (big * 4 + lomax)));
            // non-trivial data (not zeros): data-dependent power draw changes the clocks under the cap
            dev::k_fill_pattern<<<grid_for(*D, big * 4 + lomax), dev::kBlock>>>(big * 4 + lomax, scr);
            CUDA_OK(cudaGetLastError());
            double *sx = scr + lomax, *y1 = sx + big, *y2 = sx + 2 * big, *y3 = sx + 3 * big;
            // a rank whose autotuning fails must not leave the others waiting in the NCCL collectives
            // of the P2P setup: the ranks agree on the outcome first and all fail together
            Error failed{AMG_OK, ""};
            try {
                for (int l = 0; l < D->nlevels; l++) {
                    autotune_op(*D, D->lev[l].K, l, 0, sx, y1, y2, y3);
                    if (l + 1 < D->nlevels) {
                        autotune_op(*D, D->lev[l].P, l, 1, sx, y1, y2, y3);
                        autotune_op(*D, D->lev[l].R, l, 2, sx, y1, y2, y3);
                    }
                }
            } catch (const Error &e) {
                failed = e;
            } catch (...) {
                failed = Error{AMG_ECUDA, "autotuning failed"};
            }
            cudaFree(scr);
            if (want_p2p) {
                const std::vector<int64_t> all = nccl_allgather_i64(*D, std::vector<int64_t>(1, failed.st != AMG_OK));
                for (int q = 0; q < nr && failed.st == AMG_OK; q++)
                    if (all[q]) failed = Error{AMG_EINVAL, "setup failed on rank " + std::to_string(q)};
            }
            if (failed.st != AMG_OK) throw failed;
        }
        // dominant kernel (level-0 fused Chebyshev step): the operator's streamed bytes in its chosen
        // format + 56 B/row of vectors (d_old, r in/out, x in/out, invd, d_new)
        D->bytes_dominant = D->lev[0].K.alg_bytes() + 56.0 * (double)n0;
        CUDA_OK(cudaDeviceSynchronize());
        lap("autotune");
        if (want_p2p) p2p_setup(*D, plan);
        lap("p2p_setup");
    } catch (...) {
        delete D;
        throw;
    }
    return D;
}

void dev_destroy(DevState *D) { delete D; }

// Fold the elapsed times of the event pairs recorded since the last collection into the profile.
static void prof_collect(DevState &D, size_t ev0 = 0, size_t ev1 = (size_t)-1, bool reset = true) {
    if (ev1 == (size_t)-1) ev1 = D.ev_used;
    for (size_t k = ev0; k + 1 < ev1; k += 2) {
        float ms = 0.f;
        CUDA_OK(cudaEventElapsedTime(&ms, D.ev[k], D.ev[k + 1]));
        D.prof_ms += ms;
        D.prof_n++;
    }
    if (reset) D.ev_used = 0;
}

// Every captured graph (per-iteration segments, the device loop): dropped when a launch
// configuration changes.
void drop_graphs(DevState &D) {
    for (auto &sg : D.seg)
        if (sg.exec) {
            cudaGraphExecDestroy(sg.exec);
            sg.exec = nullptr;
        }
    if (D.loop.exec) {
        cudaGraphExecDestroy(D.loop.exec);
        D.loop.exec = nullptr;
    }
}

// One PCG iteration on the device: z = V(r) with ρ = rᵀz (kind 0: initial, 1: with β), p = z + βp,
// q = Kp with α = ρ/pᵀq, u += αp, r −= αq, ‖r‖², and the 64-byte scalar block copied to pinned host
// memory.  No host decision inside, so it is captured once into a CUDA graph and replayed.  In the
// device loop (ctl != nullptr) the first-iteration choice is read from the loop control and the scalars
// stay on the device.
static void enqueue_segment(DevState &D, int kind, double *u, cudaStream_t st, dev::LoopCtl *ctl = nullptr) {
    DLevel &L0 = D.lev[0];
    const int64_t n = L0.n;
    const int flex = D.krylov == 1;
    if (flex) vcycle(D, D.r, D.z, st, dev::DOT_ZQ, D.q);  // FCG: zᵀq_prev (all-reduced)
    else vcycle(D, D.r, D.z, st, dev::DOT_RZ);            // CG: ρ = rᵀz (all-reduced)
    launch_k(dev::k_p_update, grid_for(D, n), dev::kBlock, 0, st, n, D.z, D.p, D.S, kind == 0 ? 1 : 0, flex,
                                                           push_of(D, L0.K, D.p), p2p_of(D, L0.K), ctl);
    launch_k(dev::k_roll_rho, 1, 1, 0, st, D.S);
    D.launches_total += 2;
    {
        halo(D, L0.K, D.p, st);
        if (flex) {  // FCG: pᵀq and pᵀr in one pass
            dev::EpiSpmvDot2 e{D.p, D.r, D.q};
            launch_csr(D, L0.K, D.p, e, st, dev::DOT_PQ | (dev::DOT_PR << 8));
            allreduce_dot(D, dev::DOT_PQ | (dev::DOT_PR << 8), st);
        } else {
            dev::EpiSpmvDot e{D.p, D.q};
            launch_csr(D, L0.K, D.p, e, st, dev::DOT_PQ);
            allreduce_dot(D, dev::DOT_PQ, st);
        }
    }
    launch_k(dev::k_pcg_update, grid_for(D, n), dev::kBlock, 0, st, n, D.p, D.q, u, D.r, dotctx(D, dev::DOT_RR), flex);
    D.launches_total++;
    allreduce_dot(D, dev::DOT_RR, st);
    CUDA_OK(cudaGetLastError());
    if (!ctl) CUDA_OK(cudaMemcpyAsync(D.hS, D.S, sizeof(dev::Scalars), cudaMemcpyDeviceToHost, st));
}

// The whole iteration loop as ONE graph launch: a conditional WHILE node (default 1, re-armed at every
// launch) whose body is one iteration (enqueue_segment with the device loop control) followed by
// k_loop_ctl, which counts, records ‖r_k‖/‖F‖ and clears the condition on convergence, breakdown or
// maxit.  No host round trip per iteration (the paper names launch latency as what
// dominates at small local sizes).
static void run_device_loop(DevState &D, double *u, cudaStream_t st) {
    if (!D.loop.exec || D.loop.u != u) {
        if (D.loop.exec) {
            cudaGraphExecDestroy(D.loop.exec);
            D.loop.exec = nullptr;
        }
        if (!D.cap) CUDA_OK(cudaStreamCreateWithFlags(&D.cap, cudaStreamNonBlocking));
        cudaGraph_t g = nullptr;
        CUDA_OK(cudaGraphCreate(&g, 0));
        try {
            cudaGraphConditionalHandle h;
            CUDA_OK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            CUDA_OK(cudaGraphAddNode(&node, g, nullptr, 0, &cp));
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            const int64_t nk0 = D.launches_total;
            CUDA_OK(cudaStreamBeginCaptureToGraph(D.cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            try {
                enqueue_segment(D, 1, u, D.cap, D.ctl);
                launch_k(dev::k_loop_ctl, 1, 1, 0, D.cap, D.S, D.ctl, D.krylov == 1 ? 1 : 0, h);
                CUDA_OK(cudaGetLastError());
            } catch (...) {
                cudaGraph_t gb;
                cudaStreamEndCapture(D.cap, &gb);
                throw;
            }
            cudaGraph_t gb;
            CUDA_OK(cudaStreamEndCapture(D.cap, &gb));
            D.loop.nk = D.launches_total - nk0 + 1;
            D.launches_total = nk0;
            CUDA_OK(cudaGraphInstantiate(&D.loop.exec, g, 0));
        } catch (...) {
            cudaGraphDestroy(g);
            throw;
        }
        CUDA_OK(cudaGraphDestroy(g));
        D.loop.u = u;
    }
    CUDA_OK(cudaGraphLaunch(D.loop.exec, st));
}

static void run_segment(DevState &D, int kind, double *u, cudaStream_t st) {
    if (!D.graphs) {
        enqueue_segment(D, kind, u, st);
        CUDA_OK(cudaStreamSynchronize(st));
        prof_collect(D);
        level_collect(D);
        return;
    }
    DevState::Seg &S = D.seg[kind];
    if (!S.exec || S.u != u || S.prof != D.prof) {
        if (S.exec) {
            cudaGraphExecDestroy(S.exec);
            S.exec = nullptr;
        }
        if (!D.cap) CUDA_OK(cudaStreamCreateWithFlags(&D.cap, cudaStreamNonBlocking));
        // events of this graph live at a fixed index range of D.ev
        S.ev0 = D.ev_used = (kind == 0 ? 0 : 512);
        if (D.ev.size() < 1024)
            while (D.ev.size() < 1024) {
                cudaEvent_t e;
                CUDA_OK(cudaEventCreate(&e));
                D.ev.push_back(e);
            }
        const int64_t nk0 = D.launches_total;
        CUDA_OK(cudaStreamBeginCapture(D.cap, cudaStreamCaptureModeThreadLocal));
        try {
            enqueue_segment(D, kind, u, D.cap);
        } catch (...) {
            cudaGraph_t g;
            cudaStreamEndCapture(D.cap, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g;
        CUDA_OK(cudaStreamEndCapture(D.cap, &g));
        CUDA_OK(cudaGraphInstantiate(&S.exec, g, 0));
        CUDA_OK(cudaGraphDestroy(g));
        S.nk = D.launches_total - nk0;
        D.launches_total = nk0;
        S.ev1 = D.ev_used;
        S.u = u;
        S.prof = D.prof;
        D.ev_used = 0;
    }
    CUDA_OK(cudaGraphLaunch(S.exec, st));
    D.launches_total += S.nk;
    CUDA_OK(cudaStreamSynchronize(st));
    if (D.prof) prof_collect(D, S.ev0, S.ev1, false);
}

// c.19 — PCG.  F, u: device pointers of length N_0.
static amg_status pcg(DevState &D, const double *F, double *u, double rtol, int maxit, cudaStream_t st, int *iters,
                      double *relres, double *hist) {
    DLevel &L0 = D.lev[0];
    const int64_t N = L0.n;  // this rank's rows
    *iters = 0;
    *relres = 0.0;
    CUDA_OK(cudaMemsetAsync(D.S, 0, sizeof(dev::Scalars), st));
    // ‖F‖²
    launch_k(dev::k_dot, grid_for(D, N), dev::kBlock, 0, st, N, F, F, dotctx(D, dev::DOT_FF));
    D.launches_total++;
    allreduce_dot(D, dev::DOT_FF, st);
    // r = F − K u ; ‖r‖²   (u is copied into z, which has the ghost slots K_0 gathers)
    {
        if (D.p2p) {
            launch_k(dev::k_copy_push, grid_for(D, N), dev::kBlock, 0, st, N, u, D.z, push_of(D, L0.K, D.z), p2p_of(D, L0.K));
            D.launches_total++;
        } else {
            CUDA_OK(cudaMemcpyAsync(D.z, u, sizeof(double) * N, cudaMemcpyDeviceToDevice, st));
        }
        halo(D, L0.K, D.z, st);
        dev::EpiResidualFrom e{F, D.r, nullptr, nullptr};
        launch_csr(D, L0.K, D.z, e, st);
    }
    launch_k(dev::k_dot, grid_for(D, N), dev::kBlock, 0, st, N, D.r, D.r, dotctx(D, dev::DOT_RR));
    D.launches_total++;
    allreduce_dot(D, dev::DOT_RR, st);
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
    prof_collect(D);
    amg_status status = AMG_NOT_CONVERGED;
    // device loop: graphs on, no per-kernel profiling events, one GPU or the P2P transport (NCCL calls
    // stay out of conditional bodies)
    if (maxit > 0 && D.graphs && D.dev_loop && !D.prof && !D.lvl_prof && (D.nranks <= 1 || D.p2p)) {
        if (D.hist_cap < maxit + 1) {
            D.hist_cap = std::max(maxit + 1, 256);
            D.dhist = D.alloc_n<double>(D.hist_cap);
        }
        if (!D.ctl) {
            D.ctl = D.alloc_n<dev::LoopCtl>(1);
            CUDA_OK(cudaMallocHost(&D.hctl, sizeof(dev::LoopCtl)));
        }
        *D.hctl = dev::LoopCtl{0, maxit, 1, 1, nF, rtol * nF, D.dhist};
        CUDA_OK(cudaMemcpyAsync(D.ctl, D.hctl, sizeof(dev::LoopCtl), cudaMemcpyHostToDevice, st));
        run_device_loop(D, u, st);
        CUDA_OK(cudaMemcpyAsync(D.hctl, D.ctl, sizeof(dev::LoopCtl), cudaMemcpyDeviceToHost, st));
        std::vector<double> hh;
        if (hist) {
            hh.resize(maxit + 1);
            CUDA_OK(cudaMemcpyAsync(hh.data(), D.dhist, sizeof(double) * (maxit + 1), cudaMemcpyDeviceToHost, st));
        }
        CUDA_OK(cudaStreamSynchronize(st));
        const int k = D.hctl->k;
        const bool brk = D.hctl->status == -5;
        const int kl = brk ? k - 1 : k;  // the last iteration whose residual was recorded
        D.launches_total += D.loop.nk * k;
        *iters = k;
        if (kl >= 1) CUDA_OK(cudaMemcpy(relres, D.dhist + kl, sizeof(double), cudaMemcpyDeviceToHost));
        if (hist)
            for (int j = 1; j <= kl; j++) hist[j] = hh[j];
        return brk ? AMG_ENOTSPD : D.hctl->status == 0 ? AMG_OK : AMG_NOT_CONVERGED;
    }
    for (int k = 1; k <= maxit; k++) {
        // iteration k: [z = V(r); ρ = rᵀz; p = z + βp] then q = Kp, α, u += αp, r −= αq, ‖r‖²
        run_segment(D, k == 1 ? 0 : 1, u, st);
        if ((D.krylov == 0 && !(D.hS->rz > 0.0)) || !(D.hS->pq > 0.0)) {  // breakdown: rᵀz <= 0 (CG) or pᵀKp <= 0
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
    const int64_t N = D->lev[0].n;  // this rank's rows
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
    cudaStream_t st = (cudaStream_t)stream;
    if (D->nranks > 1) {  // gathered x needs ghost slots (and P2P pushes address slab vectors): run
                          // on the PCG's r/z and copy in/out
        const size_t bytes = sizeof(double) * (size_t)D->lev[0].n;
        CUDA_OK(cudaMemcpyAsync(D->r, r, bytes, cudaMemcpyDeviceToDevice, st));
        vcycle(*D, D->r, D->z, st, dev::DOT_NONE);
        CUDA_OK(cudaMemcpyAsync(z, D->z, bytes, cudaMemcpyDeviceToDevice, st));
    } else {
        vcycle(*D, r, z, st, dev::DOT_NONE);
    }
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
    if (A.halo) throw Error{AMG_EINVAL, "amg_level_apply: operator is distributed (use a single-GPU hierarchy)"};
    dev::EpiStore e{y};
    launch_csr(*D, A, x, e, (cudaStream_t)stream);
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_nccl_unique_id(unsigned char id[128]) {
    API_BEGIN
    if (!id) throw Error{AMG_EINVAL, "NULL id"};
    ncclUniqueId u;
    NCCL_OK(ncclGetUniqueId(&u));
    std::memcpy(id, &u, sizeof(u));
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_local_rows(amg_hierarchy *H, int64_t *row_begin, int64_t *row_end) {
    API_BEGIN
    if (!H || !row_begin || !row_end) throw Error{AMG_EINVAL, "NULL argument"};
    if (H->distributed) {  // host plan (also for host_only setups)
        *row_begin = H->plan.lev[0].K.row_begin;
        *row_end = H->plan.lev[0].K.row_end;
    } else {
        *row_begin = 0;
        *row_end = H->host.lev[0].N;
    }
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
    D->prof_ms = 0.0;
    D->prof_n = 0;
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_get_kernel_stats(amg_hierarchy *H, amg_kernel_stats *st) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!st) throw Error{AMG_EINVAL, "NULL stats"};
    CUDA_OK(cudaDeviceSynchronize());
    if (!D->graphs) prof_collect(*D);  // pairs recorded outside PCG (e.g. amg_vcycle)
    st->launches = D->prof_n;
    st->total_ms = D->prof_ms;
    st->bytes_per_launch = D->bytes_dominant;
    st->kernels_launched = D->launches_total;
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_get_level_times(amg_hierarchy *H, double *ms_per_vcycle, int nmax, int *nlevels) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!ms_per_vcycle || !nlevels || nmax < 1) throw Error{AMG_EINVAL, "bad argument"};
    CUDA_OK(cudaDeviceSynchronize());
    level_collect(*D);
    *nlevels = D->nlevels;
    for (int l = 0; l < std::min(nmax, D->nlevels); l++)
        ms_per_vcycle[l] = D->lvl_vcycles ? D->lvl_ms[l] / (double)D->lvl_vcycles : 0.0;
    for (int l = 0; l < 32; l++) D->lvl_ms[l] = 0.0;
    D->lvl_vcycles = 0;
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_operator_set_config(amg_hierarchy *H, int level, int op, int kernel, int G, int U) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (level < 0 || level >= D->nlevels || op < 0 || op > 2) throw Error{AMG_EINVAL, "bad level/op"};
    if (op > 0 && level == D->nlevels - 1) throw Error{AMG_EINVAL, "no transfer operator on the coarsest level"};
    DLevel &L = D->lev[level];
    DCsr &A = op == 0 ? L.K : op == 1 ? L.P : L.R;
    if (A.fmt == 2) {  // SELL-VI: only U (entries in flight per lane) is free; windowed: kernel = windows staged
        if ((A.win ? !(kernel == 1 || kernel == 2) : kernel != 0) || G != 32 || !(U == 1 || U == 2 || U == 4))
            throw Error{AMG_EINVAL, "SELL-VI operator: kernel 0 (windowed: 1 or 2), G 32 and U 1, 2 or 4"};
        CUDA_OK(cudaDeviceSynchronize());
        if (A.win && kernel == 2 &&
            8 * ((A.nvals <= kSellviSmemVals ? (A.nvals + 1) & ~1 : 0) + 2 * (int64_t)A.wmax) > 227 * 1024)
            throw Error{AMG_EINVAL, "windowed SELL-VI: two windows exceed the shared memory of a CTA"};
        A.U = U;
        if (A.win) A.nbuf = kernel;
        A.tuned_us = 0.f;
        drop_graphs(*D);
        return AMG_OK;
    }
    if (A.fmt != 0) throw Error{AMG_EINVAL, "operator is not in a CSR layout"};
    if (kernel < 0 || kernel > 15 || ((kernel & 2) && !A.off16) || ((kernel & 4) && ((kernel & 1) || A.mult < 8)) ||
        ((kernel & 8) && ((kernel & 1) || !A.vtab)))
        throw Error{AMG_EINVAL, "kernel not available for this operator"};
    if ((kernel & 1) && (A.mult < 8 || U > 4)) throw Error{AMG_EINVAL, "TMA core needs rows padded to 8 and U <= 4"};
    if (!(G == 1 || G == 2 || G == 4 || G == 8 || G == 32) || !(U == 2 || U == 4 || U == 6 || U == 8))
        throw Error{AMG_EINVAL, "G must be 1, 2, 4, 8 or 32 and U 2, 4, 6 or 8"};
    CUDA_OK(cudaDeviceSynchronize());
    A.kern = kernel & 11;
    A.pf = (kernel >> 2) & 1;
    A.G = G;
    A.U = U;
    A.tuned_us = 0.f;
    build_gorder(*D, A);
    drop_graphs(*D);  // captured graphs hold the old launch configuration
    if (level == 0 && op == 0) D->bytes_dominant = A.alg_bytes() + 56.0 * (double)L.n;
    return AMG_OK;
    API_END
}

extern "C" amg_status amg_operator_config(amg_hierarchy *H, int level, int op, amg_op_config *cfg) {
    API_BEGIN
    DevState *D = need_dev(H);
    if (!cfg || level < 0 || level >= D->nlevels || op < 0 || op > 2) throw Error{AMG_EINVAL, "bad argument"};
    if (op > 0 && level == D->nlevels - 1) throw Error{AMG_EINVAL, "no transfer operator on the coarsest level"};
    const DLevel &L = D->lev[level];
    const DCsr &A = op == 0 ? L.K : op == 1 ? L.P : L.R;
    cfg->layout = A.fmt == 2 && A.win ? 3 : A.fmt;
    cfg->kernel = A.fmt == 2 ? (A.win ? A.nbuf : 0) : A.kern | (A.pf << 2);
    cfg->G = A.G;
    cfg->U = A.U;
    cfg->stored = A.stored;
    cfg->tuned_us = A.tuned_us;
    cfg->alg_bytes = A.alg_bytes();
    cfg->nnz = A.nnz;
    cfg->n_values = A.nvals;
    cfg->value_index_bytes = !A.vtab ? 0 : (A.fmt == 2 || (A.vpk && (A.kern & 2))) ? 2 : 4;
    cfg->sellvi_parts = A.fmt == 2 ? 1 << A.lparts : 0;
    cfg->offset_bits = A.fmt == 2 ? (A.win ? A.pbits : A.obits) : 0;
    return AMG_OK;
    API_END
}
