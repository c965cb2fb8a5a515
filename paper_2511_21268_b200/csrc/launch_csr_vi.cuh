// launch_csr_vi.cuh — the value-indexed CSR launchers (kern bit 3; CSR-VI sources of kernels.cuh),
// included only by the inst_vi_*.cu files.
#pragma once
#include "launch_csr.cuh"

namespace amgb {

template <class Epi>
void launch_csr_vi(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind) {
    if (!A.vtab || !A.vidx) throw Error{AMG_EINVAL, "operator has no value index"};
    const unsigned short *off = reinterpret_cast<const unsigned short *>(A.off16);
    if ((A.kern & 2) && A.vpk) launch_csr_cols(D, A, dev::ColsD16V16{A.vpk, A.rbase, A.vtab}, g, epi, st, dotkind);
    else if (A.kern & 2) launch_csr_cols(D, A, dev::ColsD16V32{off, A.vidx, A.rbase, A.vtab}, g, epi, st, dotkind);
    else launch_csr_cols(D, A, dev::ColsI32V32{A.ci, A.vidx, A.vtab}, g, epi, st, dotkind);
}

// Value tables of up to kSellviSmemVals entries are staged in shared memory per CTA (devstate.cuh).

template <int U, class Epi, int NBUF, bool kSmem>
void launch_sellviw(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind) {
    if (((uintptr_t)g & 15) != 0) throw Error{AMG_EINVAL, "windowed SELL-VI: the multiplied vector must be 16-B aligned"};
    const int64_t nsl = (A.nrows + 31) / 32;
    const int64_t nblk = (nsl + kWinSlices - 1) / kWinSlices;
    const int tabn = kSmem ? (int)((A.nvals + 1) & ~1) : 0;
    const int smem = 8 * (tabn + NBUF * A.wmax);
    const int per_sm = resident_ctas((const void *)dev::k_sellviw<U, Epi, NBUF, kSmem>, dev::kBlock, smem, smem);
    const int64_t nitems = A.wwhole + ((nblk - A.wwhole) << A.wl);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(nitems, (int64_t)per_sm * D.nsm));
    launch_k(dev::k_sellviw<U, Epi, NBUF, kSmem>, grid, dev::kBlock, smem, st, 
        A.soff, reinterpret_cast<const uint4 *>(A.vpk), A.binfo, A.wruns, A.vtab, (int)A.nvals, A.pbits, A.wmax, g,
        A.nrows, epi, dotctx(D, dotkind), A.wwhole, A.wl,
        (dotkind != dev::DOT_NONE ? p2p_of(D, A.part) : p2p_csr(D, A)));
}

template <int U, class Epi, bool kSmem>
void launch_sellvi_us(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind) {
    if (A.win) {
        if (A.nbuf == 1) launch_sellviw<U, Epi, 1, kSmem>(D, A, g, epi, st, dotkind);
        else launch_sellviw<U, Epi, 2, kSmem>(D, A, g, epi, st, dotkind);
        return;
    }
    const int64_t nsl = (A.nrows + 31) / 32;
    const int64_t wpb = dev::kBlock / 32;
    const int smem = kSmem ? (int)(A.nvals * 8) : 0;
    const int per_sm = resident_ctas((const void *)dev::k_sellvi<U, Epi, kSmem>, dev::kBlock, smem,
                                     kSmem ? (int)(kSellviSmemVals * 8) : 0);
    const int lparts = Epi::kDot ? 0 : A.lparts;  // dot epilogues keep whole slices (fixed dot order)
    const int64_t nwhole = lparts ? A.nwhole : nsl;
    const int64_t nitems = nwhole + ((nsl - nwhole) << lparts);
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nitems + wpb - 1) / wpb, (int64_t)per_sm * D.nsm));
    launch_k(dev::k_sellvi<U, Epi, kSmem>, grid, dev::kBlock, smem, st, 
        A.soff, reinterpret_cast<const uint4 *>(A.vpk), A.rbase, A.vtab, (int)A.nvals, A.obits, g, A.nrows, epi,
        dotctx(D, dotkind), (dotkind != dev::DOT_NONE ? p2p_of(D, A.part) : p2p_csr(D, A)),
        nwhole, lparts, A.partial, A.sticket);
}

template <int U, class Epi>
void launch_sellvi_u(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind) {
    if (A.nvals <= kSellviSmemVals) launch_sellvi_us<U, Epi, true>(D, A, g, epi, st, dotkind);
    else launch_sellvi_us<U, Epi, false>(D, A, g, epi, st, dotkind);
}

template <class Epi>
void launch_sellvi(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind) {
    switch (A.U) {
        case 1: launch_sellvi_u<1, Epi>(D, A, g, epi, st, dotkind); break;
        case 2: launch_sellvi_u<2, Epi>(D, A, g, epi, st, dotkind); break;
        case 4: launch_sellvi_u<4, Epi>(D, A, g, epi, st, dotkind); break;
        default: throw Error{AMG_EINVAL, "bad SELL-VI configuration (U must be 1, 2 or 4)"};
    }
}

}  // namespace amgb
