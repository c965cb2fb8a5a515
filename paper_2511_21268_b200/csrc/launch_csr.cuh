// launch_csr.cuh — definitions of the CSR/SELL launchers (included only by the inst_*.cu files, which
// instantiate them once per epilogue).
#pragma once
#include "devstate.cuh"

namespace amgb {

template <int G, int U, class Epi, class Cols>
void launch_csr4t_gu(DevState &D, const DCsr &A, const Cols &cols, const double *g, Epi epi, cudaStream_t st,
                     int dotkind) {
    constexpr int smem = dev::TmaCfg<U, Cols::kIdxBytes>::SMEM;
    const int64_t ngroups = (A.nrows + G - 1) / G;
    const int64_t wpb = dev::kBlockT / 32;
    const int per_sm = resident_ctas((const void *)dev::k_csr4t<G, U, Epi, Cols>, dev::kBlockT, smem, smem);
    // one wave: every CTA resident, warps stride over the row groups
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((ngroups + wpb - 1) / wpb, (int64_t)per_sm * D.nsm));
    launch_k(dev::k_csr4t<G, U, Epi, Cols>, grid, dev::kBlockT, smem, st, A.rp, cols, A.v, g, A.nrows, epi, dotctx(D, dotkind),
                                                                      (dotkind != dev::DOT_NONE ? p2p_of(D, A.part) : p2p_csr(D, A)));
}

template <int G, int U, class Epi, class Cols>
void launch_csr2_gu(DevState &D, const DCsr &A, const Cols &cols, const double *g, Epi epi, cudaStream_t st,
                    int dotkind) {
    const int64_t ngroups = (A.nrows + G - 1) / G;
    const int64_t warps_per_block = dev::kBlock / 32;
    const int per_sm = resident_ctas((const void *)dev::k_csr2<G, U, Epi, Cols>, dev::kBlock, 0);
    // one wave: every CTA resident, warps stride over the row groups
    const int grid = (int)std::max<int64_t>(
        1, std::min<int64_t>((ngroups + warps_per_block - 1) / warps_per_block, (int64_t)per_sm * D.nsm));
    launch_k(dev::k_csr2<G, U, Epi, Cols>, grid, dev::kBlock, 0, st, A.rp, cols, A.v, g, A.nrows, epi, dotctx(D, dotkind),
                                                               (dotkind != dev::DOT_NONE ? p2p_of(D, A.part) : p2p_csr(D, A)),
                                                               (A.mult >= 8 ? A.pf : 0) | (A.l2keep ? 2 : 0));
}

template <class Epi, class Cols>
void launch_csr_cols(DevState &D, const DCsr &A, const Cols &cols, const double *g, Epi epi, cudaStream_t st,
                     int dotkind) {
    const bool tma = (A.kern & 1) != 0;
    if constexpr (!Cols::kVals) {  // value-indexed sources: register core only
        if (tma) throw Error{AMG_EINVAL, "the TMA core has no value-indexed source"};
    }
    switch (A.G * 16 + A.U) {
#define CASE(GG, UU)                                                                            \
    case GG * 16 + UU:                                                                          \
        if constexpr (Cols::kVals) {                                                            \
            if (tma) launch_csr4t_gu<GG, UU, Epi, Cols>(D, A, cols, g, epi, st, dotkind);       \
            else launch_csr2_gu<GG, UU, Epi, Cols>(D, A, cols, g, epi, st, dotkind);            \
        } else {                                                                                \
            launch_csr2_gu<GG, UU, Epi, Cols>(D, A, cols, g, epi, st, dotkind);                 \
        }                                                                                       \
        break;
#define CASES_G(GG) CASE(GG, 2) CASE(GG, 4) CASE(GG, 6) CASE(GG, 8)
        CASES_G(1) CASES_G(2) CASES_G(4) CASES_G(8) CASES_G(32)
#undef CASES_G
#undef CASE
        default: throw Error{AMG_EINVAL, "bad CSR kernel configuration"};
    }
}

// Value-indexed sources (kern bit 3): defined in launch_csr_vi.cuh, compiled in their own translation
// units (inst_vi_*.cu) in parallel with the streamed-value ones.
template <class Epi>
void launch_csr_vi(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind);
template <class Epi>
void launch_sellvi(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind);

template <class Epi>
void launch_csr(DevState &D, const DCsr &A, const double *g, Epi epi, cudaStream_t st, int dotkind) {
    if (A.fmt == 2) {
        launch_sellvi(D, A, g, epi, st, dotkind);  // instantiated in inst_vi_*.cu
    } else if (A.fmt == 1) {
        const int2 *ci2 = reinterpret_cast<const int2 *>(A.ci);
        const double2 *v2 = reinterpret_cast<const double2 *>(A.v);
        const int64_t nsl = (A.nrows + 31) / 32;
        const int64_t wpb = dev::kBlock / 32;
        const int per_sm = resident_ctas((const void *)dev::k_sell2<Epi>, dev::kBlock, 0);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nsl + wpb - 1) / wpb, (int64_t)per_sm * D.nsm));
        launch_k(dev::k_sell2<Epi>, grid, dev::kBlock, 0, st, A.soff, ci2, v2, g, A.nrows, epi, dotctx(D, dotkind),
                                                         (dotkind != dev::DOT_NONE ? p2p_of(D, A.part) : p2p_of(D, A)));
    } else if (A.kern & 8) {
        launch_csr_vi(D, A, g, epi, st, dotkind);  // instantiated in inst_vi_*.cu
    } else if (A.kern & 2) {
        launch_csr_cols(D, A, dev::ColsD16{reinterpret_cast<const unsigned short *>(A.off16), A.rbase}, g, epi, st, dotkind);
    } else {
        launch_csr_cols(D, A, dev::ColsI32{A.ci}, g, epi, st, dotkind);
    }
    D.launches_total++;
    CUDA_OK(cudaGetLastError());
}

}  // namespace amgb
