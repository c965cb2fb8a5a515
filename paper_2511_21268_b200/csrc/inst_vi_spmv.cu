// inst_vi_spmv.cu — explicit instantiations of the value-indexed launchers (launch_csr_vi) for the epilogues of inst_spmv.cu.
#include "launch_csr_vi.cuh"

namespace amgb {
template void launch_csr_vi<dev::EpiStore>(DevState &, const DCsr &, const double *, dev::EpiStore, cudaStream_t, int);
template void launch_csr_vi<dev::EpiSpmvDot>(DevState &, const DCsr &, const double *, dev::EpiSpmvDot, cudaStream_t, int);
template void launch_csr_vi<dev::EpiSpmvDot2>(DevState &, const DCsr &, const double *, dev::EpiSpmvDot2, cudaStream_t, int);
template void launch_csr_vi<dev::EpiResidualFrom>(DevState &, const DCsr &, const double *, dev::EpiResidualFrom, cudaStream_t, int);
template void launch_sellvi<dev::EpiStore>(DevState &, const DCsr &, const double *, dev::EpiStore, cudaStream_t, int);
template void launch_sellvi<dev::EpiSpmvDot>(DevState &, const DCsr &, const double *, dev::EpiSpmvDot, cudaStream_t, int);
template void launch_sellvi<dev::EpiSpmvDot2>(DevState &, const DCsr &, const double *, dev::EpiSpmvDot2, cudaStream_t, int);
template void launch_sellvi<dev::EpiResidualFrom>(DevState &, const DCsr &, const double *, dev::EpiResidualFrom, cudaStream_t, int);
}  // namespace amgb
