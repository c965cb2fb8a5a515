// inst_spmv.cu — explicit instantiations of launch_csr (and so of every CSR/SELL kernel variant) for: EpiStore, EpiSpmvDot, EpiSpmvDot2, EpiResidualFrom.
#include "launch_csr.cuh"

namespace amgb {
template void launch_csr<dev::EpiStore>(DevState &, const DCsr &, const double *, dev::EpiStore, cudaStream_t, int);
template void launch_csr<dev::EpiSpmvDot>(DevState &, const DCsr &, const double *, dev::EpiSpmvDot, cudaStream_t, int);
template void launch_csr<dev::EpiSpmvDot2>(DevState &, const DCsr &, const double *, dev::EpiSpmvDot2, cudaStream_t, int);
template void launch_csr<dev::EpiResidualFrom>(DevState &, const DCsr &, const double *, dev::EpiResidualFrom, cudaStream_t, int);
}  // namespace amgb
