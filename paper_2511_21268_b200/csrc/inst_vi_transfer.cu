// inst_vi_transfer.cu — explicit instantiations of the value-indexed launchers (launch_csr_vi) for the epilogues of inst_transfer.cu.
#include "launch_csr_vi.cuh"

namespace amgb {
template void launch_csr_vi<dev::EpiPostFirst>(DevState &, const DCsr &, const double *, dev::EpiPostFirst, cudaStream_t, int);
template void launch_csr_vi<dev::EpiRestrict>(DevState &, const DCsr &, const double *, dev::EpiRestrict, cudaStream_t, int);
template void launch_csr_vi<dev::EpiProlong>(DevState &, const DCsr &, const double *, dev::EpiProlong, cudaStream_t, int);
template void launch_sellvi<dev::EpiPostFirst>(DevState &, const DCsr &, const double *, dev::EpiPostFirst, cudaStream_t, int);
template void launch_sellvi<dev::EpiRestrict>(DevState &, const DCsr &, const double *, dev::EpiRestrict, cudaStream_t, int);
template void launch_sellvi<dev::EpiProlong>(DevState &, const DCsr &, const double *, dev::EpiProlong, cudaStream_t, int);
}  // namespace amgb
