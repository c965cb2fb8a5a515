// inst_transfer.cu — explicit instantiations of launch_csr (and so of every CSR/SELL kernel variant) for: EpiPostFirst, EpiRestrict, EpiProlong.
#include "launch_csr.cuh"

namespace amgb {
template void launch_csr<dev::EpiPostFirst>(DevState &, const DCsr &, const double *, dev::EpiPostFirst, cudaStream_t, int);
template void launch_csr<dev::EpiRestrict>(DevState &, const DCsr &, const double *, dev::EpiRestrict, cudaStream_t, int);
template void launch_csr<dev::EpiProlong>(DevState &, const DCsr &, const double *, dev::EpiProlong, cudaStream_t, int);
}  // namespace amgb
