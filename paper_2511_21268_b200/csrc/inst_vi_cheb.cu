// inst_vi_cheb.cu — explicit instantiations of the value-indexed launchers (launch_csr_vi) for the epilogues of inst_cheb.cu.
#include "launch_csr_vi.cuh"

namespace amgb {
template void launch_csr_vi<dev::EpiCheb<false>>(DevState &, const DCsr &, const double *, dev::EpiCheb<false>, cudaStream_t, int);
template void launch_sellvi<dev::EpiCheb<false>>(DevState &, const DCsr &, const double *, dev::EpiCheb<false>, cudaStream_t, int);
}  // namespace amgb
