// inst_vi_cheb_dot.cu — explicit instantiations of the value-indexed launchers (launch_csr_vi) for the epilogues of inst_cheb_dot.cu.
#include "launch_csr_vi.cuh"

namespace amgb {
template void launch_csr_vi<dev::EpiCheb<true>>(DevState &, const DCsr &, const double *, dev::EpiCheb<true>, cudaStream_t, int);
template void launch_sellvi<dev::EpiCheb<true>>(DevState &, const DCsr &, const double *, dev::EpiCheb<true>, cudaStream_t, int);
}  // namespace amgb
