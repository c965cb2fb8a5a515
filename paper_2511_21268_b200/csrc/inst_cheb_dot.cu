// inst_cheb_dot.cu — explicit instantiations of launch_csr (and so of every CSR/SELL kernel variant) for: EpiCheb<true>.
#include "launch_csr.cuh"

namespace amgb {
template void launch_csr<dev::EpiCheb<true>>(DevState &, const DCsr &, const double *, dev::EpiCheb<true>, cudaStream_t, int);
}  // namespace amgb
