// inst_cheb.cu — explicit instantiations of launch_csr (and so of every CSR/SELL kernel variant) for: EpiCheb<false>.
#include "launch_csr.cuh"

namespace amgb {
template void launch_csr<dev::EpiCheb<false>>(DevState &, const DCsr &, const double *, dev::EpiCheb<false>, cudaStream_t, int);
}  // namespace amgb
