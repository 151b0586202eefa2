// until.cu — Until kernels (placeholder; implemented in the next milestone).
#include "kernels.cuh"
namespace stlg {
cudaError_t launch_until_fwd(int, UParams&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_until_bwd(int, UParams&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace stlg
