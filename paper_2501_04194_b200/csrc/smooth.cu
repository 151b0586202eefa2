// smooth.cu — smooth-interval kernels (placeholder; implemented in a later milestone).
#include "kernels.cuh"
namespace stlg {
cudaError_t launch_smooth_fwd(int, SParams&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_smooth_bwd(int, SParams&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace stlg
