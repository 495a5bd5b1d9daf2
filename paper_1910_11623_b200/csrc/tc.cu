// tc.cu — tcgen05 (sm_100a) forward/adjoint kernels.  Placeholder until the
// tensor-core path lands: reports "unsupported" so KERNEL_AUTO picks SIMT.
#include "kernels.cuh"

namespace bsde {
bool tc_supported(int, int) { return false; }
size_t tc_pack_bytes(int, int, int, int) { return 16; }
size_t tc_partial_bytes(int, int, int) { return 16; }
cudaError_t launch_fwd_tc(const PassArgs&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_bwd_tc(const PassArgs&, cudaStream_t) { return cudaErrorNotSupported; }
cudaError_t launch_pack_weights(const PassArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace bsde
