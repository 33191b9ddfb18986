// k2_decode_tc.cu — placeholder until the tensor-core path lands.
#include "kvq_internal.cuh"
namespace kvqb {
bool decode_tc_supported(const DecodeArgs&) { return false; }
cudaError_t launch_decode_tc(const DecodeArgs&, cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace kvqb
