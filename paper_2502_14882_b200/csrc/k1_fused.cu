// k1_fused.cu — placeholder until the fused single-pass K1 lands.
#include "kvq_internal.cuh"
namespace kvqb {
bool quantize_fused_supported(size_t, size_t, int, int) { return false; }
cudaError_t launch_quantize_fused(const float*, size_t, size_t, size_t, int, float*, float*, uint8_t*,
                                  cudaStream_t) { return cudaErrorNotSupported; }
}  // namespace kvqb
