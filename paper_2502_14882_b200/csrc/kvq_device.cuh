// kvq_device.cuh — device helpers shared by the decode kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace kvqb {

// Code of channel c in one packed row (reference layout: LE M-bit words, MSB-first
// codes; bitpack.hpp:182, 199-200).
__device__ __forceinline__ uint32_t code_at(const uint8_t* row, size_t c, int bits, int word_bits) {
    const int g = word_bits / bits;
    const size_t wi = c / (size_t)g;
    const int nb = word_bits / 8;
    uint32_t w = 0;
    for (int b = 0; b < nb; ++b) w |= (uint32_t)row[wi * nb + b] << (8 * b);
    return (w >> (word_bits - bits * ((int)(c % (size_t)g) + 1))) & (bits >= 32 ? 0xffffffffu : (1u << bits) - 1u);
}

// g (calibrate.hpp:62-67), evaluated with the reference's exact op order.
__device__ __forceinline__ float g_apply_dev(float x, float gamma, float width, float tau1, float tau2) {
    if (width <= 0.0f) return __fsub_rn(x, tau1);
    float t = __fdiv_rn(__fsub_rn(x, gamma), width);
    return __fsub_rn(x, __fadd_rn(__fmul_rn(tau1, __fsub_rn(1.0f, t)), __fmul_rn(tau2, t)));
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_min(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Block-wide reductions (blockDim.x a multiple of 32, <= 1024). Every thread gets the
// result. `red` must hold 32 floats.
template <int OP>  // 0 sum, 1 max, 2 min
__device__ __forceinline__ float block_reduce(float v, float* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = OP == 0 ? warp_sum(v) : (OP == 1 ? warp_max(v) : warp_min(v));
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    if (wid == 0) {
        float init = OP == 0 ? 0.0f : (OP == 1 ? -INFINITY : INFINITY);
        float x = lane < nw ? red[lane] : init;
        x = OP == 0 ? warp_sum(x) : (OP == 1 ? warp_max(x) : warp_min(x));
        if (lane == 0) red[0] = x;
    }
    __syncthreads();
    float r = red[0];
    __syncthreads();
    return r;
}

}  // namespace kvqb
