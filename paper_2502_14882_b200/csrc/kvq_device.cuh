// kvq_device.cuh — device helpers shared by the decode kernels.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace kvqb {

// Byte of a packed row where channel c's code starts, and its bit shift there: the code
// sits at bit M - N(k+1) of its LE word (k = c mod codes-per-word); for N <= 8 (N | 8) it
// never straddles a byte. Hoisting this out of token loops removes per-code divisions.
__device__ __forceinline__ void code_pos(size_t c, int bits, int word_bits, uint32_t& byte, uint32_t& shift) {
    const size_t cpw = (size_t)(word_bits / bits);
    const int bitpos = word_bits - bits * ((int)(c % cpw) + 1);
    byte = (uint32_t)((c / cpw) * (size_t)(word_bits / 8) + (size_t)(bitpos / 8));
    shift = (uint32_t)(bitpos % 8);  // 0 for N = 16 (half-word aligned)
}

// The code at (byte, shift) of a row: one byte for N <= 8; a 16-bit code (the standalone
// quantizer API allows N = 16) spans the two LE bytes of its half word.
__device__ __forceinline__ uint32_t code_load(const uint8_t* row, uint32_t byte, uint32_t shift, int bits,
                                              uint32_t mask) {
    const uint32_t v = bits <= 8 ? (uint32_t)row[byte] : (uint32_t)row[byte] | ((uint32_t)row[byte + 1] << 8);
    return (v >> shift) & mask;
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
