// k1_fused.cu — K1 code pass for the decode layout (d = 128, M = 8, channel-wise or
// global stats already computed): codes + MSB-first packing with warp ballots / shuffles,
// bit-exact with quantize (quantize.hpp:91-127) and pack (bitpack.hpp:64-90).
//
// Lane c of a warp owns channels c, 32+c, 64+c, 96+c of every row it visits: a row is
// read as four coalesced 128-byte transactions, the lane's four (alpha, inv_step) pairs
// live in registers for the whole kernel, and each 32-channel group of a row is packed by
// one warp-wide collective:
//   b = 1: W = ballot(code); the LE word of bytes 4w..4w+3 is byte_perm(brev(W), 0x0123)
//          (brev maps bit 8j+k to 8(3-j)+7-k; the byte swap puts channel 8j+k at bit
//          8j+7-k: MSB-first within byte j);
//   b = 2/4/8: each lane shifts its code to its bit position inside its 32-bit word and
//          the lanes sharing a word OR-reduce with shuffles.
// Per element: one fsub, one fmul (IEEE, no contraction), roundf (half away from zero),
// clamp - the reference's quantize_one exactly.
#include "kvq_internal.cuh"

namespace kvqb {

namespace {

constexpr int kDim = 128;
constexpr int kWarpsPerCta = 8;
constexpr int kRowsPerIter = 4;  // rows in flight per warp (16 loads per lane)

__device__ __forceinline__ uint32_t code_of(float x, float a, float inv, float levels) {
    float t = roundf(__fmul_rn(__fsub_rn(x, a), inv));
    t = t < 0.0f ? 0.0f : (levels < t ? levels : t);
    return (uint32_t)t;  // NaN -> 0, as the x86 reference build
}

// M-bit pack words (M = 8, 16, 32), each 32-bit register holding 32/M of them LE: the
// channel cw-th in the register sits at bit (cw / cpM) M + M - N (cw mod cpM + 1), cpM = M/N
// (bitpack.hpp:85). For N = 1 the warp ballot's brev puts channel i at bit 31 - i, which is
// M = 32 directly, M = 16 after swapping the half words, M = 8 after reversing the bytes.
template <int BITS>
__device__ __forceinline__ void pack_store(const uint32_t (&code)[4], uint8_t* row_out, int lane, int word_bits) {
    if constexpr (BITS == 1) {
        const uint32_t sel = word_bits == 8 ? 0x0123u : (word_bits == 16 ? 0x1032u : 0x3210u);
        uint32_t words[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) words[w] = __byte_perm(__brev(__ballot_sync(0xffffffffu, code[w] != 0u)), 0, sel);
        if (lane == 0) *reinterpret_cast<uint4*>(row_out) = make_uint4(words[0], words[1], words[2], words[3]);
    } else {
        constexpr int lanes_per_word = 32 / BITS;
        const int cpm = word_bits / BITS;
        const int cw = lane % lanes_per_word;
        const int shift = (cw / cpm) * word_bits + word_bits - BITS * (cw % cpm + 1);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            uint32_t v = code[w] << shift;
#pragma unroll
            for (int o = 1; o < lanes_per_word; o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
            // word index within the row: group w covers 32 channels = BITS words
            if (cw == 0) reinterpret_cast<uint32_t*>(row_out)[w * BITS + lane / lanes_per_word] = v;
        }
    }
}

template <int BITS>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
quantize_rows_d128(const float* __restrict__ x, size_t rows, const float* __restrict__ alpha,
                   const float* __restrict__ beta, uint8_t* __restrict__ codes, int word_bits) {
    constexpr int kRowBytes = 16 * BITS;
    const float levels = (float)((1u << BITS) - 1u);
    const size_t m = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float a[4], inv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
        const int c = 32 * w + lane;
        a[w] = alpha[m * kDim + c];
        const float range = __fsub_rn(beta[m * kDim + c], a[w]);
        inv[w] = range > 0.0f ? __fdiv_rn(levels, range) : 0.0f;  // quantize.hpp:102-106
    }
    const float* src = x + m * rows * kDim;
    uint8_t* dst = codes + m * rows * kRowBytes;
    const size_t stride = (size_t)gridDim.x * kWarpsPerCta * kRowsPerIter;
    for (size_t r0 = ((size_t)blockIdx.x * kWarpsPerCta + warp) * kRowsPerIter; r0 < rows; r0 += stride) {
        float v[kRowsPerIter][4];
#pragma unroll
        for (int i = 0; i < kRowsPerIter; ++i)
#pragma unroll
            for (int w = 0; w < 4; ++w)
                v[i][w] = r0 + i < rows ? __ldcs(src + (r0 + i) * kDim + 32 * w + lane) : 0.0f;
#pragma unroll
        for (int i = 0; i < kRowsPerIter; ++i) {
            if (r0 + i >= rows) break;  // warp-uniform
            uint32_t code[4];
#pragma unroll
            for (int w = 0; w < 4; ++w) code[w] = code_of(v[i][w], a[w], inv[w], levels);
            pack_store<BITS>(code, dst + (r0 + i) * kRowBytes, lane, word_bits);
        }
    }
}

// Token-wise stats (the opt-in V mode, north_star "token-wise min/max for V"): the
// reference quantizer (quantize.hpp:64-127) with the reduction axis swapped - alpha_j /
// beta_j are the min / max over the 128 channels of token j, codes use that token's step.
// One pass (a row's stats depend on the row only): warp per row, lane c owns channels
// c + 32 w; min / max carry the channel index so ties (-0 vs +0) resolve to the first
// channel, as std::min / std::max folding in channel order do.
template <int BITS>
__global__ void __launch_bounds__(kWarpsPerCta * 32)
quantize_rows_tok_d128(const float* __restrict__ x, size_t rows, float* __restrict__ alpha, float* __restrict__ beta,
                       float2* __restrict__ step_off, uint8_t* __restrict__ codes, int word_bits) {
    constexpr int kRowBytes = 16 * BITS;
    const float levels = (float)((1u << BITS) - 1u);
    const size_t m = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* src = x + m * rows * kDim;
    uint8_t* dst = codes + m * rows * kRowBytes;
    const size_t stride = (size_t)gridDim.x * kWarpsPerCta;
    for (size_t r = (size_t)blockIdx.x * kWarpsPerCta + warp; r < rows; r += stride) {
        float v[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) v[w] = __ldcs(src + r * kDim + 32 * w + lane);
        float lo = v[0], hi = v[0];
        int li = lane, hi_i = lane;
#pragma unroll
        for (int w = 1; w < 4; ++w) {  // this lane's channels in order: lane, 32 + lane, ...
            if (v[w] < lo) lo = v[w], li = 32 * w + lane;
            if (hi < v[w]) hi = v[w], hi_i = 32 * w + lane;
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            const float l2 = __shfl_xor_sync(0xffffffffu, lo, o), h2 = __shfl_xor_sync(0xffffffffu, hi, o);
            const int li2 = __shfl_xor_sync(0xffffffffu, li, o), hi2 = __shfl_xor_sync(0xffffffffu, hi_i, o);
            if (l2 < lo || (l2 == lo && li2 < li)) lo = l2, li = li2;
            if (hi < h2 || (h2 == hi && hi2 < hi_i)) hi = h2, hi_i = hi2;
        }
        const float range = __fsub_rn(hi, lo);
        const float inv = range > 0.0f ? __fdiv_rn(levels, range) : 0.0f;  // quantize.hpp:102-106
        if (lane == 0) {
            alpha[m * rows + r] = lo, beta[m * rows + r] = hi;
            // the decode's per-token pair: step s = (beta - alpha) / L and offset o = alpha / s
            // (v = s (code + o)); a flat token keeps s = 0, o = alpha
            const float st = fmaxf(range * (1.0f / levels), 0.0f);
            step_off[m * rows + r] = make_float2(st, range > 0.0f ? __fdividef(lo * levels, range) : lo);
        }
        uint32_t code[4];
#pragma unroll
        for (int w = 0; w < 4; ++w) code[w] = code_of(v[w], lo, inv, levels);
        pack_store<BITS>(code, dst + r * kRowBytes, lane, word_bits);
    }
}

}  // namespace

cudaError_t launch_quantize_tokenwise(const float* x, size_t mats, size_t rows, int bits, int word_bits,
                                      float* alpha, float* beta, float2* step_off, uint8_t* codes, cudaStream_t s) {
    if (rows == 0 || mats == 0) return cudaSuccess;
    size_t gx = (rows + kWarpsPerCta - 1) / kWarpsPerCta;
    const size_t cap = (148 * 16 + mats - 1) / mats;
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    dim3 grid((unsigned)gx, (unsigned)mats);
    switch (bits) {
        case 1: quantize_rows_tok_d128<1><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, step_off, codes, word_bits); break;
        case 2: quantize_rows_tok_d128<2><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, step_off, codes, word_bits); break;
        case 4: quantize_rows_tok_d128<4><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, step_off, codes, word_bits); break;
        case 8: quantize_rows_tok_d128<8><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, step_off, codes, word_bits); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

bool quantize_fused_supported(size_t rows, size_t dim, int word_bits, int mode) {
    (void)rows;
    (void)mode;  // stats (either mode) come from the stats kernel; codes are per channel
    return dim == (size_t)kDim && (word_bits == 8 || word_bits == 16 || word_bits == 32);
}

cudaError_t launch_quantize_fused(const float* x, size_t mats, size_t rows, size_t dim, int bits, int word_bits,
                                  int mode, float* alpha, float* beta, uint8_t* codes, cudaStream_t s) {
    if (rows == 0 || mats == 0) return cudaSuccess;
    cudaError_t e = launch_compute_stats(x, mats, rows, dim, mode, alpha, beta, s);  // compute_stats
    if (e != cudaSuccess) return e;
    const size_t rows_per_cta = (size_t)kWarpsPerCta * kRowsPerIter;
    size_t gx = (rows + rows_per_cta - 1) / rows_per_cta;
    // enough CTAs to fill the GPU several times over, grid-striding beyond that
    const size_t cap = (148 * 16 + mats - 1) / mats;
    if (gx > cap) gx = cap < 1 ? 1 : cap;
    dim3 grid((unsigned)gx, (unsigned)mats);
    switch (bits) {
        case 1: quantize_rows_d128<1><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, codes, word_bits); break;
        case 2: quantize_rows_d128<2><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, codes, word_bits); break;
        case 4: quantize_rows_d128<4><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, codes, word_bits); break;
        case 8: quantize_rows_d128<8><<<grid, kWarpsPerCta * 32, 0, s>>>(x, rows, alpha, beta, codes, word_bits); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

}  // namespace kvqb
