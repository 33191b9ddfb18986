// k1_quantize.cu — K1: channel-wise (or global) min/max stats, uniform b-bit codes and
// MSB-first packing, bit-exact with the reference quantizer:
//   compute_stats  quantize.hpp:64-89
//   quantize       quantize.hpp:91-127  (inv_step = L/(beta-alpha) or 0; round half away
//                                        from zero; clamp to [0, L])
//   pack           bitpack.hpp:161-187  (code i of a word at bits [M-b(i+1), M-bi), LE)
//   dequantize     quantize.hpp:129-146
// Every fp32 op uses an explicit _rn intrinsic so nvcc can neither contract to FMA nor
// approximate the division; that is what makes the codes bit-exact.
//
// Generic path (any dim, b in {1,2,4,8}, M in {8,16,32}, both modes): a stats kernel
// with an order-preserving (std::min "first wins") reduction, then one thread per
// packed output word. The fused single-pass path for the d = 128 / M = 8 decode layout
// lives in k1_fused.cu.
#include "kvq_internal.cuh"

namespace kvqb {

namespace {

// std::min / std::max as the reference uses them: the LEFT operand survives unless
// the right one is strictly smaller / larger, so among equal values (-0 vs +0) the
// first in scan order wins. Reductions below only ever combine (earlier, later).
__device__ __forceinline__ float ref_min(float left, float right) { return right < left ? right : left; }
__device__ __forceinline__ float ref_max(float left, float right) { return left < right ? right : left; }

constexpr int kStatTileC = 32;  // channels per CTA (one warp width: coalesced rows)
constexpr int kStatParts = 8;   // contiguous row ranges per CTA, folded in order

// Channel-wise stats (quantize.hpp:70-78) for a 32-channel tile of one matrix. With
// GLOBAL the per-channel result also carries the first row that produced it, for the
// row-major global fold (quantize.hpp:79-87) done by stats_global_finalize.
template <bool GLOBAL>
__global__ void __launch_bounds__(kStatTileC * kStatParts)
stats_kernel(const float* __restrict__ x, size_t rows, size_t dim, float* __restrict__ alpha,
             float* __restrict__ beta, int* __restrict__ lo_row, int* __restrict__ hi_row) {
    const size_t m = blockIdx.y;
    const size_t c = (size_t)blockIdx.x * kStatTileC + threadIdx.x;
    const int part = threadIdx.y;
    const size_t r0 = rows * part / kStatParts, r1 = rows * (part + 1) / kStatParts;
    const float* src = x + m * rows * dim;

    float lo = 0.f, hi = 0.f;
    int lr = 0, hr = 0;
    bool any = false;
    if (c < dim && r0 < r1) {
        lo = hi = __ldg(src + r0 * dim + c);
        lr = hr = (int)r0;
        any = true;
        size_t r = r0 + 1;
        // 8 loads in flight per thread; the fold itself stays strictly in row order.
        for (; r + 8 <= r1; r += 8) {
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) v[i] = __ldg(src + (r + i) * dim + c);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (GLOBAL) {
                    if (v[i] < lo) { lo = v[i]; lr = (int)(r + i); }
                    if (hi < v[i]) { hi = v[i]; hr = (int)(r + i); }
                } else {
                    lo = ref_min(lo, v[i]);
                    hi = ref_max(hi, v[i]);
                }
            }
        }
        for (; r < r1; ++r) {
            float v = __ldg(src + r * dim + c);
            if (GLOBAL) {
                if (v < lo) { lo = v; lr = (int)r; }
                if (hi < v) { hi = v; hr = (int)r; }
            } else {
                lo = ref_min(lo, v);
                hi = ref_max(hi, v);
            }
        }
    }
    __shared__ float s_lo[kStatParts][kStatTileC], s_hi[kStatParts][kStatTileC];
    __shared__ int s_lr[kStatParts][kStatTileC], s_hr[kStatParts][kStatTileC];
    __shared__ bool s_any[kStatParts][kStatTileC];
    s_lo[part][threadIdx.x] = lo;
    s_hi[part][threadIdx.x] = hi;
    s_lr[part][threadIdx.x] = lr;
    s_hr[part][threadIdx.x] = hr;
    s_any[part][threadIdx.x] = any;
    __syncthreads();
    if (part != 0 || c >= dim) return;
    // Parts hold consecutive row ranges: fold the non-empty ones left to right.
    bool have = any;
    for (int p = 1; p < kStatParts; ++p) {
        if (!s_any[p][threadIdx.x]) continue;
        float plo = s_lo[p][threadIdx.x], phi = s_hi[p][threadIdx.x];
        if (!have) {
            lo = plo, hi = phi, lr = s_lr[p][threadIdx.x], hr = s_hr[p][threadIdx.x], have = true;
            continue;
        }
        if (plo < lo) { lo = plo; lr = s_lr[p][threadIdx.x]; }
        if (hi < phi) { hi = phi; hr = s_hr[p][threadIdx.x]; }
    }
    alpha[m * dim + c] = lo;
    beta[m * dim + c] = hi;
    if (GLOBAL) {
        lo_row[m * dim + c] = lr;
        hi_row[m * dim + c] = hr;
    }
}

// Global mode: the reference folds all entries row-major, so among entries that compare
// equal to the extreme the one with the smallest (row, col) survives. Each channel
// carries its first extreme row; pick the smallest row*dim+col among tied channels.
__global__ void stats_global_finalize(size_t dim, float* alpha, float* beta, const int* lo_row,
                                      const int* hi_row) {
    const size_t m = blockIdx.x;
    float* a = alpha + m * dim;
    float* b = beta + m * dim;
    const int* lr = lo_row + m * dim;
    const int* hr = hi_row + m * dim;
    __shared__ float s_lo, s_hi;
    if (threadIdx.x == 0) {
        float lo = a[0], hi = b[0];
        size_t lpos = (size_t)lr[0] * dim, hpos = (size_t)hr[0] * dim;
        for (size_t c = 1; c < dim; ++c) {
            size_t lp = (size_t)lr[c] * dim + c, hp = (size_t)hr[c] * dim + c;
            if (a[c] < lo || (a[c] == lo && lp < lpos)) { lo = a[c]; lpos = lp; }
            if (hi < b[c] || (b[c] == hi && hp < hpos)) { hi = b[c]; hpos = hp; }
        }
        s_lo = lo;
        s_hi = hi;
    }
    __syncthreads();
    for (size_t c = threadIdx.x; c < dim; c += blockDim.x) {
        a[c] = s_lo;
        b[c] = s_hi;
    }
}

// inv_step (quantize.hpp:102-106), IEEE division.
__global__ void inv_step_kernel(const float* alpha, const float* beta, size_t n, float levels,
                                float* inv) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float range = __fsub_rn(beta[i], alpha[i]);
    inv[i] = range > 0.0f ? __fdiv_rn(levels, range) : 0.0f;
}

__device__ __forceinline__ uint32_t quantize_one(float x, float a, float inv, float levels) {
    // t = round((x - alpha) * inv_step), clamp [0, L] (quantize.hpp:114-116)
    float t = roundf(__fmul_rn(__fsub_rn(x, a), inv));
    t = t < 0.0f ? 0.0f : (levels < t ? levels : t);
    return (uint32_t)t;  // NaN -> 0, matching the x86 reference build
}

// One thread per packed word: codes of channels [w*g, w*g+g) of one row, MSB-first.
__global__ void quantize_pack_kernel(const float* __restrict__ x, size_t mats, size_t rows,
                                     size_t dim, const float* __restrict__ alpha,
                                     const float* __restrict__ inv, int bits, int word_bits,
                                     size_t words_per_row, uint8_t* __restrict__ codes) {
    const size_t total = mats * rows * words_per_row;
    const int g = word_bits / bits;
    const float levels = (float)((1u << bits) - 1u);
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t w = idx % words_per_row;
        const size_t mr = idx / words_per_row;  // m * rows + r
        const size_t m = mr / rows;
        const float* src = x + mr * dim;
        const float* a = alpha + m * dim;
        const float* iv = inv + m * dim;
        uint32_t acc = 0;
        for (int i = 0; i < g; ++i) {
            size_t c = w * g + i;
            uint32_t code = 0;
            if (c < dim) code = quantize_one(__ldg(src + c), __ldg(a + c), __ldg(iv + c), levels);
            acc |= code << (word_bits - bits * (i + 1));
        }
        uint8_t* dst = codes + idx * (size_t)(word_bits / 8);
        if (word_bits == 8) {
            dst[0] = (uint8_t)acc;
        } else if (word_bits == 16) {
            *reinterpret_cast<uint16_t*>(dst) = (uint16_t)acc;
        } else if (word_bits == 32) {
            *reinterpret_cast<uint32_t*>(dst) = acc;
        } else {
            for (int b = 0; b < word_bits / 8; ++b) dst[b] = (uint8_t)(acc >> (8 * b));
        }
    }
}

__global__ void pack_codes_kernel(const uint32_t* __restrict__ codes, size_t count, int bits,
                                  int word_bits, uint8_t* __restrict__ out, int* err_flag) {
    const int g = word_bits / bits;
    const size_t words = (count + g - 1) / g;
    const uint32_t limit = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
    for (size_t w = (size_t)blockIdx.x * blockDim.x + threadIdx.x; w < words;
         w += (size_t)gridDim.x * blockDim.x) {
        uint32_t acc = 0;
        for (int i = 0; i < g; ++i) {
            size_t idx = w * g + i;
            uint32_t code = idx < count ? codes[idx] : 0u;
            if (code > limit) *err_flag = 1;
            acc |= (code & limit) << (word_bits - bits * (i + 1));
        }
        for (int b = 0; b < word_bits / 8; ++b) out[w * (word_bits / 8) + b] = (uint8_t)(acc >> (8 * b));
    }
}

__device__ __forceinline__ uint32_t load_word(const uint8_t* bytes, size_t wi, int word_bits) {
    const uint8_t* p = bytes + wi * (size_t)(word_bits / 8);
    uint32_t w = 0;
    for (int b = 0; b < word_bits / 8; ++b) w |= (uint32_t)p[b] << (8 * b);
    return w;
}

__global__ void unpack_codes_kernel(const uint8_t* __restrict__ bytes, size_t count, int bits,
                                    int word_bits, uint32_t* __restrict__ out) {
    const int g = word_bits / bits;
    const uint32_t mask = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < count;
         idx += (size_t)gridDim.x * blockDim.x) {
        uint32_t w = load_word(bytes, idx / g, word_bits);
        int i = (int)(idx % g);
        out[idx] = (w >> (word_bits - bits * (i + 1))) & mask;
    }
}

__global__ void dequantize_kernel(const uint8_t* __restrict__ codes, size_t mats, size_t rows,
                                  size_t dim, const float* __restrict__ alpha,
                                  const float* __restrict__ beta, int bits, int word_bits,
                                  size_t row_bytes, float* __restrict__ out) {
    const int g = word_bits / bits;
    const uint32_t mask = (1u << bits) - 1u;
    const float levels = (float)((1u << bits) - 1u);
    const size_t total = mats * rows * dim;
    for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (size_t)gridDim.x * blockDim.x) {
        const size_t c = idx % dim;
        const size_t mr = idx / dim;
        const size_t m = mr / rows;
        uint32_t w = load_word(codes + mr * row_bytes, c / g, word_bits);
        uint32_t code = (w >> (word_bits - bits * ((int)(c % g) + 1))) & mask;
        float a = alpha[m * dim + c];
        float range = __fsub_rn(beta[m * dim + c], a);
        float step = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
        out[idx] = __fadd_rn(__fmul_rn((float)code, step), a);  // quantize.hpp:141-142
    }
}

unsigned grid_for(size_t work, unsigned block) {
    size_t g = (work + block - 1) / block;
    if (g > 148u * 64u) g = 148u * 64u;
    return (unsigned)(g ? g : 1);
}

}  // namespace

cudaError_t launch_compute_stats(const float* x, size_t mats, size_t rows, size_t dim, int mode,
                                 float* alpha, float* beta, cudaStream_t s) {
    dim3 grid((unsigned)((dim + kStatTileC - 1) / kStatTileC), (unsigned)mats);
    dim3 block(kStatTileC, kStatParts);
    if (mode == 0) {
        stats_kernel<false><<<grid, block, 0, s>>>(x, rows, dim, alpha, beta, nullptr, nullptr);
        note_launch();
        return cudaGetLastError();
    }
    int* rowsbuf = nullptr;
    cudaError_t e = cudaMallocAsync(&rowsbuf, sizeof(int) * 2 * mats * dim, s);
    if (e != cudaSuccess) return e;
    stats_kernel<true><<<grid, block, 0, s>>>(x, rows, dim, alpha, beta, rowsbuf, rowsbuf + mats * dim);
    stats_global_finalize<<<(unsigned)mats, 128, 0, s>>>(dim, alpha, beta, rowsbuf, rowsbuf + mats * dim);
    note_launch(2);
    e = cudaGetLastError();
    cudaFreeAsync(rowsbuf, s);
    return e;
}

cudaError_t launch_quantize_pack(const float* x, size_t mats, size_t rows, size_t dim,
                                 const float* alpha, const float* beta, int bits, int word_bits,
                                 uint8_t* codes, cudaStream_t s) {
    float* inv = nullptr;
    cudaError_t e = cudaMallocAsync(&inv, sizeof(float) * mats * dim, s);
    if (e != cudaSuccess) return e;
    const float levels = (float)((1u << bits) - 1u);
    inv_step_kernel<<<grid_for(mats * dim, 256), 256, 0, s>>>(alpha, beta, mats * dim, levels, inv);
    const size_t wpr = codes_per_row(dim, bits, word_bits) / (size_t)codes_per_word(bits, word_bits);
    quantize_pack_kernel<<<grid_for(mats * rows * wpr, 256), 256, 0, s>>>(
        x, mats, rows, dim, alpha, inv, bits, word_bits, wpr, codes);
    note_launch(2);
    e = cudaGetLastError();
    cudaFreeAsync(inv, s);
    return e;
}

cudaError_t launch_pack_codes(const uint32_t* codes, size_t count, int bits, int word_bits,
                              uint8_t* out, int* err_flag, cudaStream_t s) {
    size_t words = (count + (word_bits / bits) - 1) / (word_bits / bits);
    pack_codes_kernel<<<grid_for(words, 256), 256, 0, s>>>(codes, count, bits, word_bits, out, err_flag);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_unpack_codes(const uint8_t* bytes, size_t count, int bits, int word_bits,
                                uint32_t* out, cudaStream_t s) {
    unpack_codes_kernel<<<grid_for(count, 256), 256, 0, s>>>(bytes, count, bits, word_bits, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint8_t* codes, size_t mats, size_t rows, size_t dim,
                              const float* alpha, const float* beta, int bits, int word_bits,
                              float* out, cudaStream_t s) {
    dequantize_kernel<<<grid_for(mats * rows * dim, 256), 256, 0, s>>>(
        codes, mats, rows, dim, alpha, beta, bits, word_bits, row_bytes(dim, bits, word_bits), out);
    note_launch();
    return cudaGetLastError();
}

}  // namespace kvqb
