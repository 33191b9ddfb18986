// k2_decode_generic.cu — K2, general-shape path: fused post-scaled quantized decode
// attention for any head dim, bitwidth (1/2/4/8) and pack width (8/16/32). Used for the
// reference's small-shape API (tests, arbitrary d) and whenever per-token probability
// rows are requested (decode_step_detailed). The d = 128 throughput path is
// k2_decode_tc.cu.
//
// One CTA per (unit, query head). Per head, following HybridKVCache::run_decode
// (kvcache.hpp:263-311):
//   1. qs_c = q_c*((beta_c-alpha_c)/L) (0 if degenerate), qdota = sum q_c*alpha_c
//      (detail::scale_query, kernels.hpp:183-194)
//   2. vis_j = (qs . code_j + qdota) / sqrt(d); tail_t = (q . k_t) / sqrt(d)   (284-287)
//   3. gamma/delta = min/max(vis); g on vis only; one softmax over [g(vis) | tail]
//      (calibrate.hpp:100-114)
//   4. out_c = s_c * sum_j w_j code_jc + alpha_c * sum_j w_j + sum_t w_t v_tc
//      (kernels.hpp:277-283; kvcache.hpp:297-304)
// Packed K/V are never dequantized: the scales are folded into q (K side) and into the
// epilogue (V side). DecodeArgs::dequant_dot selects BASELINE config 3's "without
// post-scaling" ablation instead: every code is dequantized in-register (alpha_c + code *
// s_c, quantize.hpp:129-146) and dotted with q / weighted by w (naive_qk / naive_wv,
// kernels.hpp:401-426) - the same scores and outputs up to fp32 reassociation.
#include "kvq_device.cuh"
#include "kvq_internal.cuh"

namespace kvqb {

namespace {

constexpr int kThreads = 256;

__global__ void __launch_bounds__(kThreads)
decode_generic_kernel(DecodeArgs a) {
    extern __shared__ float smem[];
    const size_t d = a.dim;
    const size_t cpr = codes_per_row(d, a.bits, a.word_bits);
    const size_t rb = row_bytes(d, a.bits, a.word_bits);
    float* qs = smem;            // [cpr]
    float* red = smem + cpr;     // [32]
    float* scal = red + 32;      // qdota
    // channel c's code: byte cbyte[c] of the row, bits [cshift[c], cshift[c] + b) - codes
    // never straddle a byte (b | 8), so no per-code division or word assembly
    float* kal = scal + 8;                                      // [d] K alpha (dequant_dot)
    uint16_t* cbyte = reinterpret_cast<uint16_t*>(kal + d);     // [d]
    uint8_t* cshift = reinterpret_cast<uint8_t*>(cbyte + d);    // [d]
    const bool dq = a.dequant_dot != 0;
    const size_t unit = blockIdx.x / a.group;
    const size_t g = blockIdx.x % a.group;
    const size_t b = unit / a.kv_heads;
    const size_t n = a.n_vis;
    const size_t nt = (size_t)a.tail_len[b];
    const size_t row_len = n + nt;
    const float levels = (float)((1u << a.bits) - 1u);
    const float inv_sqrt_d = __fdiv_rn(1.0f, sqrtf((float)d));  // kvcache.hpp:273

    const float* q = a.q + (unit * a.group + g) * d;
    const float* ka = a.k_alpha + unit * d;
    const float* kb = a.k_beta + unit * d;
    const uint8_t* kc = a.k_codes + unit * n * rb;
    const uint8_t* vc = a.v_codes + unit * n * rb;
    const float* kt = a.k_tail + unit * a.tail_cap * d;
    const float* vt = a.v_tail + unit * a.tail_cap * d;
    float* row = a.scratch + (unit * a.group + g) * (n + a.tail_cap);

    for (size_t c = threadIdx.x; c < cpr; c += blockDim.x) {
        float v = 0.0f;
        if (c < d) {
            float range = __fsub_rn(kb[c], ka[c]);
            const float stp = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
            v = dq ? stp : (range > 0.0f ? __fmul_rn(q[c], stp) : 0.0f);  // dequant: K step
            kal[c] = ka[c];
        }
        qs[c] = v;
    }
    if (threadIdx.x == 0) {  // sequential, as the reference accumulates it
        float qa = 0.0f;
        for (size_t c = 0; c < d; ++c) qa = __fadd_rn(qa, __fmul_rn(q[c], ka[c]));
        scal[0] = qa;
    }
    for (size_t c = threadIdx.x; c < d; c += blockDim.x) {
        uint32_t by, sh;
        code_pos(c, a.bits, a.word_bits, by, sh);
        cbyte[c] = (uint16_t)by;
        cshift[c] = (uint8_t)sh;
    }
    __syncthreads();
    const float qdota = scal[0];
    const uint32_t cmask = (1u << a.bits) - 1u;
    auto code = [&](const uint8_t* r, size_t c) { return (float)(((uint32_t)r[cbyte[c]] >> cshift[c]) & cmask); };

    // Scores. Local min/max of the visual part.
    float lo = INFINITY, hi = -INFINITY;
    for (size_t j = threadIdx.x; j < n; j += blockDim.x) {
        const uint8_t* r = kc + j * rb;
        float acc = 0.0f;
        if (dq) {  // dequantize-then-dot: k_jc = alpha_c + code * s_c, then q . k_j
            for (size_t c = 0; c < d; ++c) acc = __fmaf_rn(q[c], __fmaf_rn(code(r, c), qs[c], kal[c]), acc);
            const float s = __fmul_rn(acc, inv_sqrt_d);
            row[j] = s;
            lo = fminf(lo, s);
            hi = fmaxf(hi, s);
            continue;
        }
        if ((rb & 3) == 0 && a.bits <= 8) {  // 32-bit row words: one load per word, codes in order
            const uint32_t* r32 = reinterpret_cast<const uint32_t*>(r);
            uint32_t w = 0, cur = 0xffffffffu;
            for (size_t c = 0; c < d; ++c) {
                const uint32_t wi = cbyte[c] >> 2;
                if (wi != cur) w = __ldg(r32 + wi), cur = wi;
                acc = __fmaf_rn(qs[c], (float)((w >> (8 * (cbyte[c] & 3) + cshift[c])) & cmask), acc);
            }
        } else {
            for (size_t c = 0; c < d; ++c) acc = __fmaf_rn(qs[c], code(r, c), acc);
        }
        float s = __fmul_rn(__fadd_rn(acc, qdota), inv_sqrt_d);
        row[j] = s;
        lo = fminf(lo, s);
        hi = fmaxf(hi, s);
    }
    for (size_t t = threadIdx.x; t < nt; t += blockDim.x) {
        const float* r = kt + t * d;
        float acc = 0.0f;
        for (size_t c = 0; c < d; ++c) acc = __fmaf_rn(q[c], r[c], acc);
        row[n + t] = __fmul_rn(acc, inv_sqrt_d);
    }
    const float gamma = block_reduce<2>(lo, red);
    const float delta = block_reduce<1>(hi, red);
    const float width = __fsub_rn(delta, gamma);
    if (threadIdx.x == 0 && a.violations && n > 0) {
        // g_monotone (calibrate.hpp:52-54)
        a.violations[unit * a.group + g] = (__fadd_rn(width, __fsub_rn(a.tau1, a.tau2)) > 0.0f) ? 0 : 1;
    } else if (threadIdx.x == 0 && a.violations) {
        a.violations[unit * a.group + g] = 0;
    }

    // Calibrate the visual part; row max over the concatenation.
    float mx = -INFINITY;
    for (size_t j = threadIdx.x; j < row_len; j += blockDim.x) {
        float v = row[j];
        if (j < n) {
            v = g_apply_dev(v, gamma, width, a.tau1, a.tau2);
            row[j] = v;
        }
        mx = fmaxf(mx, v);
    }
    mx = block_reduce<1>(mx, red);
    float sum = 0.0f;
    for (size_t j = threadIdx.x; j < row_len; j += blockDim.x) {
        float e = expf(__fsub_rn(row[j], mx));
        row[j] = e;
        sum += e;
    }
    sum = block_reduce<0>(sum, red);
    float* wout = a.weights ? a.weights + (unit * a.group + g) * a.weights_stride : nullptr;
    for (size_t j = threadIdx.x; j < row_len; j += blockDim.x) {
        float w = __fdiv_rn(row[j], sum);
        row[j] = w;
        if (wout) wout[j] = w;
    }
    __syncthreads();

    // w.V over the packed segment (tokens ascending per lane), then the fp32 tail.
    const float* va = a.v_alpha + unit * d;
    const float* vb = a.v_beta + unit * d;
    float* out = a.out + (unit * a.group + g) * d;
    for (size_t c = threadIdx.x; c < d; c += blockDim.x) {
        float acc = 0.0f, wsum = 0.0f;
        if (dq) {  // dequantize-then-dot: out_c = sum_j w_j (alpha_c + code_jc s_c)
            const float range = __fsub_rn(vb[c], va[c]);
            const float step = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
            for (size_t j = 0; j < n; ++j) acc = __fmaf_rn(row[j], __fmaf_rn(code(vc + j * rb, c), step, va[c]), acc);
            float tacc = 0.0f;
            for (size_t t = 0; t < nt; ++t) tacc = __fmaf_rn(row[n + t], vt[t * d + c], tacc);
            out[c] = __fadd_rn(acc, tacc);
            continue;
        }
        for (size_t j = 0; j < n; ++j) {
            float w = row[j];
            wsum = __fadd_rn(wsum, w);
            acc = __fmaf_rn(w, code(vc + j * rb, c), acc);
        }
        float o = 0.0f;
        if (n > 0) {
            float range = __fsub_rn(vb[c], va[c]);
            float step = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
            o = __fadd_rn(__fmul_rn(step, acc), __fmul_rn(va[c], wsum));
        }
        float tacc = 0.0f;
        for (size_t t = 0; t < nt; ++t) tacc = __fmaf_rn(row[n + t], vt[t * d + c], tacc);
        out[c] = __fadd_rn(o, tacc);
    }
}

// ---- standalone kernels.hpp / calibrate.hpp entry points ------------------------

__global__ void qk_scores_kernel(const float* __restrict__ q, const uint8_t* __restrict__ codes,
                                 const float* __restrict__ alpha, const float* __restrict__ beta,
                                 size_t tokens, size_t dim, int bits, int word_bits,
                                 float* __restrict__ scores) {
    extern __shared__ float smem[];
    const size_t h = blockIdx.y;
    const size_t cpr = codes_per_row(dim, bits, word_bits);
    const size_t rb = row_bytes(dim, bits, word_bits);
    const float levels = (float)((1u << bits) - 1u);
    float* qs = smem;
    const float* qh = q + h * dim;
    const float* a = alpha + h * dim;
    const float* be = beta + h * dim;
    for (size_t c = threadIdx.x; c < cpr; c += blockDim.x) {
        float v = 0.0f;
        if (c < dim) {
            float range = __fsub_rn(be[c], a[c]);
            v = range > 0.0f ? __fmul_rn(qh[c], __fdiv_rn(range, levels)) : 0.0f;
        }
        qs[c] = v;
    }
    if (threadIdx.x == 0) {
        float qa = 0.0f;
        for (size_t c = 0; c < dim; ++c) qa = __fadd_rn(qa, __fmul_rn(qh[c], a[c]));
        smem[cpr] = qa;
    }
    uint16_t* cbyte = reinterpret_cast<uint16_t*>(smem + cpr + 1);  // [dim] code positions
    uint8_t* cshift = reinterpret_cast<uint8_t*>(cbyte + dim);
    for (size_t c = threadIdx.x; c < dim; c += blockDim.x) {
        uint32_t by, sh;
        code_pos(c, bits, word_bits, by, sh);
        cbyte[c] = (uint16_t)by;
        cshift[c] = (uint8_t)sh;
    }
    __syncthreads();
    const float qdota = smem[cpr];
    const uint32_t cmask = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
    const uint8_t* seg = codes + h * tokens * rb;
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < tokens;
         j += (size_t)gridDim.x * blockDim.x) {
        const uint8_t* r = seg + j * rb;
        float acc = 0.0f;
        if ((rb & 3) == 0) {  // 32-bit row words: one load per word, codes in channel order
            const uint32_t* r32 = reinterpret_cast<const uint32_t*>(r);
            uint32_t w = 0, cur = 0xffffffffu;
            for (size_t c = 0; c < dim; ++c) {
                const uint32_t wi = cbyte[c] >> 2;
                if (wi != cur) w = __ldg(r32 + wi), cur = wi;
                acc = __fmaf_rn(qs[c], (float)((w >> (8 * (cbyte[c] & 3) + cshift[c])) & cmask), acc);
            }
        } else {
            for (size_t c = 0; c < dim; ++c)
                acc = __fmaf_rn(qs[c], (float)code_load(r, cbyte[c], cshift[c], bits, cmask), acc);
        }
        scores[h * tokens + j] = __fadd_rn(acc, qdota);
    }
}

__global__ void wv_output_kernel(const float* __restrict__ w, const uint8_t* __restrict__ codes,
                                 const float* __restrict__ alpha, const float* __restrict__ beta,
                                 size_t tokens, size_t dim, int bits, int word_bits,
                                 float* __restrict__ out) {
    const size_t h = blockIdx.y;
    const size_t rb = row_bytes(dim, bits, word_bits);
    const float levels = (float)((1u << bits) - 1u);
    const float* wh = w + h * tokens;
    const uint8_t* seg = codes + h * tokens * rb;
    for (size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x; c < dim;
         c += (size_t)gridDim.x * blockDim.x) {
        float acc = 0.0f, wsum = 0.0f;
        uint32_t by, sh;
        code_pos(c, bits, word_bits, by, sh);
        const uint32_t cmask = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
        for (size_t j = 0; j < tokens; ++j) {
            wsum = __fadd_rn(wsum, wh[j]);
            acc = __fmaf_rn(wh[j], (float)code_load(seg + j * rb, by, sh, bits, cmask), acc);
        }
        float a = alpha[h * dim + c];
        float range = __fsub_rn(beta[h * dim + c], a);
        float step = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
        out[h * dim + c] = __fadd_rn(__fmul_rn(step, acc), __fmul_rn(a, wsum));
    }
}

__global__ void calibrated_softmax_kernel(const float* __restrict__ vis, size_t n_vis,
                                          const float* __restrict__ tail, size_t n_tail,
                                          float tau1, float tau2, float* __restrict__ out,
                                          int* violations) {
    __shared__ float red[32];
    const size_t r = blockIdx.x;
    const float* v = vis + r * n_vis;
    const float* t = tail + r * n_tail;
    float* o = out + r * (n_vis + n_tail);
    float lo = INFINITY, hi = -INFINITY;
    for (size_t j = threadIdx.x; j < n_vis; j += blockDim.x) {
        lo = fminf(lo, v[j]);
        hi = fmaxf(hi, v[j]);
    }
    const float gamma = block_reduce<2>(lo, red);
    const float delta = block_reduce<1>(hi, red);
    const float width = __fsub_rn(delta, gamma);
    if (threadIdx.x == 0 && violations)
        violations[r] = (n_vis > 0 && !(__fadd_rn(width, __fsub_rn(tau1, tau2)) > 0.0f)) ? 1 : 0;
    float mx = -INFINITY;
    for (size_t j = threadIdx.x; j < n_vis + n_tail; j += blockDim.x) {
        float x = j < n_vis ? g_apply_dev(v[j], gamma, width, tau1, tau2) : t[j - n_vis];
        o[j] = x;
        mx = fmaxf(mx, x);
    }
    mx = block_reduce<1>(mx, red);
    float sum = 0.0f;
    for (size_t j = threadIdx.x; j < n_vis + n_tail; j += blockDim.x) {
        float e = expf(__fsub_rn(o[j], mx));
        o[j] = e;
        sum += e;
    }
    sum = block_reduce<0>(sum, red);
    for (size_t j = threadIdx.x; j < n_vis + n_tail; j += blockDim.x) o[j] = __fdiv_rn(o[j], sum);
}

__global__ void naive_qk_kernel(const float* __restrict__ q, const float* __restrict__ k, size_t rows,
                                size_t cols, float* __restrict__ out) {
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < rows; j += (size_t)gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (size_t c = 0; c < cols; ++c) acc = __fadd_rn(acc, __fmul_rn(q[c], k[j * cols + c]));
        out[j] = acc;
    }
}

__global__ void naive_wv_kernel(const float* __restrict__ w, const float* __restrict__ v, size_t rows,
                                size_t cols, float* __restrict__ out) {
    for (size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x; c < cols; c += (size_t)gridDim.x * blockDim.x) {
        float acc = 0.0f;
        for (size_t j = 0; j < rows; ++j) acc = __fadd_rn(acc, __fmul_rn(w[j], v[j * cols + c]));
        out[c] = acc;
    }
}

}  // namespace

cudaError_t launch_naive_qk(const float* q, const float* k, size_t rows, size_t cols, float* out, cudaStream_t s) {
    naive_qk_kernel<<<(unsigned)((rows + 255) / 256 ? (rows + 255) / 256 : 1), 256, 0, s>>>(q, k, rows, cols, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_naive_wv(const float* w, const float* v, size_t rows, size_t cols, float* out, cudaStream_t s) {
    naive_wv_kernel<<<(unsigned)((cols + 127) / 128 ? (cols + 127) / 128 : 1), 128, 0, s>>>(w, v, rows, cols, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode_generic(const DecodeArgs& a, cudaStream_t s) {
    const size_t cpr = codes_per_row(a.dim, a.bits, a.word_bits);
    const size_t smem = sizeof(float) * (cpr + 40 + a.dim) + 3 * a.dim + 16;  // + K alpha, byte / shift
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(decode_generic_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    decode_generic_kernel<<<(unsigned)(a.units * a.group), kThreads, smem, s>>>(a);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_qk_scores(const float* q, const uint8_t* codes, const float* alpha,
                             const float* beta, size_t heads, size_t tokens, size_t dim,
                             int bits, int word_bits, float* scores, cudaStream_t s) {
    const size_t cpr = codes_per_row(dim, bits, word_bits);
    dim3 grid((unsigned)((tokens + 255) / 256 > 0 ? (tokens + 255) / 256 : 1), (unsigned)heads);
    qk_scores_kernel<<<grid, 256, sizeof(float) * (cpr + 1) + 3 * dim + 8, s>>>(q, codes, alpha, beta, tokens, dim,
                                                                   bits, word_bits, scores);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_wv_output(const float* w, const uint8_t* codes, const float* alpha,
                             const float* beta, size_t heads, size_t tokens, size_t dim,
                             int bits, int word_bits, float* out, cudaStream_t s) {
    dim3 grid((unsigned)((dim + 127) / 128), (unsigned)heads);
    wv_output_kernel<<<grid, 128, 0, s>>>(w, codes, alpha, beta, tokens, dim, bits, word_bits, out);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_calibrated_softmax(const float* vis, size_t n_vis, const float* tail,
                                      size_t n_tail, size_t rows, float tau1, float tau2,
                                      float* out, int* violations, cudaStream_t s) {
    calibrated_softmax_kernel<<<(unsigned)rows, 256, 0, s>>>(vis, n_vis, tail, n_tail, tau1, tau2, out,
                                                             violations);
    note_launch();
    return cudaGetLastError();
}

}  // namespace kvqb
