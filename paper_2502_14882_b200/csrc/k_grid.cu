// k_grid.cu — offline tau search on the device: grid_mse_table and
// grid_search (reference calibrate.hpp:160-234).
//
// prepare_samples (160-178): quant rows = post-scaled q.K of each sample (the decode's
// qk_scores kernel) / sqrt(d); exact rows = softmax(q K_exact^T / sqrt(d)).
// grid: one CTA per (cell, sample) evaluates sample_mse (180-188): the calibrated softmax
// of the quant row (g with the cell's tau on [gamma, delta]) against the exact row, the
// squared differences summed in double. The per-cell mean over samples runs in sample
// order (deterministic); the argmin tie-break (smaller tau1, then tau2) is applied by the
// caller on the returned table.
#include <cfloat>

#include "kvq_internal.cuh"

namespace kvqb {

namespace {

constexpr int kThreads = 256;

// Block reductions (fixed shape: warp shuffles, then warps in order).
template <typename T, typename Op>
__device__ T block_reduce(T v, Op op, T* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o; o >>= 1) v = op(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    T r = red[0];
    for (int w = 1; w < kThreads / 32; ++w) r = op(r, red[w]);
    return r;
}

// exact[s][j] = (q_s . k_sj) * (1/sqrt(d)): naive_qk (kernels.hpp:401-413) then the scale of
// calibrate.hpp:168-172, bit-exact with the reference: one thread per token accumulates in
// channel order with separately rounded products and sums (the reference's scalar loop).
__global__ void exact_scores_kernel(const float* __restrict__ q, const float* __restrict__ k, size_t n, size_t d,
                                    float inv_sqrt_d, float* __restrict__ out) {
    const size_t s = blockIdx.y;
    const float* qr = q + s * d;
    for (size_t j = (size_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (size_t)gridDim.x * blockDim.x) {
        const float* kr = k + (s * n + j) * d;
        float acc = 0.0f;
        for (size_t c = 0; c < d; ++c) acc = __fadd_rn(acc, __fmul_rn(qr[c], kr[c]));
        out[s * n + j] = __fmul_rn(acc, inv_sqrt_d);
    }
}

__global__ void scale_kernel(float* x, size_t count, float f);

void launch_exact_scores(const float* q, const float* k, size_t rows_sets, size_t n, size_t d, float inv_sqrt_d,
                         float* out, cudaStream_t s) {
    dim3 eg((unsigned)((n + kThreads - 1) / kThreads < 1024 ? (n + kThreads - 1) / kThreads : 1024),
            (unsigned)rows_sets);
    exact_scores_kernel<<<eg, kThreads, 0, s>>>(q, k, n, d, inv_sqrt_d, out);
}

__global__ void scale_kernel(float* x, size_t count, float f) {  // x *= f, one rounding (calibrate.hpp:170)
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        x[i] = __fmul_rn(x[i], f);
}

// One CTA per (cell, sample): sample_mse (calibrate.hpp:180-188).
__global__ void __launch_bounds__(kThreads)
grid_cell_kernel(const float* __restrict__ quant, const float* __restrict__ exact_prob, size_t n,
                 const float* __restrict__ tau1, const float* __restrict__ tau2, double* __restrict__ mse_cs,
                 size_t samples) {
    __shared__ float redf[kThreads / 32];
    __shared__ double redd[kThreads / 32];
    const size_t c = blockIdx.x, s = blockIdx.y;
    const float t1 = tau1[c], t2 = tau2[c];
    const float* row = quant + s * n;
    const float* ex = exact_prob + s * n;
    // row_range (calibrate.hpp:39-47)
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (size_t j = threadIdx.x; j < n; j += kThreads) lo = fminf(lo, row[j]), hi = fmaxf(hi, row[j]);
    const float gamma = block_reduce(lo, [](float a, float b) { return fminf(a, b); }, redf);
    const float delta = block_reduce(hi, [](float a, float b) { return fmaxf(a, b); }, redf);
    const float width = __fsub_rn(delta, gamma);
    auto g = [&](float x) {  // g_apply (calibrate.hpp:62-67), separately rounded as in the reference
        if (width <= 0.0f) return __fsub_rn(x, t1);
        const float t = __fdiv_rn(__fsub_rn(x, gamma), width);
        return __fsub_rn(x, __fadd_rn(__fmul_rn(t1, __fsub_rn(1.0f, t)), __fmul_rn(t2, t)));
    };
    // softmax_inplace (calibrate.hpp:77-87): max, exp, sum, divide
    float m = -FLT_MAX;
    for (size_t j = threadIdx.x; j < n; j += kThreads) m = fmaxf(m, g(row[j]));
    m = block_reduce(m, [](float a, float b) { return fmaxf(a, b); }, redf);
    float sum = 0.0f;
    for (size_t j = threadIdx.x; j < n; j += kThreads) sum += expf(g(row[j]) - m);
    sum = block_reduce(sum, [](float a, float b) { return a + b; }, redf);
    double acc = 0.0;
    for (size_t j = threadIdx.x; j < n; j += kThreads) {
        const float p = expf(g(row[j]) - m) / sum;
        const double diff = (double)p - (double)ex[j];
        acc += diff * diff;
    }
    acc = block_reduce(acc, [](double a, double b) { return a + b; }, redd);
    if (threadIdx.x == 0) mse_cs[c * samples + s] = acc / (double)n;
}

// mse_report, one CTA per head (calibrate.hpp:300-351). quant: the head's post-scaled q.K row
// (already x 1/sqrt(d)); exact: the exact row. Writes qc = g(quant) (the calibrated
// pre-softmax row), the bins+1 shared edges over the union of the three rows, the three
// histograms (bin_row, 272-287) and both probability MSEs (prob_mse, 289-296).
__global__ void __launch_bounds__(kThreads)
report_head_kernel(const float* __restrict__ quant, const float* __restrict__ exact, size_t n, size_t bins,
                   float t1, float t2, float* __restrict__ qc_out, float* __restrict__ edges,
                   unsigned long long* __restrict__ counts, int shared_hist, double* __restrict__ mse_q,
                   double* __restrict__ mse_qc) {
    extern __shared__ unsigned int hist[];  // [3][bins] when shared_hist
    __shared__ float redf[kThreads / 32];
    __shared__ double redd[kThreads / 32];
    const size_t h = blockIdx.x;
    const float* qrow = quant + h * n;
    const float* erow = exact + h * n;
    float* crow = qc_out + h * n;
    float* edge = edges + h * (bins + 1);
    unsigned long long* cnt = counts + h * 3 * bins;
    auto fmin_ = [](float a, float b) { return fminf(a, b); };
    auto fmax_ = [](float a, float b) { return fmaxf(a, b); };
    // row_range of the quantized row (39-47), then g_transform (69-74)
    float lo = FLT_MAX, hi = -FLT_MAX;
    for (size_t j = threadIdx.x; j < n; j += kThreads) lo = fminf(lo, qrow[j]), hi = fmaxf(hi, qrow[j]);
    const float gamma = block_reduce(lo, fmin_, redf);
    const float delta = block_reduce(hi, fmax_, redf);
    const float width = __fsub_rn(delta, gamma);
    lo = FLT_MAX, hi = -FLT_MAX;
    float mx[3] = {-FLT_MAX, -FLT_MAX, -FLT_MAX};
    for (size_t j = threadIdx.x; j < n; j += kThreads) {
        const float x = qrow[j], e = erow[j];
        float c;
        if (width <= 0.0f) {
            c = __fsub_rn(x, t1);
        } else {
            const float t = __fdiv_rn(__fsub_rn(x, gamma), width);
            c = __fsub_rn(x, __fadd_rn(__fmul_rn(t1, __fsub_rn(1.0f, t)), __fmul_rn(t2, t)));
        }
        crow[j] = c;
        lo = fminf(lo, fminf(e, fminf(x, c)));
        hi = fmaxf(hi, fmaxf(e, fmaxf(x, c)));
        mx[0] = fmaxf(mx[0], e), mx[1] = fmaxf(mx[1], x), mx[2] = fmaxf(mx[2], c);
    }
    lo = block_reduce(lo, fmin_, redf);
    hi = block_reduce(hi, fmax_, redf);
    for (int v = 0; v < 3; ++v) mx[v] = block_reduce(mx[v], fmax_, redf);
    // shared edges: lo + (hi - lo) * i / bins (322-331)
    const float span = __fsub_rn(hi, lo), fb = (float)bins;
    for (size_t i = threadIdx.x; i <= bins; i += kThreads)
        edge[i] = __fadd_rn(lo, __fdiv_rn(__fmul_rn(span, (float)i), fb));
    const float blo = lo, bhi = __fadd_rn(lo, __fdiv_rn(__fmul_rn(span, fb), fb));  // edges.front/back
    const float bw = __fsub_rn(bhi, blo);
    if (shared_hist)
        for (size_t i = threadIdx.x; i < 3 * bins; i += kThreads) hist[i] = 0u;
    __syncthreads();
    auto bin_of = [&](float v) -> size_t {
        if (!(bw > 0.0f)) return 0;
        const float t = fmaxf(0.0f, __fmul_rn(__fdiv_rn(__fsub_rn(v, blo), bw), fb));  // NaN -> 0
        const size_t i = (size_t)t;
        return i < bins - 1 ? i : bins - 1;
    };
    // written rows are re-read by the same thread (qc) -- no barrier needed for crow
    float sum[3] = {0.0f, 0.0f, 0.0f};
    for (size_t j = threadIdx.x; j < n; j += kThreads) {
        const float r[3] = {erow[j], qrow[j], crow[j]};
#pragma unroll
        for (int v = 0; v < 3; ++v) {
            const size_t b = bin_of(r[v]);
            if (shared_hist) atomicAdd(&hist[v * bins + b], 1u);
            else atomicAdd(&cnt[v * bins + b], 1ull);
            sum[v] += expf(__fsub_rn(r[v], mx[v]));
        }
    }
    for (int v = 0; v < 3; ++v) sum[v] = block_reduce(sum[v], [](float a, float b) { return a + b; }, redf);
    double aq = 0.0, ac = 0.0;
    for (size_t j = threadIdx.x; j < n; j += kThreads) {
        const float pe = __fdiv_rn(expf(__fsub_rn(erow[j], mx[0])), sum[0]);
        const float pq = __fdiv_rn(expf(__fsub_rn(qrow[j], mx[1])), sum[1]);
        const float pc = __fdiv_rn(expf(__fsub_rn(crow[j], mx[2])), sum[2]);
        const double dq = (double)pq - (double)pe, dc = (double)pc - (double)pe;
        aq += dq * dq;
        ac += dc * dc;
    }
    aq = block_reduce(aq, [](double a, double b) { return a + b; }, redd);
    ac = block_reduce(ac, [](double a, double b) { return a + b; }, redd);
    if (shared_hist) {
        __syncthreads();
        for (size_t i = threadIdx.x; i < 3 * bins; i += kThreads) cnt[i] = hist[i];
    }
    if (threadIdx.x == 0) {
        mse_q[h] = aq / (double)n;
        mse_qc[h] = ac / (double)n;
    }
}

}  // namespace

cudaError_t launch_mse_report(const float* queries, const float* keys, size_t heads, size_t n, size_t d, int bits,
                              int mode, int word_bits, float tau1, float tau2, size_t bins, float* alpha, float* beta,
                              uint8_t* codes, float* quant, float* exact, float* qc, float* edges,
                              unsigned long long* counts, double* mse_q, double* mse_qc, cudaStream_t s) {
    // per head: compute_stats + quantize (K1), qk_scores and naive_qk, both x 1/sqrt(d)
    cudaError_t e = launch_compute_stats(keys, heads, n, d, mode, alpha, beta, s);
    if (e != cudaSuccess) return e;
    e = launch_quantize_pack(keys, heads, n, d, alpha, beta, bits, word_bits, codes, s);
    if (e != cudaSuccess) return e;
    e = launch_qk_scores(queries, codes, alpha, beta, heads, n, d, bits, word_bits, quant, s);
    if (e != cudaSuccess) return e;
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    const size_t total = heads * n;
    scale_kernel<<<(unsigned)((total + 255) / 256 < 1184 ? (total + 255) / 256 : 1184), 256, 0, s>>>(quant, total,
                                                                                                    inv_sqrt_d);
    launch_exact_scores(queries, keys, heads, n, d, inv_sqrt_d, exact, s);
    const size_t hist_bytes = 3 * bins * sizeof(unsigned int);
    const int shared_hist = hist_bytes <= 48 * 1024;
    if (!shared_hist) {
        e = cudaMemsetAsync(counts, 0, heads * 3 * bins * sizeof(unsigned long long), s);
        if (e != cudaSuccess) return e;
    }
    report_head_kernel<<<(unsigned)heads, kThreads, shared_hist ? hist_bytes : 0, s>>>(
        quant, exact, n, bins, tau1, tau2, qc, edges, counts, shared_hist, mse_q, mse_qc);
    note_launch(3);
    return cudaGetLastError();
}

cudaError_t launch_grid_mse(const float* queries, const float* keys_exact, const uint8_t* codes, const float* alpha,
                            const float* beta, size_t samples, size_t n, size_t d, int bits, int word_bits,
                            const float* tau1, const float* tau2, size_t cells, float* quant, float* exact,
                            float* exact_prob, double* mse_cs, cudaStream_t s) {
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);  // kvcache.hpp:273
    cudaError_t e = launch_qk_scores(queries, codes, alpha, beta, samples, n, d, bits, word_bits, quant, s);
    if (e != cudaSuccess) return e;
    const size_t total = samples * n;
    scale_kernel<<<(unsigned)((total + 255) / 256 < 1184 ? (total + 255) / 256 : 1184), 256, 0, s>>>(quant, total,
                                                                                                    inv_sqrt_d);
    launch_exact_scores(queries, keys_exact, samples, n, d, inv_sqrt_d, exact, s);
    note_launch(2);
    // softmax of the exact rows: calibrated_softmax with tau = (0, 0) is the plain softmax
    e = launch_calibrated_softmax(exact, n, nullptr, 0, samples, 0.0f, 0.0f, exact_prob, nullptr, s);
    if (e != cudaSuccess) return e;
    dim3 gg((unsigned)cells, (unsigned)samples);
    grid_cell_kernel<<<gg, kThreads, 0, s>>>(quant, exact_prob, n, tau1, tau2, mse_cs, samples);
    note_launch();
    return cudaGetLastError();
}

}  // namespace kvqb
