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

// exact[s][j] = (q_s . k_sj) / sqrt(d) (naive_qk, kernels.hpp:401-413, then 284-style scale)
__global__ void exact_scores_kernel(const float* __restrict__ q, const float* __restrict__ k, size_t n, size_t d,
                                    float inv_sqrt_d, float* __restrict__ out) {
    const size_t s = blockIdx.y;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (size_t j = (size_t)blockIdx.x * (kThreads / 32) + warp; j < n; j += (size_t)gridDim.x * (kThreads / 32)) {
        const float* kr = k + (s * n + j) * d;
        const float* qr = q + s * d;
        float acc = 0.0f;
        for (size_t c = lane; c < d; c += 32) acc = fmaf(qr[c], kr[c], acc);
#pragma unroll
        for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (lane == 0) out[s * n + j] = acc * inv_sqrt_d;
    }
}

__global__ void scale_kernel(float* x, size_t count, float f) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
        x[i] *= f;
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

}  // namespace

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
    dim3 eg((unsigned)((n + 7) / 8 < 1024 ? (n + 7) / 8 : 1024), (unsigned)samples);
    exact_scores_kernel<<<eg, kThreads, 0, s>>>(queries, keys_exact, n, d, inv_sqrt_d, exact);
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
