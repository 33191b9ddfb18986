// kvq_internal.cuh — shared device-side declarations for the B200 kvq kernels.
//
// Layout contract (HBM), one "unit" = one (request, KV head) pair, u = b * kv_heads + h:
//   codes  [unit][n_vis][row_bytes]   reference byte layout (MSB-first codes in LE
//                                     M-bit words, rows padded to whole words;
//                                     bitpack.hpp:161-187, quantize.hpp:53-61)
//   alpha/beta [unit][dim] fp32        per-channel min/max (quantize.hpp:24-29)
//   tail   [unit][tail_cap][dim] fp32  append-only generated tokens (kvcache.hpp:99-109)
//   tail_len [batch] int32             device-resident so decode/append graph-capture
//   queries/out [unit][group][dim]     GQA: q head h*G+g reads KV head h
#pragma once
#include <cuda_runtime.h>
#include <cstddef>
#include <cstdint>
#include <mutex>

namespace kvqb {

// Status codes of the C-ABI (include/kvq_capi.h).
enum Status : int { OK = 0, CONFIG = 1, DOMAIN = 2, FORMAT = 3, CUDA = 4 };

__host__ __device__ inline int codes_per_word(int bits, int word_bits) { return word_bits / bits; }
__host__ __device__ inline size_t codes_per_row(size_t dim, int bits, int word_bits) {
    size_t g = (size_t)codes_per_word(bits, word_bits);
    return (dim + g - 1) / g * g;
}
__host__ __device__ inline size_t row_bytes(size_t dim, int bits, int word_bits) {
    return codes_per_row(dim, bits, word_bits) / (size_t)codes_per_word(bits, word_bits) *
           (size_t)(word_bits / 8);
}

// ---- K1: stats + quantize + pack ------------------------------------------
// x: [mats][rows][dim] fp32 (device). Writes alpha/beta [mats][dim] and codes
// [mats][rows][row_bytes]. mode 0 = channel_wise, 1 = global.
cudaError_t launch_compute_stats(const float* x, size_t mats, size_t rows, size_t dim, int mode,
                                 float* alpha, float* beta, cudaStream_t s);
cudaError_t launch_quantize_pack(const float* x, size_t mats, size_t rows, size_t dim,
                                 const float* alpha, const float* beta, int bits, int word_bits,
                                 uint8_t* codes, cudaStream_t s);
// K1 for the decode layout (d = 128, M = 8): stats kernel, then the warp-collective code
// pass of k1_fused.cu (coalesced rows, ballot / shuffle packing).
bool quantize_fused_supported(size_t rows, size_t dim, int word_bits, int mode);
cudaError_t launch_quantize_fused(const float* x, size_t mats, size_t rows, size_t dim, int bits, int word_bits,
                                  int mode, float* alpha, float* beta, uint8_t* codes, cudaStream_t s);
// Token-wise stats + codes (opt-in V mode; d = 128): alpha / beta [mats][rows], codes in
// the reference row layout (M-bit words).
cudaError_t launch_quantize_tokenwise(const float* x, size_t mats, size_t rows, int bits, int word_bits,
                                      float* alpha, float* beta, float2* step_off, uint8_t* codes, cudaStream_t s);
// Generic bit packing of explicit u32 codes (bitpack.hpp:161-187). err_flag set to 1 on
// an out-of-range code.
cudaError_t launch_pack_codes(const uint32_t* codes, size_t count, int bits, int word_bits,
                              uint8_t* out, int* err_flag, cudaStream_t s);
cudaError_t launch_unpack_codes(const uint8_t* bytes, size_t count, int bits, int word_bits,
                                uint32_t* out, cudaStream_t s);
cudaError_t launch_dequantize(const uint8_t* codes, size_t mats, size_t rows, size_t dim,
                              const float* alpha, const float* beta, int bits, int word_bits,
                              float* out, cudaStream_t s);

// ---- K2: decode --------------------------------------------------------------
struct DecodeArgs {
    const uint8_t* k_codes;
    const uint8_t* v_codes;
    const float* k_alpha;
    const float* k_beta;
    const float* v_alpha;
    const float* v_beta;
    const float* k_tail;
    const float* v_tail;
    const int* tail_len;  // [batch]
    const float* q;       // [units][group][dim]
    float* out;           // [units][group][dim]
    float* weights;       // nullable: [units][group][n_vis + tail_stride] probability rows
    int* violations;      // nullable: [units][group] g slope-violation flags
    float* scratch;       // generic path: [units][group][n_vis + tail_cap] score rows
    const uint8_t* v_codes_t;  // umma path: token-packed V codes (vt_layout, k2_decode_umma.cu)
    const uint8_t* v_codes_x;  // tc path: V codes as phase-B MMA operands (vx_layout, k2_decode_tc.cu)
    uint8_t* umma_qb;     // umma path: [units][NT][128][16] s8 q digit planes (prep kernel)
    float2* tc_qconst;    // umma path: [units][8] per-head score scale / offset (prep kernel)
    unsigned long long* trace;  // nullable: [ctas][64] globaltimer stamps (KVQ_TRACE_FILE)
    float* tail_lse;      // nullable: the fp32 tail is left to the tail pass (k2_tail.cu); the
                          // decode writes its base-2 log-sum-exp per (unit, head) here
    size_t units, kv_heads, group, dim, n_vis, tail_cap, weights_stride;
    size_t plan_units;    // 0, or the whole batch's units when `units` is one chunk of it: the
                          // split (and so the summation order) is the whole batch's
    size_t unit_base;     // first unit of this launch within the plan_units batch (chunks)
    int split_override;   // tensor-core decode: force this cluster size (0 = plan)
    int dequant_dot;      // generic path: dequantize-then-dot (BASELINE config 3's "without
                          // post-scaling" ablation) instead of the post-scaled products
    int dep_wait_at_end;  // tensor-core decode launched behind a sibling grid: skip the early
                          // dependency wait (the sibling did it), wait at exit instead
    // Fused append (tensor-core decode with the in-kernel tail): the step's new K / V rows
    // [units][dim] go to tail slot tail_len[request] (the reference's append after the
    // decode, kvcache.hpp:99-109); append_cnt [batch] counts the request's CTAs that read
    // tail_len, the last one bumps it. nullptr: no append.
    const float* k_new;
    const float* v_new;
    int* append_cnt;
    int* overflow;
    int v_token_wise;     // V stats per token (v_alpha / v_beta [units][n_vis]; opt-in mode,
                          // tensor-core decode only)
    const float2* v_tok_so;  // token-wise V: per token (step, alpha / step) [units][n_vis]
    int early_trigger;    // tensor-core decode: release dependents right after the dependency
                          // wait (a dependent that must overlap: the sibling grid) instead of
                          // after phase B
    int bits, word_bits;
    float tau1, tau2;
};
cudaError_t launch_decode_generic(const DecodeArgs& a, cudaStream_t s);
bool decode_tc_supported(const DecodeArgs& a);
size_t decode_tc_scratch_bytes(size_t units);
cudaError_t launch_decode_tc(const DecodeArgs& a, cudaStream_t s);
// fp32 tail pass (k2_tail.cu): attention over the dense tail rows, merged by log-sum-exp
// with the decode's output when `after_decode` (a.tail_lse set, launched right after it).
bool decode_tail_supported(const DecodeArgs& a);
cudaError_t launch_decode_tail(const DecodeArgs& a, bool after_decode, cudaStream_t s);
// Concurrent schedule: the tail pass writes (M, D, N[128]) per (unit, head) to `part`
// ([units][G][130]) on its own stream while the decode runs; launch_tail_merge combines.
cudaError_t launch_decode_tail_partials(const DecodeArgs& a, float* part, cudaStream_t s);
cudaError_t launch_tail_merge(const DecodeArgs& a, const float* part, cudaStream_t s);
#ifndef KVQ_TC_TAIL_MAX
#define KVQ_TC_TAIL_MAX 64
#endif
constexpr size_t kTcTailMax = KVQ_TC_TAIL_MAX;  // tail capacity the tensor-core decodes keep in-kernel
size_t vx_bytes(size_t units, size_t n_vis, int bits);
cudaError_t launch_unpack_vx(const uint8_t* vx, size_t units, size_t n_vis, int bits, int word_bits, uint8_t* rows,
                             cudaStream_t s);
cudaError_t launch_pack_vx(const uint8_t* rows, size_t units, size_t n_vis, int bits, int word_bits, uint8_t* vx,
                           cudaStream_t s);
// tcgen05 (UTCIMMA) path, d = 128, M = 8: needs the token-packed V copy.
size_t vt_bytes(size_t units, size_t n_vis, int bits);
cudaError_t launch_pack_vt(const uint8_t* rows, size_t units, size_t n_vis, int bits, uint8_t* vt, cudaStream_t s);
bool decode_umma_supported(const DecodeArgs& a);
size_t decode_umma_scratch_bytes(size_t units);
cudaError_t launch_decode_umma(const DecodeArgs& a, cudaStream_t s);

// Post-scaled q.K (kernels.hpp:302-363) and w.V (316-396) over `heads` segments.
cudaError_t launch_qk_scores(const float* q, const uint8_t* codes, const float* alpha,
                             const float* beta, size_t heads, size_t tokens, size_t dim,
                             int bits, int word_bits, float* scores, cudaStream_t s);
cudaError_t launch_wv_output(const float* w, const uint8_t* codes, const float* alpha,
                             const float* beta, size_t heads, size_t tokens, size_t dim,
                             int bits, int word_bits, float* out, cudaStream_t s);
// Dense fp32 products of the tail / full-precision baseline (kernels.hpp:401-426).
cudaError_t launch_naive_qk(const float* q, const float* k, size_t rows, size_t cols, float* out, cudaStream_t s);
cudaError_t launch_naive_wv(const float* w, const float* v, size_t rows, size_t cols, float* out, cudaStream_t s);
// calibrated_softmax_concat (calibrate.hpp:100-114) over `rows` independent rows.
cudaError_t launch_calibrated_softmax(const float* vis, size_t n_vis, const float* tail,
                                      size_t n_tail, size_t rows, float tau1, float tau2,
                                      float* out, int* violations, cudaStream_t s);

// Offline tau search (k_grid.cu, calibrate.hpp:160-234): per (cell, sample) softmax MSE.
cudaError_t launch_grid_mse(const float* queries, const float* keys_exact, const uint8_t* codes, const float* alpha,
                            const float* beta, size_t samples, size_t n, size_t d, int bits, int word_bits,
                            const float* tau1, const float* tau2, size_t cells, float* quant, float* exact,
                            float* exact_prob, double* mse_cs, cudaStream_t s);
// mse_report (calibrate.hpp:300-351) for `heads` heads of equal shape: K1 stats + codes into
// alpha/beta [heads][d] and codes, quant / exact / qc rows [heads][n] (scratch), edges
// [heads][bins+1], counts [heads][3][bins] (exact, quant, quant_c), MSEs [heads].
cudaError_t launch_mse_report(const float* queries, const float* keys, size_t heads, size_t n, size_t d, int bits,
                              int mode, int word_bits, float tau1, float tau2, size_t bins, float* alpha, float* beta,
                              uint8_t* codes, float* quant, float* exact, float* qc, float* edges,
                              unsigned long long* counts, double* mse_q, double* mse_qc, cudaStream_t s);

// ---- K3: append --------------------------------------------------------------
// `overflow` (device int) is set instead of writing past tail_cap.
cudaError_t launch_append(const float* k_new, const float* v_new, size_t batch, size_t kv_heads,
                          size_t dim, size_t tail_cap, float* k_tail, float* v_tail,
                          int* tail_len, int* overflow, cudaStream_t s);

// ---- misc -------------------------------------------------------------------------
// Kernel function attributes (dynamic shared memory above 48 KB, non-portable cluster
// sizes) are per device: `set` runs once per (kernel instantiation, device), under a lock so
// concurrent first launches from several host threads never race past it.
template <typename F>
inline cudaError_t once_per_device(unsigned& mask, F&& set) {
    static std::mutex m;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 32) return set();
    std::lock_guard<std::mutex> lock(m);
    if (mask & (1u << dev)) return cudaSuccess;
    e = set();
    if (e == cudaSuccess) mask |= 1u << dev;
    return e;
}

// Number of this library's kernels launched so far (bench.py's gpu_launches claim).
unsigned long long launch_count();
void note_launch(unsigned n = 1);

}  // namespace kvqb
