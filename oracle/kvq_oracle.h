/*
 * kvq_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * Plain-C restatement of the CalibQuant `kvq` reference hot path
 * (the reference headers under /root/reference/proj/include/kvq/). Every function cites the reference
 * file:line it follows and keeps the reference's fp32 evaluation order so that,
 * compiled with the reference's own flags (no FMA contraction), it reproduces the
 * reference bit for bit. It is pinned against the reference compiled from its
 * own headers (oracle/_ref/libkvq_ref.so, see oracle/Makefile) and against the
 * reference's golden vectors (tests/test_oracle.py, tests/golden/).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this code. The CUDA product path never links it.
 *
 * Deliberate deviation: the reference's qK byte-table path indexes the scaled
 * query with `w * 8` (kernels.hpp:220) instead of `w * codes_per_word`, which is
 * a heap over-read and wrong scores for bitwidth >= 2 at M = 8 and n >= 512
 * (SURVEY.md §0.4). The oracle uses `w * codes_per_word`; for b = 1 the two are
 * identical, for b >= 2 the oracle matches the reference's M = 32 wide path and
 * its dequantize-then-dense path (checked in tests/test_oracle.py).
 */
#ifndef KVQ_ORACLE_H
#define KVQ_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { KVQO_OK = 0, KVQO_CONFIG = 1, KVQO_DOMAIN = 2 };
enum { KVQO_CHANNEL_WISE = 0, KVQO_GLOBAL = 1 };

/* quantize.hpp:46-62 — packed geometry of one segment. */
size_t kvqo_codes_per_row(size_t dim, int bits, int word_bits);
size_t kvqo_row_bytes(size_t dim, int bits, int word_bits);

/* bitpack.hpp:141-149 + quantize.hpp:38-43 */
int kvqo_validate(int bits, int word_bits);

/* bitpack.hpp:161-187: MSB-first pack of `count` codes into LE words. */
int kvqo_pack(const uint32_t* codes, size_t count, int bits, int word_bits, uint8_t* out);
/* bitpack.hpp:189-203 */
int kvqo_unpack(const uint8_t* bytes, size_t count, int bits, int word_bits, uint32_t* out);

/* quantize.hpp:64-89 */
int kvqo_compute_stats(const float* m, size_t rows, size_t cols, int mode, float* alpha,
                       float* beta);
/* quantize.hpp:91-127 (codes + pack). out has rows * row_bytes bytes. */
int kvqo_quantize(const float* m, size_t rows, size_t cols, const float* alpha,
                  const float* beta, int bits, int word_bits, uint8_t* out);
/* quantize.hpp:129-146 */
void kvqo_dequantize(const uint8_t* bytes, size_t rows, size_t cols, const float* alpha,
                     const float* beta, int bits, int word_bits, float* out);

/* kernels.hpp:245-267 (+183-243, 65-82, 98-112): post-scaled q.K over one packed
 * segment; no 1/sqrt(d). */
void kvqo_qk_scores(const float* q, const uint8_t* bytes, size_t tokens, size_t dim,
                    const float* alpha, const float* beta, int bits, int word_bits,
                    float* scores);
/* kernels.hpp:316-336 (+269-284, 84-95, 114-127) */
void kvqo_wv_output(const float* w, const uint8_t* bytes, size_t tokens, size_t dim,
                    const float* alpha, const float* beta, int bits, int word_bits,
                    float* out);
/* kernels.hpp:401-413, 415-426 */
void kvqo_naive_qk(const float* q, const float* k, size_t rows, size_t cols, float* out);
void kvqo_naive_wv(const float* w, const float* v, size_t rows, size_t cols, float* out);

/* calibrate.hpp:62-67 */
float kvqo_g_apply(float x, float gamma, float delta, float tau1, float tau2);
/* calibrate.hpp:77-87 */
void kvqo_softmax_inplace(float* row, size_t n);
/* calibrate.hpp:100-114; out has n_vis + n_tail entries. */
void kvqo_calibrated_softmax_concat(const float* vis, size_t n_vis, const float* tail,
                                    size_t n_tail, float tau1, float tau2, float* out,
                                    size_t* slope_violations);

/* kvcache.hpp:263-311 for ONE head: quantized segment (K and V share tokens/dim/bits)
 * plus fp32 tails of n_tail rows. weights (nullable) gets n_vis + n_tail entries. */
void kvqo_decode_head(const float* q, size_t dim, size_t n_vis, int bits, int word_bits,
                      const uint8_t* k_bytes, const float* k_alpha, const float* k_beta,
                      const uint8_t* v_bytes, const float* v_alpha, const float* v_beta,
                      const float* k_tail, const float* v_tail, size_t n_tail, float tau1,
                      float tau2, float* out, float* weights, size_t* slope_violations);

/* workload.hpp:85-201: mt19937_64 + Marsaglia polar generator, bit-identical to
 * kvq::generate / kvq::generate_step for Distribution::gaussian. Fills one head's
 * keys (tokens x dim), values (tokens x dim) and query (dim). */
void kvqo_generate_head(uint64_t seed, uint64_t head, size_t tokens, size_t dim, double mean,
                        double stddev, float* keys, float* values, float* query);
void kvqo_generate_step_head(uint64_t seed, uint64_t head, uint64_t step, size_t dim,
                             double mean, double stddev, float* query, float* key,
                             float* value);

/* reference.hpp:26-54: double-precision attention (ground truth, tau = 0). */
void kvqo_oracle_attention(const float* q, const float* k, const float* v, size_t n,
                           size_t dim, float* out);

/* grid_mse_table / grid_search (calibrate.hpp:160-234). */
void kvqo_grid_mse_table(const float* queries, const float* keys_exact, const uint8_t* codes,
                         const float* alpha, const float* beta, size_t samples, size_t n,
                         size_t d, int bits, int word_bits, const float* tau1, const float* tau2,
                         size_t cells, double* mse, float* best);
/* calibrate.hpp:300-351 */
int kvqo_mse_report(const float* queries, const float* keys, size_t heads, size_t n, size_t d, int mode,
                    int bits, int word_bits, float tau1, float tau2, size_t bins, double* mse_q,
                    double* mse_qc, float* edges, uint64_t* counts);

#ifdef __cplusplus
}
#endif
#endif
