/*
 * kvq_capi.h — C-ABI of the B200-native CalibQuant decode hot path.
 *
 * This is the drop-in boundary. Every entry point replaces one function of the
 * reference's header-only C++ API (`kvq`, headers under /root/reference/proj/include/kvq/;
 * cited per function below) and is what the C++ drop-in headers in include/kvq/ and
 * the Python binding (paper_2502_14882_b200/kvq.py) bind. Plain pointers and sizes
 * only: no CUDA, torch or C++ types cross this boundary.
 *
 * Conventions
 *   - Return value: KVQ_OK or an error class matching the reference's exception types
 *     (errors.hpp:11-33): KVQ_ERR_CONFIG <-> kvq::config_error, KVQ_ERR_DOMAIN <->
 *     kvq::domain_error, KVQ_ERR_FORMAT <-> kvq::format_error; KVQ_ERR_CUDA for device
 *     failures. kvq_last_error() returns the message of the calling thread's last error.
 *   - Unless the name ends in _device, pointers are HOST memory; the call copies in,
 *     runs the CUDA kernels, copies out and synchronizes. _device entry points take
 *     device pointers and a cudaStream_t passed as void* (NULL = legacy default stream)
 *     and do not synchronize.
 *   - Matrices are row-major fp32 (matrix.hpp:16-60). Packed codes use the reference
 *     byte layout bit for bit (bitpack.hpp:15-90, quantize.hpp:46-62).
 *   - There is no CPU fallback: without a usable CUDA device every compute entry point
 *     returns KVQ_ERR_CUDA.
 */
#ifndef KVQ_CAPI_H
#define KVQ_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KVQ_OK 0
#define KVQ_ERR_CONFIG 1
#define KVQ_ERR_DOMAIN 2
#define KVQ_ERR_FORMAT 3
#define KVQ_ERR_CUDA 4

#define KVQ_MODE_CHANNEL_WISE 0 /* QuantMode::channel_wise (quantize.hpp:31) */
#define KVQ_MODE_GLOBAL 1       /* QuantMode::global */
/* Opt-in extension (not in the reference): K channel-wise, V token-wise - min / max per
 * visual token over its d channels (north_star; KIVI's V axis). Caches only: d = 128, a
 * quantized prefill, the tensor-core decode (no generic-path export, no KVQC snapshot, no
 * per-channel V segment stats: kvq_cache_read_value_token_stats reads them). */
#define KVQ_MODE_V_TOKEN_WISE 2
#define KVQ_FULL_PRECISION_BITS 16 /* kvcache.hpp:26 */

#define KVQ_PATH_AUTO 0    /* per-CTA IMMA path when the shape allows, else tcgen05, else generic */
#define KVQ_PATH_GENERIC 1 /* any shape; also the path that emits probability rows */
#define KVQ_PATH_TC 2      /* d = 128, M = 8 legacy mma.sync IMMA path (KVQ_ERR_CONFIG otherwise) */
#define KVQ_PATH_UMMA 3    /* d = 128, M = 8 tcgen05 UTCIMMA path (KVQ_ERR_CONFIG otherwise) */
#define KVQ_PATH_DEQUANT 4 /* BASELINE c3 ablation: generic decode, dequantize-then-dot (no post-scaling) */

/* ---- diagnostics ------------------------------------------------------------ */
/* Copies the calling thread's last error message (NUL-terminated, truncated to cap);
 * returns its full length. */
size_t kvq_last_error(char* buf, size_t cap);
/* Byte offset carried by the calling thread's last KVQ_ERR_FORMAT (format_error::offset,
 * errors.hpp:23-33). */
unsigned long long kvq_last_error_offset(void);
/* Number of CUDA kernels this library has launched in this process. */
unsigned long long kvq_launch_count(void);
/* 1 if a CUDA device is usable (the library never falls back to the CPU). */
int kvq_device_available(void);
/* Bind the calling thread's CUDA device (one process per GPU): every later
   cache of this thread lives on `device`. No reference counterpart (the reference is CPU). */
int kvq_set_device(int device);

/* ---- bitpack.hpp ------------------------------------------------------------- */
/* Bytes `pack` produces for `count` codes (PackedBuffer::word_count, bitpack.hpp:22-25). */
size_t kvq_packed_bytes(size_t count, int code_bits, int word_bits);
/* kvq::pack (bitpack.hpp:161-187). out must hold kvq_packed_bytes(...) bytes.
 * CONFIG on bad widths (bitpack.hpp:141-149), DOMAIN on a code >= 2^code_bits. */
int kvq_pack(const uint32_t* codes, size_t count, int code_bits, int word_bits, uint8_t* out,
             size_t out_cap);
/* kvq::unpack (bitpack.hpp:189-203): `count` = PackedBuffer::logical_count. */
int kvq_unpack(const uint8_t* bytes, size_t byte_len, size_t count, int code_bits, int word_bits,
               uint32_t* out);

/* ---- quantize.hpp ------------------------------------------------------------ */
/* Bytes of one packed segment: tokens * words_per_row * M/8 (quantize.hpp:56-61). */
size_t kvq_segment_bytes(size_t tokens, size_t dim, int bitwidth, int word_bits);
/* kvq::compute_stats (quantize.hpp:64-89). alpha/beta: cols floats each. */
int kvq_compute_stats(const float* m, size_t rows, size_t cols, int mode, float* alpha,
                      float* beta);
/* kvq::quantize (quantize.hpp:91-127): codes of m under the given stats, packed. */
int kvq_quantize(const float* m, size_t rows, size_t cols, const float* alpha, const float* beta,
                 int bitwidth, int word_bits, uint8_t* out, size_t out_cap);
/* kvq::dequantize (quantize.hpp:129-146). out: rows x cols. */
int kvq_dequantize(const uint8_t* codes, size_t rows, size_t cols, const float* alpha,
                   const float* beta, int bitwidth, int word_bits, float* out);
/* Batched device K1: `mats` fp32 matrices [mats][rows][dim] -> stats [mats][dim] and
 * codes [mats][rows][row_bytes] (compute_stats + quantize per matrix). */
int kvq_quantize_device(const float* x, size_t mats, size_t rows, size_t dim, int bitwidth,
                        int mode, int word_bits, uint8_t* codes, float* alpha, float* beta,
                        void* stream);

/* ---- kernels.hpp ------------------------------------------------------------- */
/* kvq::qk_scores, batched form (kernels.hpp:342-363; single form 302-314 is heads=1):
 * queries [heads][dim], codes [heads][tokens][row_bytes], alpha/beta [heads][dim]
 * -> scores [heads][tokens] = post-scaled q.K (no 1/sqrt(d)). */
int kvq_qk_scores(const float* queries, const uint8_t* codes, const float* alpha,
                  const float* beta, size_t heads, size_t tokens, size_t dim, int bitwidth,
                  int word_bits, float* scores);
/* kvq::wv_output, batched form (kernels.hpp:365-396; single 316-336): weights
 * [heads][tokens] -> out [heads][dim]. */
int kvq_wv_output(const float* weights, const uint8_t* codes, const float* alpha,
                  const float* beta, size_t heads, size_t tokens, size_t dim, int bitwidth,
                  int word_bits, float* out);

/* kvq::naive_qk (kernels.hpp:401-413): dense q . k_j for every row of k [rows][cols]. */
int kvq_naive_qk(const float* q, const float* k, size_t rows, size_t cols, float* out);
/* kvq::naive_wv (kernels.hpp:415-426): sum_j w_j v_j over the rows of v [rows][cols]. */
int kvq_naive_wv(const float* w, const float* v, size_t rows, size_t cols, float* out);

/* ---- calibrate.hpp ----------------------------------------------------------- */
/* kvq::calibrated_softmax_concat (calibrate.hpp:100-114) over `rows` rows:
 * vis [rows][n_vis], tail [rows][n_tail] -> out [rows][n_vis + n_tail]. Adds the number
 * of g slope violations (calibrate.hpp:52-54) to *slope_violations if non-NULL. */
int kvq_calibrated_softmax_concat(const float* vis, size_t n_vis, const float* tail,
                                  size_t n_tail, size_t rows, float tau1, float tau2, float* out,
                                  size_t* slope_violations);

/* kvq::grid_mse_table + kvq::grid_search (calibrate.hpp:160-234), offline tau search on
 * the device: `samples` calibration samples (queries [S][dim], exact keys [S][tokens][dim],
 * packed keys [S][tokens][row_bytes] with stats alpha/beta [S][dim]) scored against `cells`
 * candidate (tau1[c], tau2[c]) pairs. mse[c] (nullable) receives the mean softmax MSE per
 * cell; best_tau (nullable) the argmin, ties to the smaller tau1, then tau2. DOMAIN on an
 * empty set or grid. */
int kvq_grid_mse_table(const float* queries, const float* keys_exact, const uint8_t* codes,
                       const float* alpha, const float* beta, size_t samples, size_t tokens,
                       size_t dim, int bitwidth, int word_bits, const float* tau1, const float* tau2,
                       size_t cells, double* mse, float* best_tau);

/* kvq::mse_report (calibrate.hpp:300-351) for `heads` heads of equal shape (queries
 * [heads][dim], keys [heads][tokens][dim]): each head's keys are quantized with its own
 * stats (bitwidth, mode, word_bits), and its exact, quantized and calibrated (tau1, tau2)
 * pre-softmax rows are compared. Per head: mse_quant / mse_quant_c [heads] (softmax MSE vs
 * the exact row), edges [heads][bins+1] (shared by the three rows), counts
 * [heads][3][bins] in ScoreVariant order (exact, quant, quant_c). Any output may be NULL.
 * DOMAIN on no heads or an empty matrix, CONFIG on bins < 1 or a bad configuration. */
int kvq_mse_report(const float* queries, const float* keys, size_t heads, size_t tokens,
                   size_t dim, int bitwidth, int mode, int word_bits, float tau1, float tau2,
                   size_t bins, double* mse_quant, double* mse_quant_c, float* edges,
                   uint64_t* counts);

/* ---- kvcache.hpp: HybridKVCache ---------------------------------------------- */
/* A device-resident hybrid cache for `batch` independent sequences of `kv_heads` KV
 * heads each; every KV head serves `group` query heads (GQA). batch = 1, group = 1 is
 * exactly one reference HybridKVCache with kv_heads heads. */
typedef struct kvq_cache kvq_cache;

/* HybridKVCache::build (kvcache.hpp:48-66): k_vis/v_vis [batch][kv_heads][n_vis][dim].
 * bitwidth = KVQ_FULL_PRECISION_BITS gives build_full_precision (69-83): the prefill
 * becomes the fp32 tail. n_vis = 0 gives an empty prefill (pure fp32 cache). */
int kvq_cache_build(const float* k_vis, const float* v_vis, size_t batch, size_t kv_heads,
                    size_t group, size_t n_vis, size_t dim, int bitwidth, int mode, int word_bits,
                    float tau1, float tau2, kvq_cache** out);
/* Same, prefill already on the device (no host round trip). */
int kvq_cache_build_device(const float* k_vis, const float* v_vis, size_t batch, size_t kv_heads,
                           size_t group, size_t n_vis, size_t dim, int bitwidth, int mode,
                           int word_bits, float tau1, float tau2, void* stream, kvq_cache** out);
void kvq_cache_free(kvq_cache* c);
/* Preallocate fp32 tail capacity (rows per unit); append grows it on demand. */
int kvq_cache_reserve_tail(kvq_cache* c, size_t rows);
/* Reconcile the host tail counter with the device (appends issued on user streams or
   replayed from captured graphs advance it on the device only); KVQ_ERR_DOMAIN if appends
   were dropped at a full tail. info / memory / read_tail / save_image do this implicitly. */
int kvq_cache_sync_tail(kvq_cache* c);
/* Decode kernel selection (KVQ_PATH_*); never changes results beyond fp tolerance. */
int kvq_cache_set_path(kvq_cache* c, int path);

/* HybridKVCache::append (kvcache.hpp:99-109): k_new/v_new [batch][kv_heads][dim]. */
int kvq_cache_append(kvq_cache* c, const float* k_new, const float* v_new);
int kvq_cache_append_device(kvq_cache* c, const float* k_new, const float* v_new, void* stream);

/* HybridKVCache::decode_step / decode_step_detailed (kvcache.hpp:111-121, 263-311):
 * queries [batch][kv_heads][group][dim] -> out, same shape. weights (nullable) receives
 * [batch][kv_heads][group][n_vis + n_tail] probability rows; slope_violations (nullable)
 * receives the DecodeDetail::slope_violations count. */
int kvq_cache_decode(kvq_cache* c, const float* queries, float* out, float* weights,
                     size_t* slope_violations);
int kvq_cache_decode_device(kvq_cache* c, const float* queries, float* out, void* stream);
/* decode_step(queries) then append(k_new, v_new) on device buffers and a user stream
 * (graph-capturable): one kernel when the tensor-core decode owns the fp32 tail in-kernel
 * (it writes the new rows and moves tail_len on after every unit read it), else the decode
 * and the append kernel. Same results as kvq_cache_decode_device + kvq_cache_append_device. */
int kvq_cache_step_device(kvq_cache* c, const float* queries, const float* k_new, const float* v_new,
                          float* out, void* stream);

/* One serving step through host buffers, in the reference bench order (kvq_main.cpp:
 * 313-321): decode_step(queries) then append(k_new, v_new). Host->device copies, both
 * kernels and the device->host copy of `out` are issued on one stream, one sync. */
int kvq_cache_step(kvq_cache* c, const float* queries, const float* k_new, const float* v_new,
                   float* out);

/* Accessors (kvcache.hpp:85-96). info: batch, kv_heads, group, dim, n_vis, n_tail,
 * bitwidth, word_bits, mode, tail_capacity. */
int kvq_cache_info(const kvq_cache* c, size_t info[10]);
int kvq_cache_calibration(const kvq_cache* c, float tau[2]);
/* CacheMemory (kvcache.hpp:28-35, 123-135): code, stats, quantized, tail, fp32_vis, total. */
int kvq_cache_memory(const kvq_cache* c, size_t mem[6]);
/* Device bytes actually resident for the packed codes (no reference counterpart; the
   reference holds one copy, kvcache.hpp:123-135): [0] K rows, [1] V rows (reference layout,
   0 when V lives only in the decode's operand layout), [2] V operand layout (vx),
   [3] derived layouts built on demand (tcgen05 V, rebuilt V rows). */
int kvq_cache_resident_bytes(const kvq_cache* c, size_t bytes[4]);
/* key_segment / value_segment (93-94) of unit u = b*kv_heads + h, which 0 = K, 1 = V:
 * bytes (kvq_segment_bytes(n_vis, ...)) in the reference layout, alpha/beta [dim]. */
int kvq_cache_read_segment(const kvq_cache* c, size_t unit, int which, uint8_t* bytes,
                           float* alpha, float* beta);
/* key_tail / value_tail (95-96): [n_tail][dim] fp32. */
int kvq_cache_read_tail(const kvq_cache* c, size_t unit, int which, float* out);
/* Token-wise V caches (KVQ_MODE_V_TOKEN_WISE): the V stats of one unit, alpha / beta [n_vis]. */
int kvq_cache_read_value_token_stats(const kvq_cache* c, size_t unit, float* alpha, float* beta);
/* Raw device pointers (k_codes, v_codes, k_alpha, k_beta, v_alpha, v_beta, k_tail, v_tail,
 * tail_len) for zero-copy integration with a serving engine. */
int kvq_cache_device_pointers(const kvq_cache* c, void* ptrs[9]);

/* ---- cache snapshots (HybridKVCache::save / load, kvcache.hpp:137-218) -------------
 * The image is the reference's KVQC byte stream: manifest, then per unit ("head") a KVQP
 * K segment, a KVQP V segment, a KVQT K tail and a KVQT V tail (quantize.hpp:148-230,
 * tensor_io.hpp:11-128), little-endian, byte-identical to the reference's save(). */
int kvq_cache_image_bytes(const kvq_cache* c, size_t* bytes);
/* Writes the image into `image` (host memory, or device memory when image_on_device) of
 * `capacity` bytes; stream NULL = the cache's stream. DOMAIN if the buffer is too small. */
int kvq_cache_save_image(const kvq_cache* c, void* image, size_t capacity, int image_on_device,
                         void* stream);
/* Parses and validates an image in host memory (the reference's format_error messages and
 * byte offsets, kvq_last_error_offset) and builds a device cache of `batch` requests
 * (heads / batch KV heads each) with query group `group`. *consumed (nullable) = the
 * image's length; bytes beyond it are left to the caller (file loads reject them). */
int kvq_cache_load_image(const void* image, size_t bytes, size_t batch, size_t group,
                         size_t* consumed, kvq_cache** out);

/* ---- multi-GPU split (no reference counterpart - the reference splits a
 * request's heads over std::thread, kvcache.hpp:272-274, and has no multi-device code) ------
 * The (request, KV head) units rank `rank` of `world` owns, as global indices u = b * H + h:
 * contiguous request slices when batch >= world, else round-robin. *count = the share size;
 * units (nullable) receives it (DOMAIN when capacity is smaller). */
int kvq_shard_assign(size_t batch, size_t kv_heads, int world, int rank, long long* units, size_t capacity,
                     size_t* count);
/* The gather's last hop on the destination rank: `parts` (device) = [world][width] floats,
 * rank r's output rows ([share_r][row], row = group * dim, in kvq_shard_assign order) at
 * parts + r * width; scattered to out [batch * kv_heads][row] (host, or device when
 * out_on_device) by one kernel on `stream`, then synchronised. */
int kvq_shard_place(const float* parts, int world, size_t width, size_t batch, size_t kv_heads, size_t row,
                    float* out, int out_on_device, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* KVQ_CAPI_H */
