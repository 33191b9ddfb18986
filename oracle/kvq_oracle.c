/*
 * kvq_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the kvq reference
 * hot path; see kvq_oracle.h for scope and pinning. Compile WITHOUT fast-math and
 * with -ffp-contract=off so every fp32 operation rounds exactly as the reference's
 * own -O3 x86-64 build does (no FMA in the baseline ISA).
 */
#include "kvq_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- geometry / validation ------------------------------------------------ */

int kvqo_validate(int bits, int word_bits) {
    /* quantize.hpp:38-43 (bitwidth set) then bitpack.hpp:141-149 (widths). */
    if (bits != 1 && bits != 2 && bits != 4 && bits != 8) return KVQO_CONFIG;
    if (word_bits < 8 || word_bits > 32 || word_bits % 8 != 0) return KVQO_CONFIG;
    if (word_bits % bits != 0) return KVQO_CONFIG;
    return KVQO_OK;
}

static size_t group_of(int bits, int word_bits) { return (size_t)(word_bits / bits); }

size_t kvqo_codes_per_row(size_t dim, int bits, int word_bits) {
    /* quantize.hpp:56-59 */
    size_t g = group_of(bits, word_bits);
    return (dim + g - 1) / g * g;
}

size_t kvqo_row_bytes(size_t dim, int bits, int word_bits) {
    /* quantize.hpp:61 words_per_row times M/8 bytes per word */
    return kvqo_codes_per_row(dim, bits, word_bits) / group_of(bits, word_bits) *
           (size_t)(word_bits / 8);
}

static uint32_t word_at(const uint8_t* bytes, size_t i, int word_bits) {
    /* bitpack.hpp:29-36: little-endian words */
    size_t nb = (size_t)word_bits / 8;
    uint32_t w = 0;
    for (size_t b = 0; b < nb; ++b) w |= (uint32_t)bytes[i * nb + b] << (8 * b);
    return w;
}

/* ---- bitpack.hpp ----------------------------------------------------------- */

int kvqo_pack(const uint32_t* codes, size_t count, int bits, int word_bits, uint8_t* out) {
    /* bitpack.hpp:161-187 */
    if (bits < 1 || word_bits < 8 || word_bits > 32 || word_bits % 8 != 0 ||
        word_bits % bits != 0)
        return KVQO_CONFIG;
    const uint32_t limit = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
    const size_t group = group_of(bits, word_bits);
    const size_t words = (count + group - 1) / group;
    const size_t nb = (size_t)word_bits / 8;
    for (size_t w = 0; w < words; ++w) {
        uint32_t acc = 0;
        for (size_t i = 0; i < group; ++i) {
            size_t idx = w * group + i;
            uint32_t code = idx < count ? codes[idx] : 0u;
            if (code > limit) return KVQO_DOMAIN;
            acc |= code << (word_bits - bits * (int)(i + 1));
        }
        for (size_t b = 0; b < nb; ++b) out[w * nb + b] = (uint8_t)(acc >> (8 * b));
    }
    return KVQO_OK;
}

int kvqo_unpack(const uint8_t* bytes, size_t count, int bits, int word_bits, uint32_t* out) {
    /* bitpack.hpp:189-203 */
    if (bits < 1 || word_bits < 8 || word_bits > 32 || word_bits % 8 != 0 ||
        word_bits % bits != 0)
        return KVQO_CONFIG;
    const size_t group = group_of(bits, word_bits);
    const uint32_t mask = bits >= 32 ? 0xffffffffu : (1u << bits) - 1u;
    for (size_t idx = 0; idx < count; ++idx) {
        uint32_t word = word_at(bytes, idx / group, word_bits);
        size_t i = idx % group;
        int shift = word_bits - bits * (int)(i + 1);
        out[idx] = (word >> shift) & mask;
    }
    return KVQO_OK;
}

/* ---- quantize.hpp ---------------------------------------------------------- */

/* std::min / std::max semantics: keep the left operand unless the right one is
 * strictly smaller / larger (so the first of equal values, e.g. -0 vs +0, wins). */
static inline float ref_min(float a, float b) { return b < a ? b : a; }
static inline float ref_max(float a, float b) { return a < b ? b : a; }

int kvqo_compute_stats(const float* m, size_t rows, size_t cols, int mode, float* alpha,
                       float* beta) {
    /* quantize.hpp:64-89 */
    if (rows == 0 || cols == 0) return KVQO_DOMAIN;
    if (mode == KVQO_CHANNEL_WISE) {
        for (size_t c = 0; c < cols; ++c) { /* column-outer, row-inner (70-78) */
            float lo = m[c], hi = m[c];
            for (size_t r = 1; r < rows; ++r) {
                lo = ref_min(lo, m[r * cols + c]);
                hi = ref_max(hi, m[r * cols + c]);
            }
            alpha[c] = lo;
            beta[c] = hi;
        }
    } else {
        float lo = m[0], hi = m[0]; /* row-major fold over all entries (79-87) */
        for (size_t i = 0; i < rows * cols; ++i) {
            lo = ref_min(lo, m[i]);
            hi = ref_max(hi, m[i]);
        }
        for (size_t c = 0; c < cols; ++c) {
            alpha[c] = lo;
            beta[c] = hi;
        }
    }
    return KVQO_OK;
}

int kvqo_quantize(const float* m, size_t rows, size_t cols, const float* alpha,
                  const float* beta, int bits, int word_bits, uint8_t* out) {
    /* quantize.hpp:91-127 */
    int st = kvqo_validate(bits, word_bits);
    if (st) return st;
    const float levels = (float)((1u << bits) - 1u);
    const size_t stride = kvqo_codes_per_row(cols, bits, word_bits);
    float* inv_step = (float*)malloc(sizeof(float) * (cols ? cols : 1));
    uint32_t* codes = (uint32_t*)calloc(rows * stride + 1, sizeof(uint32_t));
    for (size_t c = 0; c < cols; ++c) { /* 102-106 */
        float range = beta[c] - alpha[c];
        inv_step[c] = range > 0.0f ? levels / range : 0.0f;
    }
    for (size_t r = 0; r < rows; ++r) { /* 109-118 */
        const float* src = m + r * cols;
        uint32_t* dst = codes + r * stride;
        for (size_t c = 0; c < cols; ++c) {
            float t = roundf((src[c] - alpha[c]) * inv_step[c]); /* half away from zero */
            /* std::clamp(t, 0, levels): t < 0 ? 0 : (levels < t ? levels : t) */
            t = t < 0.0f ? 0.0f : (levels < t ? levels : t);
            dst[c] = t != t ? 0u : (uint32_t)t; /* NaN -> 0 as x86 cvttss2si/trunc does */
        }
    }
    st = kvqo_pack(codes, rows * stride, bits, word_bits, out);
    free(codes);
    free(inv_step);
    return st;
}

void kvqo_dequantize(const uint8_t* bytes, size_t rows, size_t cols, const float* alpha,
                     const float* beta, int bits, int word_bits, float* out) {
    /* quantize.hpp:129-146 */
    const float levels = (float)((1u << bits) - 1u);
    const size_t stride = kvqo_codes_per_row(cols, bits, word_bits);
    uint32_t* codes = (uint32_t*)malloc(sizeof(uint32_t) * (rows * stride + 1));
    kvqo_unpack(bytes, rows * stride, bits, word_bits, codes);
    for (size_t r = 0; r < rows; ++r) {
        for (size_t c = 0; c < cols; ++c) {
            float range = beta[c] - alpha[c];
            float step = range > 0.0f ? range / levels : 0.0f;
            out[r * cols + c] = (float)codes[r * stride + c] * step + alpha[c];
        }
    }
    free(codes);
}

/* ---- kernels.hpp ----------------------------------------------------------- */

/* ByteTable<N> entry k of byte v (kernels.hpp:46-63). */
static inline float lut(int bits, unsigned v, int k) {
    return (float)((v >> (8 - bits * (k + 1))) & ((1u << bits) - 1u));
}

/* detail::scale_query (kernels.hpp:183-194); qs has codes_per_row entries. */
static float scale_query(const float* q, size_t dim, const float* alpha, const float* beta,
                         int bits, size_t cpr, float* qs) {
    const float levels = (float)((1u << bits) - 1u);
    for (size_t c = 0; c < cpr; ++c) qs[c] = 0.0f;
    float qdota = 0.0f;
    for (size_t c = 0; c < dim; ++c) {
        float range = beta[c] - alpha[c];
        qs[c] = range > 0.0f ? q[c] * (range / levels) : 0.0f;
        qdota += q[c] * alpha[c];
    }
    return qdota;
}

void kvqo_qk_scores(const float* q, const uint8_t* bytes, size_t tokens, size_t dim,
                    const float* alpha, const float* beta, int bits, int word_bits,
                    float* scores) {
    /* detail::qk_head (kernels.hpp:245-267) */
    const size_t group = group_of(bits, word_bits);
    const size_t cpr = kvqo_codes_per_row(dim, bits, word_bits);
    const size_t wpr = cpr / group;
    const size_t row_bytes = wpr * (size_t)(word_bits / 8);
    float* qs = (float*)malloc(sizeof(float) * (cpr ? cpr : 1));
    float qdota = scale_query(q, dim, alpha, beta, bits, cpr, qs);
    if (word_bits == 8 && tokens >= 512) {
        /* build_query_table + dot_table_row (kernels.hpp:196-243). The scaled
         * query chunk for word w starts at w * group (the reference writes w * 8,
         * which only coincides for bits == 1; see kvq_oracle.h). */
        float* qtab = (float*)malloc(sizeof(float) * wpr * 256);
        for (size_t w = 0; w < wpr; ++w) {
            const float* qw = qs + w * group;
            for (unsigned v = 0; v < 256; ++v) {
                float acc = 0.0f;
                for (size_t k = 0; k < group; ++k) acc += qw[k] * lut(bits, v, (int)k);
                qtab[w * 256 + v] = acc;
            }
        }
        for (size_t j = 0; j < tokens; ++j) {
            const uint8_t* row = bytes + j * wpr;
            float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
            size_t w = 0;
            for (; w + 4 <= wpr; w += 4) {
                a0 += qtab[(w + 0) * 256 + row[w + 0]];
                a1 += qtab[(w + 1) * 256 + row[w + 1]];
                a2 += qtab[(w + 2) * 256 + row[w + 2]];
                a3 += qtab[(w + 3) * 256 + row[w + 3]];
            }
            for (; w < wpr; ++w) a0 += qtab[w * 256 + row[w]];
            scores[j] = ((a0 + a1) + (a2 + a3)) + qdota;
        }
        free(qtab);
    } else if (word_bits == 8) {
        /* dot_row_byte<N> (kernels.hpp:65-82): lane-striped partials, summed last. */
        for (size_t j = 0; j < tokens; ++j) {
            const uint8_t* row = bytes + j * wpr;
            float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
            for (size_t w = 0; w < wpr; ++w) {
                const float* qw = qs + w * group;
                for (size_t k = 0; k < group; ++k) acc[k] += qw[k] * lut(bits, row[w], (int)k);
            }
            float total = 0.0f;
            for (size_t k = 0; k < group; ++k) total += acc[k];
            scores[j] = total + qdota;
        }
    } else {
        /* dot_row_wide (kernels.hpp:98-112) */
        const uint32_t mask = (1u << bits) - 1u;
        for (size_t j = 0; j < tokens; ++j) {
            float acc = 0.0f;
            for (size_t w = 0; w < wpr; ++w) {
                uint32_t word = word_at(bytes + j * row_bytes, w, word_bits);
                for (size_t k = 0; k < group; ++k) {
                    int shift = word_bits - bits * (int)(k + 1);
                    acc += qs[w * group + k] * (float)((word >> shift) & mask);
                }
            }
            scores[j] = acc + qdota;
        }
    }
    free(qs);
}

void kvqo_wv_output(const float* w, const uint8_t* bytes, size_t tokens, size_t dim,
                    const float* alpha, const float* beta, int bits, int word_bits,
                    float* out) {
    /* wv_output (kernels.hpp:316-336) -> wv_block (269-284). The head_block split
     * only partitions lanes; each lane sums tokens ascending, so one block covering
     * every word gives the identical result. */
    const size_t group = group_of(bits, word_bits);
    const size_t cpr = kvqo_codes_per_row(dim, bits, word_bits);
    const size_t wpr = cpr / group;
    const size_t row_bytes = wpr * (size_t)(word_bits / 8);
    const uint32_t mask = (1u << bits) - 1u;
    float wsum = 0.0f;
    for (size_t j = 0; j < tokens; ++j) wsum += w[j];
    float* acc = (float*)calloc(cpr + 1, sizeof(float));
    for (size_t j = 0; j < tokens; ++j) {
        for (size_t ww = 0; ww < wpr; ++ww) {
            if (word_bits == 8) { /* axpy_row_byte (84-95) */
                unsigned v = bytes[j * row_bytes + ww];
                for (size_t k = 0; k < group; ++k) acc[ww * group + k] += w[j] * lut(bits, v, (int)k);
            } else { /* axpy_row_wide (114-127) */
                uint32_t word = word_at(bytes + j * row_bytes, ww, word_bits);
                for (size_t k = 0; k < group; ++k) {
                    int shift = word_bits - bits * (int)(k + 1);
                    acc[ww * group + k] += w[j] * (float)((word >> shift) & mask);
                }
            }
        }
    }
    const float levels = (float)((1u << bits) - 1u);
    for (size_t c = 0; c < dim; ++c) { /* 277-283 */
        float range = beta[c] - alpha[c];
        float step = range > 0.0f ? range / levels : 0.0f;
        out[c] = step * acc[c] + alpha[c] * wsum;
    }
    free(acc);
}

void kvqo_naive_qk(const float* q, const float* k, size_t rows, size_t cols, float* out) {
    /* kernels.hpp:401-413 */
    for (size_t j = 0; j < rows; ++j) {
        float acc = 0.0f;
        for (size_t c = 0; c < cols; ++c) acc += q[c] * k[j * cols + c];
        out[j] = acc;
    }
}

void kvqo_naive_wv(const float* w, const float* v, size_t rows, size_t cols, float* out) {
    /* kernels.hpp:415-426 */
    for (size_t c = 0; c < cols; ++c) out[c] = 0.0f;
    for (size_t j = 0; j < rows; ++j)
        for (size_t c = 0; c < cols; ++c) out[c] += w[j] * v[j * cols + c];
}

/* ---- calibrate.hpp --------------------------------------------------------- */

float kvqo_g_apply(float x, float gamma, float delta, float tau1, float tau2) {
    /* calibrate.hpp:62-67 */
    float width = delta - gamma;
    if (width <= 0.0f) return x - tau1;
    float t = (x - gamma) / width;
    return x - (tau1 * (1.0f - t) + tau2 * t);
}

void kvqo_softmax_inplace(float* row, size_t n) {
    /* calibrate.hpp:77-87 */
    if (n == 0) return;
    float m = row[0];
    for (size_t i = 0; i < n; ++i) m = ref_max(m, row[i]);
    float sum = 0.0f;
    for (size_t i = 0; i < n; ++i) {
        row[i] = expf(row[i] - m);
        sum += row[i];
    }
    for (size_t i = 0; i < n; ++i) row[i] /= sum;
}

void kvqo_calibrated_softmax_concat(const float* vis, size_t n_vis, const float* tail,
                                    size_t n_tail, float tau1, float tau2, float* out,
                                    size_t* slope_violations) {
    /* calibrate.hpp:100-114 (row_range 39-47, g_monotone 52-54) */
    if (n_vis > 0) {
        float gamma = vis[0], delta = vis[0];
        for (size_t i = 0; i < n_vis; ++i) {
            gamma = ref_min(gamma, vis[i]);
            delta = ref_max(delta, vis[i]);
        }
        if (slope_violations && !((delta - gamma) + (tau1 - tau2) > 0.0f)) ++*slope_violations;
        for (size_t i = 0; i < n_vis; ++i) out[i] = kvqo_g_apply(vis[i], gamma, delta, tau1, tau2);
    }
    for (size_t i = 0; i < n_tail; ++i) out[n_vis + i] = tail[i];
    kvqo_softmax_inplace(out, n_vis + n_tail);
}

/* Offline tau search (calibrate.hpp:160-234): grid_mse_table / grid_search over `samples`
 * calibration samples (query [S][d], exact keys [S][n][d], packed keys [S][n][row bytes]
 * with stats [S][d]); mse[c] = mean over samples of the mean squared difference between
 * calibrated_softmax_concat(quant / sqrt(d), {}, cell) and softmax(exact / sqrt(d)), in
 * double (sample_mse, 180-188). best = argmin, ties to the smaller tau1, then tau2. */
void kvqo_grid_mse_table(const float* queries, const float* keys_exact, const uint8_t* codes,
                         const float* alpha, const float* beta, size_t samples, size_t n,
                         size_t d, int bits, int word_bits, const float* tau1, const float* tau2,
                         size_t cells, double* mse, float* best) {
    const size_t g = (size_t)(word_bits / bits);
    const size_t rb = (d + g - 1) / g * g / g * (size_t)(word_bits / 8);
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    float* quant = (float*)malloc(sizeof(float) * (samples * n + 1));
    float* exact = (float*)malloc(sizeof(float) * (samples * n + 1));
    float* prob = (float*)malloc(sizeof(float) * (n + 1));
    for (size_t s = 0; s < samples; ++s) { /* prepare_samples, 160-178 */
        kvqo_qk_scores(queries + s * d, codes + s * n * rb, n, d, alpha + s * d, beta + s * d, bits,
                       word_bits, quant + s * n);
        for (size_t j = 0; j < n; ++j) quant[s * n + j] *= inv_sqrt_d;
        kvqo_naive_qk(queries + s * d, keys_exact + s * n * d, n, d, exact + s * n);
        for (size_t j = 0; j < n; ++j) exact[s * n + j] *= inv_sqrt_d;
        kvqo_softmax_inplace(exact + s * n, n);
    }
    size_t bi = 0;
    for (size_t c = 0; c < cells; ++c) {
        double acc = 0.0;
        for (size_t s = 0; s < samples; ++s) {
            kvqo_calibrated_softmax_concat(quant + s * n, n, NULL, 0, tau1[c], tau2[c], prob, NULL);
            double a2 = 0.0;
            for (size_t j = 0; j < n; ++j) {
                double diff = (double)prob[j] - (double)exact[s * n + j];
                a2 += diff * diff;
            }
            acc += a2 / (double)n;
        }
        mse[c] = acc / (double)samples;
        if (c > 0 && (mse[c] < mse[bi] ||
                      (mse[c] == mse[bi] && (tau1[c] < tau1[bi] || (tau1[c] == tau1[bi] && tau2[c] < tau2[bi])))))
            bi = c;
    }
    if (best && cells) {
        best[0] = tau1[bi];
        best[1] = tau2[bi];
    }
    free(quant);
    free(exact);
    free(prob);
}

/* mse_report (calibrate.hpp:300-351) over `heads` heads of equal shape. Per head: stats +
 * quantize of the keys (mode, bits, word_bits), exact = naive_qk * inv_sqrt_d, quant =
 * qk_scores * inv_sqrt_d, qc = g_transform(quant, row_range(quant), tau); edges [bins+1] =
 * lo + (hi - lo) * i / bins over the union of the three rows (322-331); counts [3][bins]
 * by bin_row (272-287); mse_q / mse_qc = prob_mse of the softmaxes vs the exact softmax
 * (289-296). Returns 0, or -1 on an empty matrix (compute_stats). */
int kvqo_mse_report(const float* queries, const float* keys, size_t heads, size_t n, size_t d, int mode,
                    int bits, int word_bits, float tau1, float tau2, size_t bins, double* mse_q,
                    double* mse_qc, float* edges, uint64_t* counts) {
    if (n == 0 || d == 0) return -1;
    const size_t rb = kvqo_row_bytes(d, bits, word_bits);
    const float inv_sqrt_d = 1.0f / sqrtf((float)d);
    float* alpha = (float*)malloc(sizeof(float) * d);
    float* beta = (float*)malloc(sizeof(float) * d);
    uint8_t* codes = (uint8_t*)malloc(n * rb + 1);
    float* rows[3];
    float* prob[3];
    for (int v = 0; v < 3; ++v) {
        rows[v] = (float*)malloc(sizeof(float) * n);
        prob[v] = (float*)malloc(sizeof(float) * n);
    }
    for (size_t h = 0; h < heads; ++h) {
        const float* k = keys + h * n * d;
        const float* q = queries + h * d;
        kvqo_compute_stats(k, n, d, mode, alpha, beta);
        kvqo_quantize(k, n, d, alpha, beta, bits, word_bits, codes);
        kvqo_naive_qk(q, k, n, d, rows[0]);
        for (size_t j = 0; j < n; ++j) rows[0][j] *= inv_sqrt_d;
        kvqo_qk_scores(q, codes, n, d, alpha, beta, bits, word_bits, rows[1]);
        for (size_t j = 0; j < n; ++j) rows[1][j] *= inv_sqrt_d;
        float gamma = rows[1][0], delta = rows[1][0];
        for (size_t j = 0; j < n; ++j) {
            if (rows[1][j] < gamma) gamma = rows[1][j];
            if (delta < rows[1][j]) delta = rows[1][j];
        }
        for (size_t j = 0; j < n; ++j) rows[2][j] = kvqo_g_apply(rows[1][j], gamma, delta, tau1, tau2);
        float lo = rows[0][0], hi = rows[0][0];
        for (int v = 0; v < 3; ++v)
            for (size_t j = 0; j < n; ++j) {
                if (rows[v][j] < lo) lo = rows[v][j];
                if (hi < rows[v][j]) hi = rows[v][j];
            }
        float* e = edges + h * (bins + 1);
        for (size_t i = 0; i <= bins; ++i) e[i] = lo + (hi - lo) * (float)i / (float)bins;
        const float blo = e[0], bw = e[bins] - e[0];
        for (int v = 0; v < 3; ++v) {
            uint64_t* c = counts + (h * 3 + (size_t)v) * bins;
            for (size_t b = 0; b < bins; ++b) c[b] = 0;
            for (size_t j = 0; j < n; ++j) {
                size_t idx = 0;
                if (bw > 0.0f) {
                    float t = (rows[v][j] - blo) / bw * (float)bins;
                    size_t i = (size_t)(0.0f < t ? t : 0.0f);
                    idx = i < bins - 1 ? i : bins - 1;
                }
                ++c[idx];
            }
            memcpy(prob[v], rows[v], sizeof(float) * n);
            kvqo_softmax_inplace(prob[v], n);
        }
        double aq = 0.0, ac = 0.0;
        for (size_t j = 0; j < n; ++j) {
            double dq = (double)prob[1][j] - (double)prob[0][j];
            double dc = (double)prob[2][j] - (double)prob[0][j];
            aq += dq * dq;
            ac += dc * dc;
        }
        mse_q[h] = aq / (double)n;
        mse_qc[h] = ac / (double)n;
    }
    for (int v = 0; v < 3; ++v) {
        free(rows[v]);
        free(prob[v]);
    }
    free(alpha);
    free(beta);
    free(codes);
    return 0;
}

/* ---- kvcache.hpp ----------------------------------------------------------- */

void kvqo_decode_head(const float* q, size_t dim, size_t n_vis, int bits, int word_bits,
                      const uint8_t* k_bytes, const float* k_alpha, const float* k_beta,
                      const uint8_t* v_bytes, const float* v_alpha, const float* v_beta,
                      const float* k_tail, const float* v_tail, size_t n_tail, float tau1,
                      float tau2, float* out, float* weights, size_t* slope_violations) {
    /* HybridKVCache::run_decode body for one head (kvcache.hpp:279-304). */
    const float inv_sqrt_d = 1.0f / sqrtf((float)dim); /* 273 */
    float* vis = (float*)malloc(sizeof(float) * (n_vis + 1));
    float* tail = (float*)malloc(sizeof(float) * (n_tail + 1));
    float* row = (float*)malloc(sizeof(float) * (n_vis + n_tail + 1));
    float* tmp = (float*)malloc(sizeof(float) * (dim + 1));
    if (n_vis > 0) {
        kvqo_qk_scores(q, k_bytes, n_vis, dim, k_alpha, k_beta, bits, word_bits, vis);
        for (size_t j = 0; j < n_vis; ++j) vis[j] *= inv_sqrt_d; /* 284 */
    }
    kvqo_naive_qk(q, k_tail, n_tail, dim, tail); /* 286-287 */
    for (size_t j = 0; j < n_tail; ++j) tail[j] *= inv_sqrt_d;
    kvqo_calibrated_softmax_concat(vis, n_vis, tail, n_tail, tau1, tau2, row, slope_violations);
    if (weights) memcpy(weights, row, sizeof(float) * (n_vis + n_tail)); /* 290-294 */
    for (size_t c = 0; c < dim; ++c) out[c] = 0.0f;
    if (n_vis > 0) kvqo_wv_output(row, v_bytes, n_vis, dim, v_alpha, v_beta, bits, word_bits, out);
    kvqo_naive_wv(row + n_vis, v_tail, n_tail, dim, tmp); /* 302-304 */
    for (size_t c = 0; c < dim; ++c) out[c] += tmp[c];
    free(vis);
    free(tail);
    free(row);
    free(tmp);
}

/* ---- workload.hpp (gaussian) ---------------------------------------------- */

typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & 0xFFFFFFFF80000000ULL) | (g->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t xa = x >> 1;
            if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ULL;
    y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
    y ^= (y << 37) & 0xFFF7EEE000000000ULL;
    y ^= y >> 43;
    return y;
}

typedef struct {
    mt64 eng;
    double spare;
    int have_spare;
} normal_sampler;

static double ns_uniform01(normal_sampler* s) { /* workload.hpp:107 */
    return (double)(mt64_next(&s->eng) >> 11) * 0x1.0p-53;
}

static double ns_next(normal_sampler* s) { /* workload.hpp:89-104 */
    if (s->have_spare) {
        s->have_spare = 0;
        return s->spare;
    }
    double u, v, q;
    do {
        u = 2.0 * ns_uniform01(s) - 1.0;
        v = 2.0 * ns_uniform01(s) - 1.0;
        q = u * u + v * v;
    } while (q >= 1.0 || q == 0.0);
    double factor = sqrt(-2.0 * log(q) / q);
    s->spare = v * factor;
    s->have_spare = 1;
    return u * factor;
}

static uint64_t mix_seed(uint64_t seed, uint64_t salt) { /* workload.hpp:115-121 */
    uint64_t z = seed ^ (salt * 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d49b6d1b3e9349ULL;
    return z ^ (z >> 31);
}

static void fill(normal_sampler* s, float* m, size_t count, double mean, double stddev) {
    for (size_t i = 0; i < count; ++i) m[i] = (float)(mean + stddev * ns_next(s));
}

void kvqo_generate_head(uint64_t seed, uint64_t head, size_t tokens, size_t dim, double mean,
                        double stddev, float* keys, float* values, float* query) {
    /* kvq::generate (workload.hpp:164-179), one head */
    normal_sampler* s = (normal_sampler*)calloc(1, sizeof(normal_sampler));
    mt64_seed(&s->eng, mix_seed(seed, head));
    fill(s, keys, tokens * dim, mean, stddev);
    fill(s, values, tokens * dim, mean, stddev);
    fill(s, query, dim, mean, stddev);
    free(s);
}

void kvqo_generate_step_head(uint64_t seed, uint64_t head, uint64_t step, size_t dim,
                             double mean, double stddev, float* query, float* key,
                             float* value) {
    /* kvq::generate_step (workload.hpp:183-201), one head */
    normal_sampler* s = (normal_sampler*)calloc(1, sizeof(normal_sampler));
    mt64_seed(&s->eng, mix_seed(seed, 0x5347ULL + head * 0x10001ULL + step * 0x2b9ULL));
    fill(s, query, dim, mean, stddev);
    fill(s, key, dim, mean, stddev);
    fill(s, value, dim, mean, stddev);
    free(s);
}

/* ---- reference.hpp --------------------------------------------------------- */

void kvqo_oracle_attention(const float* q, const float* k, const float* v, size_t n,
                           size_t dim, float* out) {
    /* reference.hpp:26-54 */
    const double inv_sqrt_d = 1.0 / sqrt((double)dim);
    double* scores = (double*)calloc(n + 1, sizeof(double));
    for (size_t c = 0; c < dim; ++c) {
        double qc = q[c];
        for (size_t j = 0; j < n; ++j) scores[j] += qc * (double)k[j * dim + c];
    }
    double m = n ? scores[0] : 0.0;
    for (size_t j = 0; j < n; ++j) m = m < scores[j] ? scores[j] : m;
    double sum = 0.0;
    for (size_t j = 0; j < n; ++j) {
        scores[j] = exp(scores[j] * inv_sqrt_d - m * inv_sqrt_d);
        sum += scores[j];
    }
    for (size_t c = 0; c < dim; ++c) {
        double acc = 0.0;
        for (size_t j = 0; j < n; ++j) acc += (scores[j] / sum) * (double)v[j * dim + c];
        out[c] = (float)acc;
    }
    free(scores);
}
