// ref_shim.cpp — TEST INFRASTRUCTURE ONLY. A C-ABI shim over the UNMODIFIED kvq
// reference headers (/root/reference/proj/include, included read-only via -I, never
// copied). Built by oracle/Makefile into oracle/_ref/libkvq_ref.so with the
// reference's own flags (-std=c++20 -O3 -DNDEBUG, proj/CMakeLists.txt:3-14).
//
// Used for two things only:
//   * pinning the C restatement (kvq_oracle.c) against the real reference, and
//     generating golden fixtures (tests/golden/make_golden.py);
//   * the CPU baseline arm of bench.py (`--impl reference`, cpu_baseline): the
//     reference's own HybridKVCache::decode_step timed on the host cores.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <span>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "kvq/kvq.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const kvq::config_error*>(&e)) return 1;
    if (dynamic_cast<const kvq::domain_error*>(&e)) return 2;
    if (dynamic_cast<const kvq::format_error*>(&e)) return 3;
    return 9;
}

kvq::DenseMatrix mat(const float* p, std::size_t r, std::size_t c) {
    return kvq::DenseMatrix(r, c, std::vector<float>(p, p + r * c));
}

kvq::QuantizedSegment seg_from(const std::uint8_t* bytes, std::size_t tokens, std::size_t dim,
                               const float* alpha, const float* beta, int bits, int word_bits) {
    kvq::QuantizedSegment s;
    s.codes.code_bits = bits;
    s.codes.word_bits = word_bits;
    s.tokens = tokens;
    s.dim = dim;
    s.bitwidth = bits;
    std::size_t g = static_cast<std::size_t>(word_bits / bits);
    std::size_t cpr = (dim + g - 1) / g * g;
    s.codes.logical_count = tokens * cpr;
    std::size_t nbytes = s.codes.word_count() * static_cast<std::size_t>(word_bits / 8);
    s.codes.bytes.assign(bytes, bytes + nbytes);
    s.stats.alpha.assign(alpha, alpha + dim);
    s.stats.beta.assign(beta, beta + dim);
    return s;
}

}  // namespace

extern "C" {

const char* kvqr_last_error() { return g_err.c_str(); }

int kvqr_pack(const std::uint32_t* codes, std::size_t count, int bits, int word_bits,
              std::uint8_t* out, std::size_t* out_len) {
    try {
        kvq::PackedBuffer b = kvq::pack(std::span<const std::uint32_t>(codes, count), bits, word_bits);
        std::memcpy(out, b.bytes.data(), b.bytes.size());
        *out_len = b.bytes.size();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_unpack(const std::uint8_t* bytes, std::size_t count, int bits, int word_bits,
                std::uint32_t* out) {
    try {
        kvq::PackedBuffer b;
        b.code_bits = bits;
        b.word_bits = word_bits;
        b.logical_count = count;
        std::size_t g = word_bits / bits;
        b.bytes.assign(bytes, bytes + (count + g - 1) / g * (word_bits / 8));
        std::vector<std::uint32_t> c = kvq::unpack(b);
        std::copy(c.begin(), c.end(), out);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_compute_stats(const float* m, std::size_t rows, std::size_t cols, int mode,
                       float* alpha, float* beta) {
    try {
        kvq::ChannelStats s = kvq::compute_stats(
            mat(m, rows, cols), mode == 0 ? kvq::QuantMode::channel_wise : kvq::QuantMode::global);
        std::copy(s.alpha.begin(), s.alpha.end(), alpha);
        std::copy(s.beta.begin(), s.beta.end(), beta);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_quantize(const float* m, std::size_t rows, std::size_t cols, const float* alpha,
                  const float* beta, int bits, int word_bits, std::uint8_t* out,
                  std::size_t* out_len) {
    try {
        kvq::ChannelStats s{std::vector<float>(alpha, alpha + cols),
                            std::vector<float>(beta, beta + cols)};
        kvq::QuantizedSegment q = kvq::quantize(mat(m, rows, cols), s, bits, word_bits);
        std::memcpy(out, q.codes.bytes.data(), q.codes.bytes.size());
        *out_len = q.codes.bytes.size();
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_dequantize(const std::uint8_t* bytes, std::size_t rows, std::size_t cols,
                    const float* alpha, const float* beta, int bits, int word_bits, float* out) {
    try {
        kvq::DenseMatrix d = kvq::dequantize(seg_from(bytes, rows, cols, alpha, beta, bits, word_bits));
        std::copy(d.data.begin(), d.data.end(), out);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_qk_scores(const float* q, const std::uint8_t* bytes, std::size_t tokens,
                   std::size_t dim, const float* alpha, const float* beta, int bits,
                   int word_bits, float* scores) {
    try {
        std::vector<float> s = kvq::qk_scores(std::span<const float>(q, dim),
                                              seg_from(bytes, tokens, dim, alpha, beta, bits, word_bits),
                                              kvq::KernelConfig{});
        std::copy(s.begin(), s.end(), scores);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_wv_output(const float* w, const std::uint8_t* bytes, std::size_t tokens,
                   std::size_t dim, const float* alpha, const float* beta, int bits,
                   int word_bits, float* out) {
    try {
        std::vector<float> o = kvq::wv_output(std::span<const float>(w, tokens),
                                              seg_from(bytes, tokens, dim, alpha, beta, bits, word_bits),
                                              kvq::KernelConfig{});
        std::copy(o.begin(), o.end(), out);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// grid_mse_table / grid_search (calibrate.hpp:195-234) over `samples` calibration samples:
// queries [S][d], keys_exact [S][n][d], packed keys [S][n][row_bytes] + alpha/beta [S][d].
int kvqr_grid_mse_table(const float* queries, const float* keys_exact, const std::uint8_t* codes,
                        const float* alpha, const float* beta, std::size_t samples, std::size_t n,
                        std::size_t d, int bits, int word_bits, const float* tau1, const float* tau2,
                        std::size_t cells, double* mse, float* best) {
    try {
        std::vector<kvq::CalibrationSample> set(samples);
        std::size_t g = static_cast<std::size_t>(word_bits / bits);
        std::size_t rb = (d + g - 1) / g * g / g * static_cast<std::size_t>(word_bits / 8);
        for (std::size_t s = 0; s < samples; ++s) {
            set[s].query.assign(queries + s * d, queries + (s + 1) * d);
            set[s].keys_exact = mat(keys_exact + s * n * d, n, d);
            set[s].keys_quant = seg_from(codes + s * n * rb, n, d, alpha + s * d, beta + s * d, bits, word_bits);
        }
        std::vector<kvq::CalibrationParams> grid(cells);
        for (std::size_t c = 0; c < cells; ++c) grid[c] = {tau1[c], tau2[c]};
        std::vector<kvq::GridCell> table = kvq::grid_mse_table(set, grid);
        for (std::size_t c = 0; c < cells; ++c) mse[c] = table[c].mse;
        kvq::CalibrationParams b = kvq::grid_search(set, grid);
        best[0] = b.tau1;
        best[1] = b.tau2;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_mse_report(const float* queries, const float* keys, std::size_t heads, std::size_t n, std::size_t d,
                    int mode, int bits, int word_bits, float tau1, float tau2, std::size_t bins, double* mse_q,
                    double* mse_qc, float* edges, std::uint64_t* counts, double* means) {
    try {
        std::vector<kvq::HeadWorkload> hw(heads);
        for (std::size_t h = 0; h < heads; ++h) {
            hw[h].keys = mat(keys + h * n * d, n, d);
            hw[h].values = kvq::DenseMatrix(n, d);
            hw[h].query = mat(queries + h * d, 1, d);
        }
        kvq::QuantizationConfig qcfg{bits, mode ? kvq::QuantMode::global : kvq::QuantMode::channel_wise, word_bits};
        kvq::MseReport r = kvq::mse_report(hw, qcfg, kvq::CalibrationParams{tau1, tau2}, bins);
        for (std::size_t h = 0; h < heads; ++h) {
            mse_q[h] = r.rows[h].mse_quant;
            mse_qc[h] = r.rows[h].mse_quant_c;
            const kvq::HeadHistogram& hh = r.histograms[h];
            std::copy(hh.edges.begin(), hh.edges.end(), edges + h * (bins + 1));
            for (int v = 0; v < 3; ++v)
                std::copy(hh.counts[v].begin(), hh.counts[v].end(), counts + (h * 3 + v) * bins);
        }
        means[0] = r.mean_mse_quant;
        means[1] = r.mean_mse_quant_c;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_calibrated_softmax_concat(const float* vis, std::size_t n_vis, const float* tail,
                                   std::size_t n_tail, float tau1, float tau2, float* out,
                                   std::size_t* violations) {
    try {
        std::vector<float> r = kvq::calibrated_softmax_concat(
            std::span<const float>(vis, n_vis), std::span<const float>(tail, n_tail),
            kvq::CalibrationParams{tau1, tau2}, violations);
        std::copy(r.begin(), r.end(), out);
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

float kvqr_g_apply(float x, float gamma, float delta, float tau1, float tau2) {
    return kvq::g_apply(x, kvq::ScoreRange{gamma, delta}, kvq::CalibrationParams{tau1, tau2});
}

int kvqr_generate(std::uint64_t seed, std::size_t heads, std::size_t tokens, std::size_t dim,
                  float* keys, float* values, float* queries) {
    try {
        kvq::WorkloadSpec spec;
        spec.heads = heads;
        spec.tokens = tokens;
        spec.head_dim = dim;
        spec.seed = seed;
        std::vector<kvq::HeadWorkload> hw = kvq::generate(spec);
        for (std::size_t h = 0; h < heads; ++h) {
            std::copy(hw[h].keys.data.begin(), hw[h].keys.data.end(), keys + h * tokens * dim);
            std::copy(hw[h].values.data.begin(), hw[h].values.data.end(), values + h * tokens * dim);
            std::copy(hw[h].query.data.begin(), hw[h].query.data.end(), queries + h * dim);
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_generate_step(std::uint64_t seed, std::size_t heads, std::size_t dim, std::uint64_t step,
                       float* q, float* k, float* v) {
    try {
        kvq::WorkloadSpec spec;
        spec.heads = heads;
        spec.tokens = 1;
        spec.head_dim = dim;
        spec.seed = seed;
        kvq::StepTokens st = kvq::generate_step(spec, step);
        for (std::size_t h = 0; h < heads; ++h) {
            std::copy(st.query[h].data.begin(), st.query[h].data.end(), q + h * dim);
            std::copy(st.key[h].data.begin(), st.key[h].data.end(), k + h * dim);
            std::copy(st.value[h].data.begin(), st.value[h].data.end(), v + h * dim);
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

void kvqr_oracle_attention(const float* q, const float* k, const float* v, std::size_t n,
                           std::size_t dim, float* out) {
    std::vector<float> o = kvq::oracle_attention(std::span<const float>(q, dim), mat(k, n, dim),
                                                 mat(v, n, dim));
    std::copy(o.begin(), o.end(), out);
}

// ---- HybridKVCache handle -----------------------------------------------------

struct kvqr_cache {
    kvq::HybridKVCache cache;
};

// k_vis/v_vis: [heads][n][dim] fp32. bits == 16 selects build_full_precision.
int kvqr_cache_build(const float* k_vis, const float* v_vis, std::size_t heads, std::size_t n,
                     std::size_t dim, int bits, int mode, int word_bits, float tau1, float tau2,
                     kvqr_cache** out) {
    try {
        std::vector<kvq::DenseMatrix> ks, vs;
        for (std::size_t h = 0; h < heads; ++h) {
            ks.push_back(mat(k_vis + h * n * dim, n, dim));
            vs.push_back(mat(v_vis + h * n * dim, n, dim));
        }
        auto* c = new kvqr_cache;
        if (bits == kvq::kFullPrecisionBits) {
            c->cache = kvq::HybridKVCache::build_full_precision(ks, vs);
        } else {
            c->cache = kvq::HybridKVCache::build(
                ks, vs,
                kvq::QuantizationConfig{bits, mode == 0 ? kvq::QuantMode::channel_wise : kvq::QuantMode::global,
                                        word_bits},
                kvq::CalibrationParams{tau1, tau2});
        }
        *out = c;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

void kvqr_cache_free(kvqr_cache* c) { delete c; }

int kvqr_cache_append(kvqr_cache* c, const float* k_new, const float* v_new) {
    try {
        std::size_t h = c->cache.heads(), d = c->cache.dim();
        c->cache.append(mat(k_new, h, d), mat(v_new, h, d));
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// queries [heads][dim] -> out [heads][dim]; weights (nullable) [heads][n_vis+n_tail]
int kvqr_cache_decode(const kvqr_cache* c, const float* queries, float* out, float* weights,
                      std::size_t* violations) {
    try {
        std::size_t h = c->cache.heads(), d = c->cache.dim();
        kvq::DecodeDetail det = c->cache.decode_step_detailed(mat(queries, h, d));
        std::copy(det.outputs.data.begin(), det.outputs.data.end(), out);
        if (weights) std::copy(det.weights.data.begin(), det.weights.data.end(), weights);
        if (violations) *violations = det.slope_violations;
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// Segment readback in the reference layout: bytes of head h's K (which=0) or V (1).
int kvqr_cache_segment(const kvqr_cache* c, std::size_t h, int which, std::uint8_t* bytes,
                       float* alpha, float* beta) {
    const kvq::QuantizedSegment& s = which == 0 ? c->cache.key_segment(h) : c->cache.value_segment(h);
    std::memcpy(bytes, s.codes.bytes.data(), s.codes.bytes.size());
    std::copy(s.stats.alpha.begin(), s.stats.alpha.end(), alpha);
    std::copy(s.stats.beta.begin(), s.stats.beta.end(), beta);
    return 0;
}

// HybridKVCache::save into a caller buffer (*len = bytes needed; copies only if it fits).
int kvqr_cache_save(const kvqr_cache* c, std::uint8_t* buf, std::size_t cap, std::size_t* len) {
    try {
        std::stringstream ss;
        c->cache.save(ss);
        const std::string b = ss.str();
        *len = b.size();
        if (b.size() <= cap) std::memcpy(buf, b.data(), b.size());
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

// HybridKVCache::load from a byte image; *err_off = format_error::offset() on failure.
int kvqr_cache_load(const std::uint8_t* buf, std::size_t len, kvqr_cache** out, std::uint64_t* err_off) {
    try {
        std::stringstream ss(std::string(reinterpret_cast<const char*>(buf), len));
        std::uint64_t off = 0;
        auto* c = new kvqr_cache;
        try {
            c->cache = kvq::HybridKVCache::load(ss, off);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
        return 0;
    } catch (const kvq::format_error& e) {
        *err_off = e.offset();
        return fail(e);
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_cache_memory(const kvqr_cache* c, std::size_t* out6) {
    kvq::CacheMemory m = c->cache.memory();
    out6[0] = m.code_bytes;
    out6[1] = m.stats_bytes;
    out6[2] = m.quantized_bytes;
    out6[3] = m.tail_bytes;
    out6[4] = m.fp32_vis_bytes;
    out6[5] = m.total_bytes;
    return 0;
}

// ---- CPU baseline harness (bench.py --impl reference / cpu_baseline) -----------
//
// `requests` independent single-sequence caches of `kv_heads` heads each, built from
// the given fp32 prefill ([requests][kv_heads][n][dim], untimed). One timed step =
// for every request, G = group calls of HybridKVCache::decode_step (GQA emulated as
// in SURVEY.md §8c rule 5: call g uses query row h_kv <- q head h_kv*G + g), then
// one append of the step's new K/V rows. Requests are spread over `threads` host
// threads (outer pool, KernelConfig{32, 64, 1} inside — the reference's fastest mode,
// BASELINE.md §4). Returns per-step wall seconds in step_seconds[steps].
// Shared by the two bench arms: per-request caches built with the reference's own API.
static std::vector<kvq::HybridKVCache> bench_build(const float* k_vis, const float* v_vis, std::size_t requests,
                                                   std::size_t kv_heads, std::size_t n, std::size_t dim, int bits,
                                                   int word_bits, float tau1, float tau2, const float* k_new,
                                                   const float* v_new, int threads, std::size_t prefill_tail) {
    std::vector<kvq::HybridKVCache> caches(requests);
    std::vector<std::thread> pool;
    std::atomic<std::size_t> next{0};
    for (int t = 0; t < threads; ++t) {
        pool.emplace_back([&] {
            for (std::size_t r = next++; r < requests; r = next++) {
                std::vector<kvq::DenseMatrix> ks, vs;
                for (std::size_t h = 0; h < kv_heads; ++h) {
                    std::size_t off = (r * kv_heads + h) * n * dim;
                    ks.push_back(mat(k_vis + off, n, dim));
                    vs.push_back(mat(v_vis + off, n, dim));
                }
                caches[r] = kvq::HybridKVCache::build(
                    ks, vs, kvq::QuantizationConfig{bits, kvq::QuantMode::channel_wise, word_bits},
                    kvq::CalibrationParams{tau1, tau2});
                // generated tokens already in the fp32 tail before the timed steps
                for (std::size_t t = 0; t < prefill_tail; ++t)
                    caches[r].append(mat(k_new + r * kv_heads * dim, kv_heads, dim),
                                     mat(v_new + r * kv_heads * dim, kv_heads, dim));
            }
        });
    }
    for (auto& th : pool) th.join();
    return caches;
}

// One head of the "without post-scaling" ablation (BASELINE config 3): dequantize the
// packed segments (quantize.hpp:129-146), then the dense products naive_qk / naive_wv
// (kernels.hpp:401-426) around the same calibrated softmax (calibrate.hpp:100-114).
static void decode_head_dequant(const kvq::HybridKVCache& c, std::size_t h, std::span<const float> q, float* out) {
    const std::size_t d = q.size();
    const float isd = 1.0f / std::sqrt(float(d));
    const kvq::DenseMatrix kd = kvq::dequantize(c.key_segment(h));
    const kvq::DenseMatrix vd = kvq::dequantize(c.value_segment(h));
    std::vector<float> vis = kvq::naive_qk(q, kd);
    for (float& x : vis) x *= isd;
    std::vector<float> tail = kvq::naive_qk(q, c.key_tail(h));
    for (float& x : tail) x *= isd;
    const std::vector<float> p = kvq::calibrated_softmax_concat(vis, tail, c.calibration());
    const std::vector<float> ov = kvq::naive_wv(std::span<const float>(p.data(), vis.size()), vd);
    const std::vector<float> ot = kvq::naive_wv(std::span<const float>(p.data() + vis.size(), tail.size()), c.value_tail(h));
    for (std::size_t i = 0; i < d; ++i) out[i] = ov[i] + ot[i];
}

// mode 0: HybridKVCache::decode_step (post-scaled, the reference as shipped);
// mode 1: dequantize-then-dot (decode_head_dequant) over the same caches.
static int bench_decode_mode(int mode, const float* k_vis, const float* v_vis, std::size_t requests,
                             std::size_t kv_heads, std::size_t group, std::size_t n, std::size_t dim, int bits,
                             int word_bits, float tau1, float tau2, const float* queries, const float* k_new,
                             const float* v_new, int threads, int steps, std::size_t prefill_tail,
                             double* step_seconds, float* out_last) {
    try {
        std::vector<kvq::HybridKVCache> caches = bench_build(k_vis, v_vis, requests, kv_heads, n, dim, bits, word_bits,
                                                             tau1, tau2, k_new, v_new, threads, prefill_tail);
        const kvq::KernelConfig inner{32, 64, 1};
        for (int s = 0; s < steps; ++s) {
            auto t0 = std::chrono::steady_clock::now();
            std::vector<std::thread> pool;
            std::atomic<std::size_t> next{0};
            for (int t = 0; t < threads; ++t) {
                pool.emplace_back([&] {
                    kvq::DenseMatrix q(kv_heads, dim);
                    std::vector<float> o1(dim);
                    for (std::size_t r = next++; r < requests; r = next++) {
                        for (std::size_t g = 0; g < group; ++g) {
                            for (std::size_t h = 0; h < kv_heads; ++h) {
                                const float* src = queries + ((r * kv_heads + h) * group + g) * dim;
                                std::copy(src, src + dim, q.row(h));
                            }
                            const bool keep = out_last && s == steps - 1;
                            if (mode == 0) {
                                kvq::DenseMatrix o = caches[r].decode_step(q, inner);
                                if (keep)
                                    for (std::size_t h = 0; h < kv_heads; ++h)
                                        std::copy(o.row(h), o.row(h) + dim,
                                                  out_last + ((r * kv_heads + h) * group + g) * dim);
                            } else {
                                for (std::size_t h = 0; h < kv_heads; ++h) {
                                    decode_head_dequant(caches[r], h, q.row_span(h), o1.data());
                                    if (keep)
                                        std::copy(o1.begin(), o1.end(), out_last + ((r * kv_heads + h) * group + g) * dim);
                                }
                            }
                        }
                        caches[r].append(mat(k_new + r * kv_heads * dim, kv_heads, dim),
                                         mat(v_new + r * kv_heads * dim, kv_heads, dim));
                    }
                });
            }
            for (auto& th : pool) th.join();
            step_seconds[s] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        }
        return 0;
    } catch (const std::exception& e) { return fail(e); }
}

int kvqr_bench_decode(const float* k_vis, const float* v_vis, std::size_t requests,
                      std::size_t kv_heads, std::size_t group, std::size_t n, std::size_t dim,
                      int bits, int word_bits, float tau1, float tau2, const float* queries,
                      const float* k_new, const float* v_new, int threads, int steps,
                      std::size_t prefill_tail, double* step_seconds, float* out_last) {
    return bench_decode_mode(0, k_vis, v_vis, requests, kv_heads, group, n, dim, bits, word_bits, tau1, tau2, queries,
                             k_new, v_new, threads, steps, prefill_tail, step_seconds, out_last);
}

int kvqr_bench_decode_dequant(const float* k_vis, const float* v_vis, std::size_t requests,
                              std::size_t kv_heads, std::size_t group, std::size_t n, std::size_t dim,
                              int bits, int word_bits, float tau1, float tau2, const float* queries,
                              const float* k_new, const float* v_new, int threads, int steps,
                              std::size_t prefill_tail, double* step_seconds, float* out_last) {
    return bench_decode_mode(1, k_vis, v_vis, requests, kv_heads, group, n, dim, bits, word_bits, tau1, tau2, queries,
                             k_new, v_new, threads, steps, prefill_tail, step_seconds, out_last);
}

}  // extern "C"
