// kvq/kernels.hpp — post-scaled q.K and w.V over packed segments (reference
// kernels.hpp:30-40, 302-426), executed by CUDA kernels through the C-ABI.
// KernelConfig is validated exactly like the reference but never changes results
// (the reference guarantees bit-identical output across configs, kernels.hpp:22-26).
#pragma once

#include <span>
#include <string>
#include <vector>

#include "kvq/quantize.hpp"

namespace kvq {

struct KernelConfig {
    std::size_t head_block = 32;
    std::size_t token_block = 64;
    int workers = 1;
    void validate() const {
        if (head_block < 1 || token_block < 1 || workers < 1)
            throw config_error("kernel blocks and workers must be >= 1");
    }
};

namespace detail {

inline void require_uniform(std::span<const QuantizedSegment> segs, const char* who) {
    for (const auto& s : segs)
        if (s.tokens != segs[0].tokens || s.dim != segs[0].dim || s.bitwidth != segs[0].bitwidth ||
            s.codes.word_bits != segs[0].codes.word_bits)
            throw domain_error(std::string(who) + ": head segments have mismatched shapes");
}

// Concatenate per-head segments into the C-ABI's [heads][...] buffers.
struct Stacked {
    std::vector<std::uint8_t> codes;
    std::vector<float> alpha, beta;
};
inline Stacked stack(std::span<const QuantizedSegment> segs) {
    Stacked st;
    for (const auto& s : segs) {
        st.codes.insert(st.codes.end(), s.codes.bytes.begin(), s.codes.bytes.end());
        st.alpha.insert(st.alpha.end(), s.stats.alpha.begin(), s.stats.alpha.end());
        st.beta.insert(st.beta.end(), s.stats.beta.begin(), s.stats.beta.end());
    }
    if (st.codes.empty()) st.codes.push_back(0);
    return st;
}

}  // namespace detail

inline std::vector<float> qk_scores(std::span<const float> q, const QuantizedSegment& keys, const KernelConfig& cfg) {
    cfg.validate();
    if (q.size() != keys.dim)
        throw domain_error("qk_scores: query length " + std::to_string(q.size()) + " does not match segment dim " +
                           std::to_string(keys.dim));
    std::vector<float> out(keys.tokens);
    auto st = detail::stack(std::span<const QuantizedSegment>(&keys, 1));
    capi::check(kvq_qk_scores(q.data(), st.codes.data(), st.alpha.data(), st.beta.data(), 1, keys.tokens, keys.dim,
                              keys.bitwidth, keys.codes.word_bits, out.data()));
    return out;
}

inline std::vector<float> wv_output(std::span<const float> w, const QuantizedSegment& values, const KernelConfig& cfg) {
    cfg.validate();
    if (w.size() != values.tokens)
        throw domain_error("wv_output: weight length " + std::to_string(w.size()) +
                           " does not match segment tokens " + std::to_string(values.tokens));
    std::vector<float> out(values.dim);
    auto st = detail::stack(std::span<const QuantizedSegment>(&values, 1));
    std::vector<float> wbuf(w.begin(), w.end());
    if (wbuf.empty()) wbuf.push_back(0.f);
    capi::check(kvq_wv_output(wbuf.data(), st.codes.data(), st.alpha.data(), st.beta.data(), 1, values.tokens,
                              values.dim, values.bitwidth, values.codes.word_bits, out.data()));
    return out;
}

inline DenseMatrix qk_scores(const DenseMatrix& queries, std::span<const QuantizedSegment> keys, const KernelConfig& cfg) {
    cfg.validate();
    if (queries.rows != keys.size()) throw domain_error("qk_scores: query rows != head count");
    if (keys.empty()) return DenseMatrix();
    detail::require_uniform(keys, "qk_scores");
    if (queries.cols != keys[0].dim) throw domain_error("qk_scores: query cols do not match segment dim");
    DenseMatrix out(keys.size(), keys[0].tokens);
    auto st = detail::stack(keys);
    capi::check(kvq_qk_scores(queries.data.data(), st.codes.data(), st.alpha.data(), st.beta.data(), keys.size(),
                              keys[0].tokens, keys[0].dim, keys[0].bitwidth, keys[0].codes.word_bits, out.data.data()));
    return out;
}

inline DenseMatrix wv_output(const DenseMatrix& weights, std::span<const QuantizedSegment> values, const KernelConfig& cfg) {
    cfg.validate();
    if (weights.rows != values.size()) throw domain_error("wv_output: weight rows != head count");
    if (values.empty()) return DenseMatrix();
    detail::require_uniform(values, "wv_output");
    if (weights.cols != values[0].tokens) throw domain_error("wv_output: weight cols do not match segment tokens");
    DenseMatrix out(values.size(), values[0].dim);
    auto st = detail::stack(values);
    std::vector<float> wbuf = weights.data;
    if (wbuf.empty()) wbuf.push_back(0.f);
    capi::check(kvq_wv_output(wbuf.data(), st.codes.data(), st.alpha.data(), st.beta.data(), values.size(),
                              values[0].tokens, values[0].dim, values[0].bitwidth, values[0].codes.word_bits,
                              out.data.data()));
    return out;
}

inline std::vector<float> naive_qk(std::span<const float> q, const DenseMatrix& k) {
    if (q.size() != k.cols) throw domain_error("naive_qk: query length does not match key cols");
    std::vector<float> out(k.rows);
    capi::check(kvq_naive_qk(q.data(), k.data.data(), k.rows, k.cols, out.data()));
    return out;
}

inline std::vector<float> naive_wv(std::span<const float> w, const DenseMatrix& v) {
    if (w.size() != v.rows) throw domain_error("naive_wv: weight length does not match value rows");
    std::vector<float> out(v.cols);
    capi::check(kvq_naive_wv(w.data(), v.data.data(), v.rows, v.cols, out.data()));
    return out;
}

}  // namespace kvq
