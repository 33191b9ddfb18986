// kvq/kvcache.hpp — HybridKVCache (reference kvcache.hpp:43-319) backed by a
// device-resident kvq_cache: packed K/V segments, stats and the fp32 tail live in HBM;
// build runs K1, append runs K3, decode runs K2 (tensor-core path at d = 128, generic
// path otherwise and for decode_step_detailed).
//
// Ownership differs from the reference in one respect: the cache owns device memory,
// so it is move-only (copying would silently duplicate HBM state). Accessors return
// host copies instead of references into host vectors.
#pragma once

#include <fstream>
#include <istream>
#include <iterator>
#include <memory>
#include <ostream>
#include <span>
#include <string>
#include <vector>

#include "kvq/calibrate.hpp"

namespace kvq {

inline constexpr int kFullPrecisionBits = KVQ_FULL_PRECISION_BITS;

struct CacheMemory {
    std::size_t code_bytes = 0;
    std::size_t stats_bytes = 0;
    std::size_t quantized_bytes = 0;
    std::size_t tail_bytes = 0;
    std::size_t fp32_vis_bytes = 0;
    std::size_t total_bytes = 0;
};

struct DecodeDetail {
    DenseMatrix outputs;  // heads x dim
    DenseMatrix weights;  // heads x (n_vis + n_tail)
    std::size_t slope_violations = 0;
};

class HybridKVCache {
public:
    static HybridKVCache build(std::span<const DenseMatrix> k_vis, std::span<const DenseMatrix> v_vis,
                               const QuantizationConfig& cfg, const CalibrationParams& cal) {
        cfg.validate();
        return make(k_vis, v_vis, cfg.bitwidth, to_capi(cfg.mode), cfg.word_bits, cal);
    }

    static HybridKVCache build_full_precision(std::span<const DenseMatrix> k, std::span<const DenseMatrix> v) {
        return make(k, v, kFullPrecisionBits, KVQ_MODE_CHANNEL_WISE, 8, CalibrationParams{});
    }

    std::size_t heads() const { return info(1); }
    std::size_t dim() const { return info(3); }
    int bitwidth() const { return static_cast<int>(info(6)); }
    CalibrationParams calibration() const {
        float tau[2];
        kvq_cache_calibration(handle_.get(), tau);
        return CalibrationParams{tau[0], tau[1]};
    }
    std::size_t vis_tokens() const { return info(4); }
    std::size_t tail_tokens() const { return info(5); }
    std::size_t total_tokens() const { return vis_tokens() + tail_tokens(); }

    QuantizedSegment key_segment(std::size_t h) const { return segment(h, 0); }
    QuantizedSegment value_segment(std::size_t h) const { return segment(h, 1); }
    DenseMatrix key_tail(std::size_t h) const { return tail(h, 0); }
    DenseMatrix value_tail(std::size_t h) const { return tail(h, 1); }

    void append(const DenseMatrix& k_new, const DenseMatrix& v_new) {
        if (k_new.rows != heads() || v_new.rows != heads() || k_new.cols != dim() || v_new.cols != dim())
            throw domain_error("append: expected " + std::to_string(heads()) + " x " + std::to_string(dim()) +
                               " new key/value rows");
        capi::check(kvq_cache_append(handle_.get(), k_new.data.data(), v_new.data.data()));
    }

    DenseMatrix decode_step(const DenseMatrix& queries, const KernelConfig& cfg = {}) const {
        check_queries(queries, cfg);
        DenseMatrix out(heads(), dim());
        capi::check(kvq_cache_decode(handle_.get(), queries.data.data(), out.data.data(), nullptr, nullptr));
        return out;
    }

    DecodeDetail decode_step_detailed(const DenseMatrix& queries, const KernelConfig& cfg = {}) const {
        check_queries(queries, cfg);
        DecodeDetail d;
        d.outputs = DenseMatrix(heads(), dim());
        d.weights = DenseMatrix(heads(), total_tokens());
        std::vector<float> w(std::max<std::size_t>(d.weights.data.size(), 1));
        capi::check(kvq_cache_decode(handle_.get(), queries.data.data(), d.outputs.data.data(), w.data(),
                                     &d.slope_violations));
        std::copy(w.begin(), w.begin() + static_cast<std::ptrdiff_t>(d.weights.data.size()), d.weights.data.begin());
        return d;
    }

    CacheMemory memory() const {
        std::size_t m[6];
        kvq_cache_memory(handle_.get(), m);
        return CacheMemory{m[0], m[1], m[2], m[3], m[4], m[5]};
    }

    // ---- snapshots (kvcache.hpp:137-218): the reference's KVQC bytes; the device cache
    // is gathered into the image by strided device->host copies (kvq_cache_save_image).
    void save(std::ostream& os) const {
        std::size_t n = 0;
        capi::check(kvq_cache_image_bytes(handle_.get(), &n));
        std::vector<char> img(n);
        capi::check(kvq_cache_save_image(handle_.get(), img.data(), n, 0, nullptr));
        os.write(img.data(), static_cast<std::streamsize>(n));
    }

    void save(const std::string& path) const {
        std::ofstream os(path, std::ios::binary);
        if (!os) throw format_error("cannot open for writing: " + path, 0);
        save(os);
        if (!os) throw format_error("write failed: " + path, 0);
    }

    // Reads the stream's remaining bytes, parses one cache image from them and leaves the
    // stream just past it (seekable streams); `off` advances like the reference's.
    static HybridKVCache load(std::istream& is, std::uint64_t& off) {
        const std::istream::pos_type start = is.tellg();
        std::string img((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
        std::size_t used = 0;
        HybridKVCache out = from_image(img, off, &used);
        is.clear();
        if (start != std::istream::pos_type(-1)) is.seekg(start + static_cast<std::streamoff>(used));
        return out;
    }

    static HybridKVCache load(const std::string& path) {
        std::ifstream is(path, std::ios::binary);
        if (!is) throw format_error("cannot open for reading: " + path, 0);
        std::string img((std::istreambuf_iterator<char>(is)), std::istreambuf_iterator<char>());
        std::uint64_t off = 0;
        std::size_t used = 0;
        HybridKVCache out = from_image(img, off, &used);
        if (used != img.size()) throw format_error("trailing bytes after cache data", used);
        return out;
    }

    kvq_cache* native() const { return handle_.get(); }

private:
    struct Free {
        void operator()(kvq_cache* c) const { kvq_cache_free(c); }
    };
    std::unique_ptr<kvq_cache, Free> handle_;

    static HybridKVCache make(std::span<const DenseMatrix> k, std::span<const DenseMatrix> v, int bits, int mode,
                              int word_bits, const CalibrationParams& cal) {
        // check_prefill (kvcache.hpp:224-236)
        if (k.empty() || k.size() != v.size())
            throw domain_error("cache build: need matching per-head key/value lists");
        for (std::size_t h = 0; h < k.size(); ++h)
            if (k[h].rows != k[0].rows || k[h].cols != k[0].cols || v[h].rows != k[0].rows || v[h].cols != k[0].cols)
                throw domain_error("cache build: head " + std::to_string(h) + " shape differs from head 0");
        if (k[0].cols == 0) throw domain_error("cache build: head dim must be positive");
        const std::size_t n = k[0].rows, d = k[0].cols;
        std::vector<float> kf, vf;
        kf.reserve(k.size() * n * d + 1);
        vf.reserve(k.size() * n * d + 1);
        for (std::size_t h = 0; h < k.size(); ++h) {
            kf.insert(kf.end(), k[h].data.begin(), k[h].data.end());
            vf.insert(vf.end(), v[h].data.begin(), v[h].data.end());
        }
        kf.push_back(0.f);
        vf.push_back(0.f);
        kvq_cache* c = nullptr;
        capi::check(kvq_cache_build(kf.data(), vf.data(), 1, k.size(), 1, n, d, bits, mode, word_bits, cal.tau1,
                                    cal.tau2, &c));
        HybridKVCache out;
        out.handle_.reset(c);
        return out;
    }

    static HybridKVCache from_image(const std::string& img, std::uint64_t& off, std::size_t* used) {
        kvq_cache* c = nullptr;
        const int st = kvq_cache_load_image(img.data(), img.size(), 1, 1, used, &c);
        if (st == KVQ_ERR_FORMAT) throw format_error(capi::last_error(), off + kvq_last_error_offset());
        capi::check(st);
        off += *used;
        HybridKVCache out;
        out.handle_.reset(c);
        return out;
    }

    std::size_t info(int i) const {
        std::size_t v[10];
        kvq_cache_info(handle_.get(), v);
        return v[i];
    }

    void check_queries(const DenseMatrix& q, const KernelConfig& cfg) const {
        cfg.validate();
        if (q.rows != heads() || q.cols != dim())
            throw domain_error("decode_step: expected " + std::to_string(heads()) + " x " + std::to_string(dim()) +
                               " queries");
    }

    QuantizedSegment segment(std::size_t h, int which) const {
        QuantizedSegment s;
        const int bits = bitwidth() == kFullPrecisionBits ? 8 : bitwidth();
        const int wb = static_cast<int>(info(7));
        s.codes.code_bits = bits;
        s.codes.word_bits = wb;
        s.tokens = vis_tokens();
        s.dim = dim();
        s.bitwidth = bits;
        s.codes.bytes.resize(kvq_segment_bytes(s.tokens, s.dim, bits, wb));
        s.stats.alpha.resize(s.dim);
        s.stats.beta.resize(s.dim);
        capi::check(kvq_cache_read_segment(handle_.get(), h, which, s.codes.bytes.data(), s.stats.alpha.data(),
                                           s.stats.beta.data()));
        s.codes.logical_count = s.tokens * s.codes_per_row();
        return s;
    }

    DenseMatrix tail(std::size_t h, int which) const {
        DenseMatrix m(tail_tokens(), dim());
        if (!m.data.empty()) capi::check(kvq_cache_read_tail(handle_.get(), h, which, m.data.data()));
        return m;
    }
};

}  // namespace kvq
