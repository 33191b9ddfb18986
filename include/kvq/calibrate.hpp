// kvq/calibrate.hpp — decode-time score calibration (reference calibrate.hpp:26-125).
// The softmax entry points run on the GPU (kvq_calibrated_softmax_concat). g itself is
// an affine scalar formula kept inline for API parity (no hot-path compute runs here).
#pragma once

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <span>
#include <string>
#include <vector>

#include "kvq/kernels.hpp"
#include "kvq/quantize.hpp"
#include "kvq/workload.hpp"

namespace kvq {

struct CalibrationParams {
    float tau1 = 0.0f;
    float tau2 = 0.0f;
    bool identity() const { return tau1 == 0.0f && tau2 == 0.0f; }
    bool operator==(const CalibrationParams&) const = default;
};

struct ScoreRange {
    float gamma = 0.0f;  // row minimum
    float delta = 0.0f;  // row maximum
};

inline ScoreRange row_range(std::span<const float> row) {
    if (row.empty()) throw domain_error("row_range: empty row");
    const auto [lo, hi] = std::minmax_element(row.begin(), row.end());
    return ScoreRange{*lo, *hi};
}

// Slope of g is positive iff (delta - gamma) + (tau1 - tau2) > 0 (calibrate.hpp:52-54).
inline bool g_monotone(const ScoreRange& r, const CalibrationParams& p) {
    return (r.delta - r.gamma) + (p.tau1 - p.tau2) > 0.0f;
}

// g maps [gamma, delta] onto [gamma - tau1, delta - tau2] (calibrate.hpp:62-67).
inline float g_apply(float x, const ScoreRange& r, const CalibrationParams& p) {
    const float width = r.delta - r.gamma;
    if (width <= 0.0f) return x - p.tau1;
    const float frac = (x - r.gamma) / width;
    return x - (p.tau1 * (1.0f - frac) + p.tau2 * frac);
}

inline std::vector<float> calibrated_softmax_concat(std::span<const float> vis, std::span<const float> tail,
                                                    const CalibrationParams& p,
                                                    std::size_t* slope_violations = nullptr) {
    std::vector<float> out(vis.size() + tail.size());
    if (out.empty()) return out;
    capi::check(kvq_calibrated_softmax_concat(vis.data(), vis.size(), tail.data(), tail.size(), 1, p.tau1, p.tau2,
                                              out.data(), slope_violations));
    return out;
}

inline std::vector<float> softmax_row(std::span<const float> row) {
    return calibrated_softmax_concat({}, row, CalibrationParams{});
}

inline std::vector<float> calibrated_scores(std::span<const float> q, const QuantizedSegment& keys,
                                            const CalibrationParams& p, const KernelConfig& cfg = {}) {
    std::vector<float> s = qk_scores(q, keys, cfg);
    const float inv_sqrt_d = 1.0f / std::sqrt(static_cast<float>(keys.dim));
    for (float& v : s) v *= inv_sqrt_d;
    return calibrated_softmax_concat(s, {}, p);
}

// ---- offline tau search (calibrate.hpp:127-234), scored on the GPU ---------------------

struct CalibrationSample {
    std::vector<float> query;
    DenseMatrix keys_exact;       // n x d full-precision keys
    QuantizedSegment keys_quant;  // same tokens, packed
};

struct GridCell {
    CalibrationParams params;
    double mse = 0.0;
};

inline std::vector<CalibrationParams> make_grid(std::vector<float> values) {
    if (values.empty()) throw domain_error("make_grid: empty value list");
    std::sort(values.begin(), values.end());
    std::vector<CalibrationParams> cells;
    cells.reserve(values.size() * values.size());
    for (float t1 : values)
        for (float t2 : values) cells.push_back({t1, t2});
    return cells;
}

inline std::vector<CalibrationParams> default_grid() { return make_grid({0.0f, 1.0f, 2.0f, 3.0f}); }

namespace detail {
// One C-ABI call: the mean MSE per cell and the argmin (ties: smaller tau1, then tau2).
inline std::vector<double> grid_call(std::span<const CalibrationSample> set, std::span<const CalibrationParams> cells,
                                     CalibrationParams* best) {
    if (set.empty()) throw domain_error("grid_mse_table: empty calibration set");
    if (cells.empty()) throw domain_error("grid_mse_table: empty grid");
    const std::size_t n = set[0].keys_exact.rows, d = set[0].keys_exact.cols;
    const int bits = set[0].keys_quant.bitwidth, wb = set[0].keys_quant.codes.word_bits;
    std::vector<float> q, ke, alpha, beta;
    std::vector<std::uint8_t> codes;
    for (std::size_t i = 0; i < set.size(); ++i) {
        const CalibrationSample& s = set[i];
        if (s.query.size() != d || s.keys_exact.rows != n || s.keys_exact.cols != d || s.keys_quant.dim != d ||
            s.keys_quant.tokens != n || s.keys_quant.bitwidth != bits || s.keys_quant.codes.word_bits != wb)
            throw domain_error("calibration sample " + std::to_string(i) + " has inconsistent shapes");
        q.insert(q.end(), s.query.begin(), s.query.end());
        ke.insert(ke.end(), s.keys_exact.data.begin(), s.keys_exact.data.end());
        codes.insert(codes.end(), s.keys_quant.codes.bytes.begin(), s.keys_quant.codes.bytes.end());
        alpha.insert(alpha.end(), s.keys_quant.stats.alpha.begin(), s.keys_quant.stats.alpha.end());
        beta.insert(beta.end(), s.keys_quant.stats.beta.begin(), s.keys_quant.stats.beta.end());
    }
    std::vector<float> t1, t2;
    for (const auto& c : cells) t1.push_back(c.tau1), t2.push_back(c.tau2);
    std::vector<double> mse(cells.size());
    float b[2] = {0.0f, 0.0f};
    capi::check(kvq_grid_mse_table(q.data(), ke.data(), codes.data(), alpha.data(), beta.data(), set.size(), n, d,
                                   bits, wb, t1.data(), t2.data(), cells.size(), mse.data(), b));
    if (best) *best = CalibrationParams{b[0], b[1]};
    return mse;
}
}  // namespace detail

inline std::vector<GridCell> grid_mse_table(std::span<const CalibrationSample> set,
                                            std::span<const CalibrationParams> cells, const KernelConfig& cfg = {}) {
    cfg.validate();
    std::vector<double> mse = detail::grid_call(set, cells, nullptr);
    std::vector<GridCell> table(cells.size());
    for (std::size_t c = 0; c < cells.size(); ++c) table[c] = {cells[c], mse[c]};
    return table;
}

inline CalibrationParams grid_search(std::span<const CalibrationSample> set, std::span<const CalibrationParams> cells,
                                     const KernelConfig& cfg = {}) {
    cfg.validate();
    CalibrationParams best;
    detail::grid_call(set, cells, &best);
    return best;
}

inline CalibrationParams grid_search(std::span<const CalibrationSample> set, const KernelConfig& cfg = {}) {
    std::vector<CalibrationParams> cells = default_grid();
    return grid_search(set, cells, cfg);
}

// ---- diagnostics (calibrate.hpp:236-397): per-head softmax MSE of the quant / quant_c
// rows against the exact row and shared-edge histograms, computed on the GPU
// (kvq_mse_report); the CSV writers are host formatting.

enum class ScoreVariant { exact = 0, quant = 1, quant_c = 2 };

inline const char* variant_name(ScoreVariant v) {
    switch (v) {
        case ScoreVariant::exact: return "exact";
        case ScoreVariant::quant: return "quant";
        default: return "quant_c";
    }
}

struct MseRow {
    std::size_t head = 0;
    double mse_quant = 0.0;
    double mse_quant_c = 0.0;
};

struct HeadHistogram {
    std::size_t head = 0;
    std::vector<float> edges;                          // bins + 1, shared by the variants
    std::array<std::vector<std::uint64_t>, 3> counts;  // indexed by ScoreVariant
};

struct MseReport {
    std::vector<MseRow> rows;
    std::vector<HeadHistogram> histograms;
    double mean_mse_quant = 0.0;
    double mean_mse_quant_c = 0.0;
};

inline MseReport mse_report(std::span<const HeadWorkload> heads, const QuantizationConfig& qcfg,
                            const CalibrationParams& p, std::size_t bins = 40, const KernelConfig& kcfg = {}) {
    if (heads.empty()) throw domain_error("mse_report: no heads");
    if (bins < 1) throw config_error("mse_report: bins must be >= 1");
    qcfg.validate();
    kcfg.validate();
    MseReport report;
    for (std::size_t i = 0; i < heads.size();) {  // runs of equal-shape heads: one device call
        const std::size_t n = heads[i].keys.rows, d = heads[i].keys.cols;
        std::size_t j = i;
        std::vector<float> q, k;
        for (; j < heads.size() && heads[j].keys.rows == n && heads[j].keys.cols == d; ++j) {
            if (heads[j].query.data.size() != d) throw domain_error("naive_qk: query length does not match key cols");
            q.insert(q.end(), heads[j].query.data.begin(), heads[j].query.data.end());
            k.insert(k.end(), heads[j].keys.data.begin(), heads[j].keys.data.end());
        }
        const std::size_t h = j - i;
        std::vector<double> mq(h), mc(h);
        std::vector<float> edges(h * (bins + 1));
        std::vector<std::uint64_t> counts(h * 3 * bins);
        capi::check(kvq_mse_report(q.data(), k.data(), h, n, d, qcfg.bitwidth, static_cast<int>(qcfg.mode),
                                   qcfg.word_bits, p.tau1, p.tau2, bins, mq.data(), mc.data(), edges.data(),
                                   counts.data()));
        for (std::size_t x = 0; x < h; ++x) {
            report.rows.push_back({i + x, mq[x], mc[x]});
            HeadHistogram hist;
            hist.head = i + x;
            hist.edges.assign(edges.begin() + x * (bins + 1), edges.begin() + (x + 1) * (bins + 1));
            for (int v = 0; v < 3; ++v)
                hist.counts[v].assign(counts.begin() + (x * 3 + v) * bins, counts.begin() + (x * 3 + v + 1) * bins);
            report.histograms.push_back(std::move(hist));
        }
        i = j;
    }
    for (const MseRow& r : report.rows) {
        report.mean_mse_quant += r.mse_quant;
        report.mean_mse_quant_c += r.mse_quant_c;
    }
    report.mean_mse_quant /= static_cast<double>(heads.size());
    report.mean_mse_quant_c /= static_cast<double>(heads.size());
    return report;
}

namespace detail {
inline std::string fmt_real(double v) {
    char buf[48];
    std::snprintf(buf, sizeof(buf), "%.9g", v);
    return buf;
}
inline std::ofstream open_csv(const std::string& path) {
    std::ofstream os(path);
    if (!os) throw format_error("cannot open for writing: " + path, 0);
    return os;
}
}  // namespace detail

// columns: variant,head,mse (exact rows carry 0 by definition)
inline void write_mse_csv(const std::string& path, const MseReport& report) {
    std::ofstream os = detail::open_csv(path);
    os << "variant,head,mse\n";
    for (const MseRow& r : report.rows) os << "exact," << r.head << ",0\n";
    for (const MseRow& r : report.rows) os << "quant," << r.head << "," << detail::fmt_real(r.mse_quant) << "\n";
    for (const MseRow& r : report.rows) os << "quant_c," << r.head << "," << detail::fmt_real(r.mse_quant_c) << "\n";
    if (!os) throw format_error("write failed: " + path, 0);
}

// columns: variant,head,bin_left,bin_right,count
inline void write_histogram_csv(const std::string& path, const MseReport& report) {
    std::ofstream os = detail::open_csv(path);
    os << "variant,head,bin_left,bin_right,count\n";
    for (const HeadHistogram& h : report.histograms)
        for (int v = 0; v < 3; ++v)
            for (std::size_t b = 0; b + 1 < h.edges.size(); ++b)
                os << variant_name(static_cast<ScoreVariant>(v)) << "," << h.head << "," << detail::fmt_real(h.edges[b])
                   << "," << detail::fmt_real(h.edges[b + 1]) << "," << h.counts[static_cast<std::size_t>(v)][b]
                   << "\n";
    if (!os) throw format_error("write failed: " + path, 0);
}

}  // namespace kvq
