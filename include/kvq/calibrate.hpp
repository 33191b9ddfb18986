// kvq/calibrate.hpp — decode-time score calibration (reference calibrate.hpp:26-125).
// The softmax entry points run on the GPU (kvq_calibrated_softmax_concat). g itself is
// an affine scalar formula kept inline for API parity (no hot-path compute runs here).
#pragma once

#include <algorithm>
#include <cmath>
#include <span>
#include <vector>

#include "kvq/kernels.hpp"

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

}  // namespace kvq
