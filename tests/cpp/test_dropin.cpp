// test_dropin.cpp — the reference's own known-answer tests, re-run against the B200
// drop-in headers (include/kvq/*.hpp -> libkvq_b200.so). Plain asserts (Catch2 is not
// available); exit 0 = pass. Cited per case: /root/reference/proj/tests/*.cpp.
#include <cmath>
#include <cstdio>
#include <random>
#include <sstream>
#include <fstream>
#include <vector>

#include "kvq/kvq.hpp"

using namespace kvq;

static int g_fail = 0;
#define CHECK(cond)                                                        \
    do {                                                                   \
        if (!(cond)) {                                                     \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);    \
            ++g_fail;                                                      \
        }                                                                  \
    } while (0)
#define CHECK_THROWS(expr, type)                                           \
    do {                                                                   \
        bool caught = false;                                               \
        try { (void)(expr); } catch (const type&) { caught = true; }       \
        if (!caught) { std::printf("FAIL %s:%d: no " #type "\n", __FILE__, __LINE__); ++g_fail; } \
    } while (0)

static DenseMatrix random_matrix(std::mt19937_64& eng, std::size_t r, std::size_t c, float lo, float hi) {
    std::uniform_real_distribution<float> d(lo, hi);
    DenseMatrix m(r, c);
    for (float& v : m.data) v = d(eng);
    return m;
}

// double-precision attention (reference.hpp:26-54 restated)
static std::vector<double> attention(std::span<const float> q, const DenseMatrix& k, const DenseMatrix& v) {
    std::vector<double> s(k.rows);
    double m = -1e300;
    for (std::size_t j = 0; j < k.rows; ++j) {
        double a = 0;
        for (std::size_t c = 0; c < k.cols; ++c) a += (double)q[c] * k.at(j, c);
        s[j] = a / std::sqrt((double)k.cols);
        m = std::max(m, s[j]);
    }
    double sum = 0;
    for (double& x : s) sum += (x = std::exp(x - m));
    std::vector<double> out(v.cols, 0.0);
    for (std::size_t c = 0; c < v.cols; ++c)
        for (std::size_t j = 0; j < k.rows; ++j) out[c] += s[j] / sum * v.at(j, c);
    return out;
}

int main() {
    // test_bitpack.cpp:12-52, 126-140
    CHECK(pack(std::vector<std::uint32_t>{3, 1, 0, 2}, 2, 8).bytes == std::vector<std::uint8_t>{210});
    CHECK(pack(std::vector<std::uint32_t>{1, 0, 1, 1, 0, 0, 1, 0}, 1, 8).bytes[0] == 178);
    {
        PackedBuffer b = pack(std::vector<std::uint32_t>{1, 2, 3}, 4, 16);
        CHECK(b.word_at(0) == 0x1230u && b.bytes[0] == 0x30 && b.bytes[1] == 0x12);
        CHECK((unpack(b) == std::vector<std::uint32_t>{1, 2, 3}));
    }
    CHECK_THROWS(pack(std::vector<std::uint32_t>{4}, 2, 8), domain_error);
    CHECK_THROWS(pack(std::vector<std::uint32_t>{1}, 3, 8), config_error);

    // test_quantize.cpp:34-67
    {
        DenseMatrix m(2, 2, {1, 5, 3, 2});
        ChannelStats s = compute_stats(m, QuantMode::channel_wise);
        CHECK((s.alpha == std::vector<float>{1, 2}) && (s.beta == std::vector<float>{3, 5}));
        ChannelStats gs = compute_stats(m, QuantMode::global);
        CHECK((gs.alpha == std::vector<float>{1, 1}) && (gs.beta == std::vector<float>{5, 5}));
        CHECK_THROWS(compute_stats(DenseMatrix(0, 3), QuantMode::channel_wise), domain_error);
        auto q1 = [](float x, float a, float b, int bits) {
            return unpack(quantize(DenseMatrix(1, 1, {x}), ChannelStats{{a}, {b}}, bits).codes)[0];
        };
        CHECK(q1(1.4f, 0, 3, 2) == 1 && q1(0.1f, -2, 2, 1) == 1);
        CHECK(q1(0.5f, 0, 3, 2) == 1 && q1(1.5f, 0, 3, 2) == 2 && q1(2.5f, 0, 3, 2) == 3);
        CHECK(q1(99.f, -1.5f, 2.5f, 4) == 15 && q1(-99.f, -1.5f, 2.5f, 4) == 0);
    }

    // test_kernels.cpp:37-46, 111-121
    {
        QuantizedSegment seg = quantize(DenseMatrix(1, 2, {1, 0}), ChannelStats{{0, 0}, {1, 1}}, 1);
        std::vector<float> q = {2, 3};
        CHECK(qk_scores(q, seg, KernelConfig{})[0] == 2.0f);
        std::mt19937_64 rng(6);
        DenseMatrix m = random_matrix(rng, 9, 11, -2, 2);
        QuantizedSegment s4 = quantize(m, compute_stats(m, QuantMode::channel_wise), 4);
        DenseMatrix deq = dequantize(s4);
        std::vector<float> w(9, 0.0f);
        w[4] = 1.0f;
        std::vector<float> out = wv_output(w, s4, KernelConfig{});
        for (std::size_t c = 0; c < 11; ++c) CHECK(out[c] == deq.at(4, c));
        CHECK_THROWS(qk_scores(std::vector<float>(3), s4, KernelConfig{}), domain_error);
        CHECK_THROWS(qk_scores(std::vector<float>(11), s4, KernelConfig{0, 1, 1}), config_error);
    }

    // test_calibrate.cpp:60-66, 134-147
    {
        ScoreRange r{0.0f, 10.0f};
        CalibrationParams p{2.0f, 1.0f};
        CHECK(g_apply(0.0f, r, p) == -2.0f && g_apply(10.0f, r, p) == 9.0f && g_apply(5.0f, r, p) == 3.5f);
        std::vector<float> got = calibrated_softmax_concat(std::vector<float>{0, 10}, std::vector<float>{9}, p);
        std::vector<float> want = softmax_row(std::vector<float>{-2, 9, 9});
        for (int i = 0; i < 3; ++i) CHECK(std::abs(got[i] - want[i]) <= 1e-6f);
        std::size_t viol = 0;
        calibrated_softmax_concat(std::vector<float>{0.0f, 1e-4f}, {}, CalibrationParams{0, 3}, &viol);
        CHECK(viol == 1);
    }

    // test_kvcache.cpp:82-110 (8-bit decode tracks the oracle through appends), 112-140
    // (append never touches codes), 161-182 (weights sum to 1), 272-293 (memory law)
    {
        std::mt19937_64 rng(2);
        const std::size_t h = 2, n = 48, d = 12;
        std::vector<DenseMatrix> ks, vs;
        for (std::size_t i = 0; i < h; ++i) {
            ks.push_back(random_matrix(rng, n, d, 4, 12));
            vs.push_back(random_matrix(rng, n, d, 4, 12));
        }
        HybridKVCache cache = HybridKVCache::build(ks, vs, QuantizationConfig{8, QuantMode::channel_wise, 8},
                                                   CalibrationParams{});
        std::vector<std::uint8_t> before = cache.key_segment(0).codes.bytes;
        std::vector<DenseMatrix> fk = ks, fv = vs;
        for (int step = 0; step < 6; ++step) {
            DenseMatrix kn = random_matrix(rng, h, d, 4, 12), vn = random_matrix(rng, h, d, 4, 12);
            cache.append(kn, vn);
            for (std::size_t i = 0; i < h; ++i) {
                fk[i].append_row(kn.row_span(i));
                fv[i].append_row(vn.row_span(i));
            }
            DenseMatrix q = random_matrix(rng, h, d, -0.5f, 0.5f);
            DenseMatrix out = cache.decode_step(q);
            for (std::size_t i = 0; i < h; ++i) {
                std::vector<double> want = attention(q.row_span(i), fk[i], fv[i]);
                for (std::size_t c = 0; c < d; ++c)
                    CHECK(std::abs(out.at(i, c) - want[c]) <= 1e-3 * std::max(std::abs(want[c]), 1e-6));
            }
            DecodeDetail det = cache.decode_step_detailed(q);
            for (std::size_t i = 0; i < h; ++i) {
                double sum = 0;
                for (float w : det.weights.row_span(i)) sum += w;
                CHECK(std::abs(sum - 1.0) <= 1e-5);
            }
        }
        CHECK(cache.key_segment(0).codes.bytes == before);
        CHECK(cache.vis_tokens() == n && cache.tail_tokens() == 6);
        CHECK_THROWS(cache.append(DenseMatrix(h, d + 1), DenseMatrix(h, d + 1)), domain_error);
    }
    {
        std::mt19937_64 rng(9);
        DenseMatrix k = random_matrix(rng, 1024, 64, -1, 1);
        HybridKVCache cache = HybridKVCache::build(std::vector<DenseMatrix>{k}, std::vector<DenseMatrix>{k},
                                                   QuantizationConfig{1, QuantMode::channel_wise, 8}, CalibrationParams{});
        CHECK(cache.memory().quantized_bytes == 17408);
        CHECK_THROWS(HybridKVCache::build(std::vector<DenseMatrix>{k}, std::vector<DenseMatrix>{k},
                                          QuantizationConfig{3, QuantMode::channel_wise, 8}, CalibrationParams{}),
                     config_error);
    }
    // d = 128 tensor-core path through the drop-in: 1-bit, calibration, vs a generic-path
    // twin of the same cache (same codes, different kernels).
    {
        std::mt19937_64 rng(12);
        std::vector<DenseMatrix> ks, vs;
        for (int i = 0; i < 2; ++i) {
            ks.push_back(random_matrix(rng, 700, 128, -2, 2));
            vs.push_back(random_matrix(rng, 700, 128, -2, 2));
        }
        HybridKVCache a = HybridKVCache::build(ks, vs, QuantizationConfig{1, QuantMode::channel_wise, 8},
                                               CalibrationParams{1, 0});
        DenseMatrix q = random_matrix(rng, 2, 128, -1, 1);
        DenseMatrix fast = a.decode_step(q);
        DenseMatrix slow = a.decode_step_detailed(q).outputs;  // generic path (weights export)
        double err = 0, norm = 0;
        for (std::size_t i = 0; i < fast.data.size(); ++i) {
            err += (fast.data[i] - slow.data[i]) * (double)(fast.data[i] - slow.data[i]);
            norm += (double)slow.data[i] * slow.data[i];
        }
        CHECK(std::sqrt(err / norm) <= 1e-4);
    }
    // Offline tau search (test_calibrate.cpp:212-263 analogue): outlier-channel keys at 1 bit
    // prefer a non-identity calibration; the table's argmin is grid_search's answer.
    {
        std::mt19937_64 rng(31);
        std::vector<CalibrationSample> set;
        for (int s = 0; s < 2; ++s) {
            DenseMatrix k = random_matrix(rng, 384, 64, -1, 1);
            for (std::size_t r = 0; r < k.rows; ++r)
                for (std::size_t c = 0; c < 3; ++c) k.at(r, c) *= 8.0f;
            ChannelStats st = compute_stats(k, QuantMode::channel_wise);
            DenseMatrix qm = random_matrix(rng, 1, 64, -1, 1);
            set.push_back({qm.data, k, quantize(k, st, 1, 8)});
        }
        std::vector<GridCell> table = grid_mse_table(set, default_grid());
        CHECK(table.size() == 16);
        CalibrationParams best = grid_search(set);
        std::size_t arg = 0;
        for (std::size_t i = 1; i < table.size(); ++i)
            if (table[i].mse < table[arg].mse) arg = i;
        CHECK(table[arg].params == best);
        CHECK_THROWS(grid_search(std::span<const CalibrationSample>{}), domain_error);
    }
    // mse_report (test_calibrate.cpp:272-305 analogue): every head and bin covered, ragged heads.
    {
        std::mt19937_64 rng(41);
        std::vector<HeadWorkload> heads;
        for (std::size_t n : {50, 50, 70}) {
            HeadWorkload w{random_matrix(rng, n, 8, -1, 1), random_matrix(rng, n, 8, -1, 1), random_matrix(rng, 1, 8, -1, 1)};
            heads.push_back(std::move(w));
        }
        QuantizationConfig qcfg{1, QuantMode::channel_wise, 8};
        MseReport report = mse_report(heads, qcfg, CalibrationParams{1.0f, 0.0f}, 12);
        CHECK(report.rows.size() == 3 && report.histograms.size() == 3);
        double mq = 0.0;
        for (std::size_t h = 0; h < 3; ++h) {
            CHECK(report.rows[h].head == h && report.rows[h].mse_quant >= 0.0);
            mq += report.rows[h].mse_quant;
            CHECK(report.histograms[h].edges.size() == 13);
            for (const auto& counts : report.histograms[h].counts) {
                std::uint64_t total = 0;
                for (std::uint64_t c : counts) total += c;
                CHECK(total == heads[h].keys.rows);
            }
        }
        CHECK(std::abs(report.mean_mse_quant - mq / 3.0) <= 1e-12);
        CHECK_THROWS(mse_report(std::span<const HeadWorkload>{}, qcfg, CalibrationParams{}), domain_error);
        CHECK_THROWS(mse_report(heads, qcfg, CalibrationParams{}, 0), config_error);
    }
    // Snapshots (test_kvcache.cpp:307-395, test_quantize.cpp:233-290, test_tensor.cpp:69-141).
    {
        std::mt19937_64 rng(11);
        std::vector<DenseMatrix> ks, vs;
        for (int h = 0; h < 2; ++h) ks.push_back(random_matrix(rng, 24, 8, -2, 2)), vs.push_back(random_matrix(rng, 24, 8, -2, 2));
        HybridKVCache cache = HybridKVCache::build(ks, vs, QuantizationConfig{4, QuantMode::channel_wise, 8},
                                                   CalibrationParams{2.0f, 1.0f});
        DenseMatrix kn = random_matrix(rng, 2, 8, -2, 2);
        cache.append(kn, kn);
        DenseMatrix q = random_matrix(rng, 2, 8, -1, 1);
        std::stringstream ss;
        cache.save(ss);
        ss << "after";  // data following the image stays in the stream
        std::uint64_t off = 0;
        HybridKVCache back = HybridKVCache::load(ss, off);
        std::string rest;
        ss >> rest;
        CHECK(rest == "after");
        CHECK(off == ss.str().size() - 5);
        CHECK(back.heads() == 2 && back.dim() == 8 && back.bitwidth() == 4 && back.tail_tokens() == 1);
        CHECK(back.calibration() == (CalibrationParams{2.0f, 1.0f}));
        CHECK(back.decode_step(q).data == cache.decode_step(q).data);
        CHECK(back.memory().total_bytes == cache.memory().total_bytes);
        const std::string path = "/tmp/kvq_dropin_cache.kvqc";
        cache.save(path);
        CHECK(HybridKVCache::load(path).decode_step(q).data == cache.decode_step(q).data);
        { std::ofstream os(path, std::ios::binary | std::ios::app); os << "x"; }
        CHECK_THROWS(HybridKVCache::load(path), format_error);
        std::string bytes = ss.str().substr(0, ss.str().size() - 5);
        bytes[0] = 'Z';
        std::stringstream bad(bytes);
        off = 0;
        try {
            HybridKVCache::load(bad, off);
            CHECK(false);
        } catch (const format_error& e) {
            CHECK(e.offset() == 0);
        }
        // KVQP + KVQT records
        QuantizedSegment seg = cache.key_segment(0);
        std::stringstream s2;
        write_segment(s2, seg);
        off = 0;
        QuantizedSegment seg2 = read_segment(s2, off);
        CHECK(seg2.codes.bytes == seg.codes.bytes && seg2.stats.alpha == seg.stats.alpha && seg2.tokens == 24);
        DenseMatrix t = cache.key_tail(1);
        std::stringstream s3;
        write_tensor(s3, t);
        off = 0;
        CHECK(read_tensor(s3, off) == t);
        CHECK(off == 24 + 4 * 8);
    }
    std::printf(g_fail ? "test_dropin: %d failures\n" : "test_dropin: all passed%.0d\n", g_fail);
    return g_fail ? 1 : 0;
}
