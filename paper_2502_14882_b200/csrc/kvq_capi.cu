// kvq_capi.cu — the stateless C-ABI entry points (include/kvq_capi.h): packing, the
// quantizer, the kernel-level products, calibration and the offline calibration
// diagnostics, with the reference's argument validation and error classes. No compute
// happens on the host: every numeric result comes out of a CUDA kernel, and a missing
// device is a hard KVQ_ERR_CUDA. Cache objects: kvq_cache.cu; snapshots: kvq_snapshot.cu.
#include <atomic>

#include "capi_internal.cuh"

namespace kvqb {
static std::atomic<unsigned long long> g_launches{0};
void note_launch(unsigned n) { g_launches += n; }
unsigned long long launch_count() { return g_launches.load(); }
}  // namespace kvqb

using namespace kvqb::capi;

extern "C" {

size_t kvq_last_error(char* buf, size_t cap) {
    if (buf && cap) {
        size_t k = g_err.size() < cap - 1 ? g_err.size() : cap - 1;
        std::memcpy(buf, g_err.data(), k);
        buf[k] = '\0';
    }
    return g_err.size();
}

unsigned long long kvq_last_error_offset(void) { return g_err_offset; }

unsigned long long kvq_launch_count(void) { return kvqb::launch_count(); }

int kvq_set_device(int device) {
    return guarded([&] {
        int n = 0;
        ck(cudaGetDeviceCount(&n), "cudaGetDeviceCount");
        if (device < 0 || device >= n) raise(KVQ_ERR_DOMAIN, "set_device: no such CUDA device");
        ck(cudaSetDevice(device), "cudaSetDevice");
    });
}

int kvq_device_available(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n > 0 ? 1 : 0;
}

size_t kvq_packed_bytes(size_t count, int code_bits, int word_bits) {
    if (code_bits < 1 || word_bits < 8 || word_bits % code_bits) return 0;
    size_t g = (size_t)(word_bits / code_bits);
    return (count + g - 1) / g * (size_t)(word_bits / 8);
}

int kvq_pack(const uint32_t* codes, size_t count, int code_bits, int word_bits, uint8_t* out,
             size_t out_cap) {
    return guarded([&] {
        validate_widths(code_bits, word_bits);
        size_t nbytes = kvq_packed_bytes(count, code_bits, word_bits);
        if (out_cap < nbytes) raise(KVQ_ERR_DOMAIN, "pack: output buffer too small");
        if (count == 0) return;
        require_device();
        DevBuf<uint32_t> dc(count);
        DevBuf<uint8_t> db(nbytes);
        DevBuf<int> flag(1);
        dc.upload(codes, count);
        ck(cudaMemsetAsync(flag.p, 0, sizeof(int)), "memset");
        ck(kvqb::launch_pack_codes(dc.p, count, code_bits, word_bits, db.p, flag.p, 0), "pack");
        int bad = 0;
        flag.download(&bad, 1);
        db.download(out, nbytes);
        sync(0);
        if (bad) {
            // Report the first offending code, as the reference does (bitpack.hpp:178-181).
            uint32_t limit = code_bits >= 32 ? 0xffffffffu : (1u << code_bits) - 1u;
            for (size_t i = 0; i < count; ++i)
                if (codes[i] > limit)
                    raise(KVQ_ERR_DOMAIN, "code " + std::to_string(codes[i]) + " exceeds " +
                                              std::to_string(code_bits) + "-bit range");
        }
    });
}

int kvq_unpack(const uint8_t* bytes, size_t byte_len, size_t count, int code_bits, int word_bits,
               uint32_t* out) {
    return guarded([&] {
        validate_widths(code_bits, word_bits);
        size_t nbytes = kvq_packed_bytes(count, code_bits, word_bits);
        if (byte_len < nbytes) raise(KVQ_ERR_DOMAIN, "unpack: buffer shorter than logical_count implies");
        if (count == 0) return;
        require_device();
        DevBuf<uint8_t> db(nbytes);
        DevBuf<uint32_t> dc(count);
        db.upload(bytes, nbytes);
        ck(kvqb::launch_unpack_codes(db.p, count, code_bits, word_bits, dc.p, 0), "unpack");
        dc.download(out, count);
        sync(0);
    });
}

size_t kvq_segment_bytes(size_t tokens, size_t dim, int bitwidth, int word_bits) {
    if (bitwidth < 1 || word_bits < 8 || word_bits % bitwidth) return 0;
    return tokens * row_bytes(dim, bitwidth, word_bits);
}

int kvq_compute_stats(const float* m, size_t rows, size_t cols, int mode, float* alpha, float* beta) {
    return guarded([&] {
        if (rows == 0 || cols == 0) raise(KVQ_ERR_DOMAIN, "compute_stats: empty matrix");
        if (mode != KVQ_MODE_CHANNEL_WISE && mode != KVQ_MODE_GLOBAL) raise(KVQ_ERR_CONFIG, "unknown quant mode");
        require_device();
        DevBuf<float> dm(rows * cols), da(cols), dbt(cols);
        dm.upload(m, rows * cols);
        ck(kvqb::launch_compute_stats(dm.p, 1, rows, cols, mode, da.p, dbt.p, 0), "compute_stats");
        da.download(alpha, cols);
        dbt.download(beta, cols);
        sync(0);
    });
}

int kvq_quantize(const float* m, size_t rows, size_t cols, const float* alpha, const float* beta,
                 int bitwidth, int word_bits, uint8_t* out, size_t out_cap) {
    return guarded([&] {
        validate_quant_bits(bitwidth, word_bits);
        size_t nbytes = kvq_segment_bytes(rows, cols, bitwidth, word_bits);
        if (out_cap < nbytes) raise(KVQ_ERR_DOMAIN, "quantize: output buffer too small");
        if (nbytes == 0) return;
        require_device();
        DevBuf<float> dm(rows * cols), da(cols), dbt(cols);
        DevBuf<uint8_t> dc(nbytes);
        dm.upload(m, rows * cols);
        da.upload(alpha, cols);
        dbt.upload(beta, cols);
        ck(kvqb::launch_quantize_pack(dm.p, 1, rows, cols, da.p, dbt.p, bitwidth, word_bits, dc.p, 0), "quantize");
        dc.download(out, nbytes);
        sync(0);
    });
}

int kvq_dequantize(const uint8_t* codes, size_t rows, size_t cols, const float* alpha,
                   const float* beta, int bitwidth, int word_bits, float* out) {
    return guarded([&] {
        validate_quant_bits(bitwidth, word_bits);
        if (rows == 0 || cols == 0) return;
        require_device();
        size_t nbytes = kvq_segment_bytes(rows, cols, bitwidth, word_bits);
        DevBuf<uint8_t> dc(nbytes);
        DevBuf<float> da(cols), dbt(cols), dout(rows * cols);
        dc.upload(codes, nbytes);
        da.upload(alpha, cols);
        dbt.upload(beta, cols);
        ck(kvqb::launch_dequantize(dc.p, 1, rows, cols, da.p, dbt.p, bitwidth, word_bits, dout.p, 0), "dequantize");
        dout.download(out, rows * cols);
        sync(0);
    });
}

int kvq_quantize_device(const float* x, size_t mats, size_t rows, size_t dim, int bitwidth, int mode,
                        int word_bits, uint8_t* codes, float* alpha, float* beta, void* stream) {
    return guarded([&] {
        validate_config(bitwidth, word_bits);
        if (rows == 0 || dim == 0) raise(KVQ_ERR_DOMAIN, "compute_stats: empty matrix");
        require_device();
        cudaStream_t s = (cudaStream_t)stream;
        if (kvqb::quantize_fused_supported(rows, dim, word_bits, mode)) {
            ck(kvqb::launch_quantize_fused(x, mats, rows, dim, bitwidth, word_bits, mode, alpha, beta, codes, s),
               "quantize");
        } else {
            ck(kvqb::launch_compute_stats(x, mats, rows, dim, mode, alpha, beta, s), "compute_stats");
            ck(kvqb::launch_quantize_pack(x, mats, rows, dim, alpha, beta, bitwidth, word_bits, codes, s), "quantize");
        }
    });
}

int kvq_qk_scores(const float* queries, const uint8_t* codes, const float* alpha, const float* beta,
                  size_t heads, size_t tokens, size_t dim, int bitwidth, int word_bits, float* scores) {
    return guarded([&] {
        validate_quant_bits(bitwidth, word_bits);
        if (heads == 0 || tokens == 0) return;
        if (dim == 0) raise(KVQ_ERR_DOMAIN, "qk_scores: zero head dim");
        require_device();
        size_t seg = kvq_segment_bytes(tokens, dim, bitwidth, word_bits);
        DevBuf<float> dq(heads * dim), da(heads * dim), dbt(heads * dim), ds(heads * tokens);
        DevBuf<uint8_t> dc(heads * seg);
        dq.upload(queries, heads * dim);
        da.upload(alpha, heads * dim);
        dbt.upload(beta, heads * dim);
        dc.upload(codes, heads * seg);
        ck(kvqb::launch_qk_scores(dq.p, dc.p, da.p, dbt.p, heads, tokens, dim, bitwidth, word_bits, ds.p, 0),
           "qk_scores");
        ds.download(scores, heads * tokens);
        sync(0);
    });
}

int kvq_wv_output(const float* weights, const uint8_t* codes, const float* alpha, const float* beta,
                  size_t heads, size_t tokens, size_t dim, int bitwidth, int word_bits, float* out) {
    return guarded([&] {
        validate_quant_bits(bitwidth, word_bits);
        if (heads == 0 || dim == 0) return;
        require_device();
        size_t seg = kvq_segment_bytes(tokens, dim, bitwidth, word_bits);
        DevBuf<float> dw(heads * tokens), da(heads * dim), dbt(heads * dim), dout(heads * dim);
        DevBuf<uint8_t> dc(heads * seg);
        dw.upload(weights, heads * tokens);
        da.upload(alpha, heads * dim);
        dbt.upload(beta, heads * dim);
        dc.upload(codes, heads * seg);
        ck(kvqb::launch_wv_output(dw.p, dc.p, da.p, dbt.p, heads, tokens, dim, bitwidth, word_bits, dout.p, 0),
           "wv_output");
        dout.download(out, heads * dim);
        sync(0);
    });
}

int kvq_naive_qk(const float* q, const float* k, size_t rows, size_t cols, float* out) {
    return guarded([&] {
        if (rows == 0) return;
        require_device();
        DevBuf<float> dq(cols ? cols : 1), dk(rows * cols ? rows * cols : 1), dout(rows);
        dq.upload(q, cols);
        dk.upload(k, rows * cols);
        ck(kvqb::launch_naive_qk(dq.p, dk.p, rows, cols, dout.p, 0), "naive_qk");
        dout.download(out, rows);
        sync(0);
    });
}

int kvq_naive_wv(const float* w, const float* v, size_t rows, size_t cols, float* out) {
    return guarded([&] {
        if (cols == 0) return;
        require_device();
        DevBuf<float> dw(rows ? rows : 1), dv(rows * cols ? rows * cols : 1), dout(cols);
        dw.upload(w, rows);
        dv.upload(v, rows * cols);
        ck(kvqb::launch_naive_wv(dw.p, dv.p, rows, cols, dout.p, 0), "naive_wv");
        dout.download(out, cols);
        sync(0);
    });
}

int kvq_calibrated_softmax_concat(const float* vis, size_t n_vis, const float* tail, size_t n_tail,
                                  size_t rows, float tau1, float tau2, float* out,
                                  size_t* slope_violations) {
    return guarded([&] {
        if (rows == 0 || n_vis + n_tail == 0) return;
        require_device();
        DevBuf<float> dv(rows * n_vis), dt(rows * n_tail), dout(rows * (n_vis + n_tail));
        DevBuf<int> dviol(rows);
        dv.upload(vis, rows * n_vis);
        dt.upload(tail, rows * n_tail);
        ck(kvqb::launch_calibrated_softmax(dv.p, n_vis, dt.p, n_tail, rows, tau1, tau2, dout.p, dviol.p, 0),
           "calibrated_softmax_concat");
        dout.download(out, rows * (n_vis + n_tail));
        std::vector<int> v(rows);
        dviol.download(v.data(), rows);
        sync(0);
        if (slope_violations)
            for (int x : v) *slope_violations += (size_t)x;
    });
}

int kvq_grid_mse_table(const float* queries, const float* keys_exact, const uint8_t* codes, const float* alpha,
                       const float* beta, size_t samples, size_t tokens, size_t dim, int bitwidth, int word_bits,
                       const float* tau1, const float* tau2, size_t cells, double* mse, float* best_tau) {
    return guarded([&] {
        // grid_mse_table (calibrate.hpp:195-200) argument checks, then shapes (165-169)
        if (samples == 0) raise(KVQ_ERR_DOMAIN, "grid_mse_table: empty calibration set");
        if (cells == 0) raise(KVQ_ERR_DOMAIN, "grid_mse_table: empty grid");
        validate_config(bitwidth, word_bits);
        if (dim == 0 || tokens == 0) raise(KVQ_ERR_DOMAIN, "calibration sample 0 has inconsistent shapes");
        require_device();
        const size_t rb = row_bytes(dim, bitwidth, word_bits);
        DevBuf<float> dq(samples * dim), dk(samples * tokens * dim), da(samples * dim), dbt(samples * dim);
        DevBuf<uint8_t> dc(samples * tokens * rb);
        DevBuf<float> t1(cells), t2(cells), quant(samples * tokens), exact(samples * tokens),
            prob(samples * tokens);
        DevBuf<double> mse_cs(cells * samples);
        dq.upload(queries, dq.n);
        dk.upload(keys_exact, dk.n);
        dc.upload(codes, dc.n);
        da.upload(alpha, da.n);
        dbt.upload(beta, dbt.n);
        t1.upload(tau1, cells);
        t2.upload(tau2, cells);
        ck(kvqb::launch_grid_mse(dq.p, dk.p, dc.p, da.p, dbt.p, samples, tokens, dim, bitwidth, word_bits, t1.p, t2.p,
                                 cells, quant.p, exact.p, prob.p, mse_cs.p, 0),
           "grid_mse_table");
        std::vector<double> h(cells * samples);
        mse_cs.download(h.data(), h.size());
        sync(0);
        // per-cell mean in sample order; argmin with the reference's tie-break (213-228)
        size_t best = 0;
        std::vector<double> m(cells);
        for (size_t c = 0; c < cells; ++c) {
            double acc = 0.0;
            for (size_t s = 0; s < samples; ++s) acc += h[c * samples + s];
            m[c] = acc / (double)samples;
            if (c > 0 && (m[c] < m[best] || (m[c] == m[best] && (tau1[c] < tau1[best] ||
                                                                 (tau1[c] == tau1[best] && tau2[c] < tau2[best])))))
                best = c;
        }
        if (mse) std::copy(m.begin(), m.end(), mse);
        if (best_tau) {
            best_tau[0] = tau1[best];
            best_tau[1] = tau2[best];
        }
    });
}

int kvq_mse_report(const float* queries, const float* keys, size_t heads, size_t tokens, size_t dim, int bitwidth,
                   int mode, int word_bits, float tau1, float tau2, size_t bins, double* mse_quant,
                   double* mse_quant_c, float* edges, uint64_t* counts) {
    return guarded([&] {
        // mse_report argument checks in the reference's order (calibrate.hpp:302-305), then
        // compute_stats on each head (quantize.hpp:64-68)
        if (heads == 0) raise(KVQ_ERR_DOMAIN, "mse_report: no heads");
        if (bins < 1) raise(KVQ_ERR_CONFIG, "mse_report: bins must be >= 1");
        validate_config(bitwidth, word_bits);
        if (mode != KVQ_MODE_CHANNEL_WISE && mode != KVQ_MODE_GLOBAL) raise(KVQ_ERR_CONFIG, "unknown quant mode");
        if (tokens == 0 || dim == 0) raise(KVQ_ERR_DOMAIN, "compute_stats: empty matrix");
        require_device();
        const size_t rb = row_bytes(dim, bitwidth, word_bits);
        DevBuf<float> dq(heads * dim), dk(heads * tokens * dim), da(heads * dim), dbt(heads * dim);
        DevBuf<uint8_t> dc(heads * tokens * rb);
        DevBuf<float> quant(heads * tokens), exact(heads * tokens), qc(heads * tokens), de(heads * (bins + 1));
        DevBuf<unsigned long long> dcnt(heads * 3 * bins);
        DevBuf<double> mq(heads), mc(heads);
        dq.upload(queries, dq.n);
        dk.upload(keys, dk.n);
        ck(kvqb::launch_mse_report(dq.p, dk.p, heads, tokens, dim, bitwidth, mode, word_bits, tau1, tau2, bins, da.p,
                                   dbt.p, dc.p, quant.p, exact.p, qc.p, de.p, dcnt.p, mq.p, mc.p, 0),
           "mse_report");
        if (mse_quant) mq.download(mse_quant, heads);
        if (mse_quant_c) mc.download(mse_quant_c, heads);
        if (edges) de.download(edges, de.n);
        if (counts) dcnt.download(reinterpret_cast<unsigned long long*>(counts), dcnt.n);
        sync(0);
    });
}

}  // extern "C"
