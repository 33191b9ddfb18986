// kvq_capi.cu — the C-ABI (include/kvq_capi.h): argument validation with the
// reference's error classes, device memory management for the hybrid cache, and
// dispatch to the K1/K2/K3 kernels. No compute happens on the host: every numeric
// result comes out of a CUDA kernel, and a missing device is a hard KVQ_ERR_CUDA.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "kvq_capi.h"
#include "kvq_internal.cuh"

namespace kvqb {
static std::atomic<unsigned long long> g_launches{0};
void note_launch(unsigned n) { g_launches += n; }
unsigned long long launch_count() { return g_launches.load(); }
}  // namespace kvqb

namespace {

using kvqb::codes_per_row;
using kvqb::row_bytes;

thread_local std::string g_err;
thread_local unsigned long long g_err_offset = 0;

struct Error {
    int code;
    std::string msg;
    unsigned long long offset = 0;  // byte offset of a FORMAT error (format_error::offset)
};

[[noreturn]] void raise(int code, const std::string& msg) { throw Error{code, msg}; }
[[noreturn]] void raise_format(const std::string& msg, unsigned long long off) {
    throw Error{KVQ_ERR_FORMAT, msg, off};
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(KVQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void require_device() {
    static int state = -1;  // -1 unknown, 0 none, 1 ok
    if (state < 0) {
        int n = 0;
        cudaError_t e = cudaGetDeviceCount(&n);
        state = (e == cudaSuccess && n > 0) ? 1 : 0;
        if (e != cudaSuccess) cudaGetLastError();
    }
    if (state != 1) raise(KVQ_ERR_CUDA, "no usable CUDA device (this library has no CPU fallback)");
}

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return KVQ_OK;
    } catch (const Error& e) {
        g_err = e.msg;
        g_err_offset = e.offset;
        return e.code;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return KVQ_ERR_CUDA;
    }
}

// bitpack.hpp:141-149 (same messages as the reference).
void validate_widths(int code_bits, int word_bits) {
    if (code_bits < 1 || word_bits < 8 || word_bits > 32 || word_bits % 8 != 0)
        raise(KVQ_ERR_CONFIG, "word bits must be 8, 16, or 32 and code bits >= 1");
    if (word_bits % code_bits != 0)
        raise(KVQ_ERR_CONFIG, "code bits " + std::to_string(code_bits) + " must divide word bits " +
                                  std::to_string(word_bits));
}

// QuantizationConfig::validate (quantize.hpp:38-43).
void validate_config(int bitwidth, int word_bits) {
    if (bitwidth != 1 && bitwidth != 2 && bitwidth != 4 && bitwidth != 8)
        raise(KVQ_ERR_CONFIG, "bitwidth must be 1, 2, 4, or 8");
    validate_widths(bitwidth, word_bits);
}

// Codes wider than 16 bits have no defined level count in the reference
// ((1u << 32) - 1 is UB at quantize.hpp:98); the quantizer entry points reject them.
void validate_quant_bits(int bits, int word_bits) {
    validate_widths(bits, word_bits);
    if (bits > 16) raise(KVQ_ERR_CONFIG, "quantizer code bits must be <= 16");
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t n = 0;
    DevBuf() = default;
    explicit DevBuf(size_t count) { alloc(count); }
    void alloc(size_t count) {
        release();
        n = count;
        if (count) ck(cudaMalloc(&p, sizeof(T) * count), "cudaMalloc");
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DevBuf() { release(); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void upload(const T* h, size_t count, cudaStream_t s = 0) {
        if (count) ck(cudaMemcpyAsync(p, h, sizeof(T) * count, cudaMemcpyHostToDevice, s), "H2D");
    }
    void download(T* h, size_t count, cudaStream_t s = 0) const {
        if (count) ck(cudaMemcpyAsync(h, p, sizeof(T) * count, cudaMemcpyDeviceToHost, s), "D2H");
    }
};

void sync(cudaStream_t s) { ck(cudaStreamSynchronize(s), "kernel execution"); }

}  // namespace

// The host buffers and cache state a captured step graph is valid for.
struct StepKey {
    const void *q = nullptr, *k = nullptr, *v = nullptr;
    void* out = nullptr;
    size_t tail_cap = 0;
    int path = -1;
    size_t chunks = 0;
    bool operator==(const StepKey& o) const {
        return q == o.q && k == o.k && v == o.v && out == o.out && tail_cap == o.tail_cap && path == o.path &&
               chunks == o.chunks;
    }
};

// ------------------------------------------------------------------------------------
struct kvq_cache {
    size_t batch = 0, kv_heads = 0, group = 0, n_vis = 0, dim = 0, units = 0;
    int bits = 8, mode = 0, word_bits = 8;
    float tau1 = 0.f, tau2 = 0.f;
    size_t rb = 0;
    size_t n_tail = 0, tail_cap = 0;
    int path = KVQ_PATH_AUTO;
    cudaStream_t stream = nullptr;
    cudaStream_t side = nullptr;       // kvq_cache_step: new K/V rows upload + append
    cudaEvent_t decoded = nullptr;     // kvq_cache_step: decode retired -> append may run
    cudaStream_t d2h = nullptr;        // kvq_cache_step (chunked): output downloads
    std::vector<cudaEvent_t> ev_q, ev_dec;  // kvq_cache_step (chunked): per-chunk hand-offs
    std::vector<cudaStream_t> chunk_streams;  // kvq_cache_step (chunked): one decode stream per chunk
    cudaEvent_t ev_fork = nullptr, ev_kv = nullptr, ev_join = nullptr;  // kvq_cache_step fork / join
    cudaGraphExec_t step_exec = nullptr;  // kvq_cache_step replay for the buffers in step_key
    StepKey step_key;
    DevBuf<uint8_t> codes;   // [2][units][n_vis][rb]  (K then V)
    DevBuf<uint8_t> vt;      // token-packed V codes for the tcgen05 decode (d = 128, M = 8)
    DevBuf<uint8_t> vx;      // V codes pre-arranged as IMMA operands for the default decode
    DevBuf<float> stats;     // [2 (K,V)][2 (alpha,beta)][units][dim]
    DevBuf<float> k_tail, v_tail;  // [units][tail_cap][dim]
    DevBuf<float> lse;             // [units][group] decode log-sum-exp for the tail pass
    DevBuf<int> tail_len;    // [batch]
    DevBuf<float> d_q, d_out, d_knew, d_vnew, scratch, weights;
    DevBuf<uint8_t> tc_scratch;  // prep-kernel outputs of the tcgen05 decode path
    DevBuf<int> viol;

    uint8_t* k_codes() const { return codes.p; }
    uint8_t* v_codes() const { return codes.p ? codes.p + units * n_vis * rb : nullptr; }
    float* k_alpha() const { return stats.p; }
    float* k_beta() const { return stats.p + units * dim; }
    float* v_alpha() const { return stats.p + 2 * units * dim; }
    float* v_beta() const { return stats.p + 3 * units * dim; }
    size_t q_elems() const { return units * group * dim; }
    ~kvq_cache() {
        if (stream) cudaStreamDestroy(stream);
        if (side) cudaStreamDestroy(side);
        if (decoded) cudaEventDestroy(decoded);
        if (d2h) cudaStreamDestroy(d2h);
        for (cudaEvent_t e : ev_q) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_dec) cudaEventDestroy(e);
        for (cudaStream_t x : chunk_streams) cudaStreamDestroy(x);
        for (cudaEvent_t e : {ev_fork, ev_kv, ev_join})
            if (e) cudaEventDestroy(e);
        if (step_exec) cudaGraphExecDestroy(step_exec);
    }
};

namespace {

void grow_tail(kvq_cache* c, size_t need) {
    if (need <= c->tail_cap) return;
    size_t cap = c->tail_cap ? c->tail_cap : 16;
    while (cap < need) cap *= 2;
    DevBuf<float> nk(c->units * cap * c->dim), nv(c->units * cap * c->dim);
    if (c->n_tail) {
        size_t w = c->n_tail * c->dim * sizeof(float);
        ck(cudaMemcpy2DAsync(nk.p, cap * c->dim * sizeof(float), c->k_tail.p,
                             c->tail_cap * c->dim * sizeof(float), w, c->units, cudaMemcpyDeviceToDevice,
                             c->stream), "tail grow");
        ck(cudaMemcpy2DAsync(nv.p, cap * c->dim * sizeof(float), c->v_tail.p,
                             c->tail_cap * c->dim * sizeof(float), w, c->units, cudaMemcpyDeviceToDevice,
                             c->stream), "tail grow");
    }
    sync(c->stream);
    std::swap(c->k_tail.p, nk.p);
    std::swap(c->k_tail.n, nk.n);
    std::swap(c->v_tail.p, nv.p);
    std::swap(c->v_tail.n, nv.n);
    c->tail_cap = cap;
    c->scratch.release();  // sized by tail_cap; rebuilt lazily
}

kvqb::DecodeArgs decode_args(kvq_cache* c, const float* q, float* out) {
    kvqb::DecodeArgs a{};
    a.k_codes = c->k_codes();
    a.v_codes = c->v_codes();
    a.v_codes_t = c->vt.p;
    a.v_codes_x = c->vx.p;
    a.k_alpha = c->k_alpha();
    a.k_beta = c->k_beta();
    a.v_alpha = c->v_alpha();
    a.v_beta = c->v_beta();
    a.k_tail = c->k_tail.p;
    a.v_tail = c->v_tail.p;
    a.tail_len = c->tail_len.p;
    a.q = q;
    a.out = out;
    a.units = c->units;
    a.kv_heads = c->kv_heads;
    a.group = c->group;
    a.dim = c->dim;
    a.n_vis = c->n_vis;
    a.tail_cap = c->tail_cap;
    a.bits = c->bits == KVQ_FULL_PRECISION_BITS ? 8 : c->bits;
    a.word_bits = c->word_bits;
    a.tau1 = c->tau1;
    a.tau2 = c->tau2;
    return a;
}

// Debug timeline: KVQ_TRACE_FILE=path dumps 256 globaltimer stamps per CTA of each
// tensor-core decode (tools/trace_decode.py reads it). Off the measured path.
template <typename F>
void traced(kvq_cache* c, kvqb::DecodeArgs& a, cudaStream_t s, F&& launch) {
    static const char* trace_file = std::getenv("KVQ_TRACE_FILE");
    if (!trace_file) {
        launch();
        return;
    }
    const size_t trace_n = c->units * 256 * 16;
    DevBuf<unsigned long long> trace(trace_n);
    ck(cudaMemsetAsync(trace.p, 0, trace_n * 8, s), "trace");
    a.trace = trace.p;
    launch();
    std::vector<unsigned long long> h(trace_n);
    trace.download(h.data(), trace_n, s);
    sync(s);
    if (FILE* f = std::fopen(trace_file, "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
    }
    a.trace = nullptr;
}

void ensure_vt(kvq_cache* c, cudaStream_t s);
void ensure_vx(kvq_cache* c, cudaStream_t s);

void run_decode(kvq_cache* c, const float* q, float* out, bool want_weights, bool want_viol,
                cudaStream_t s) {
    kvqb::DecodeArgs a = decode_args(c, q, out);
    const bool plain = !want_weights && !want_viol;
    if (plain && c->path != KVQ_PATH_GENERIC && c->path != KVQ_PATH_UMMA) {
        ensure_vx(c, s);
        a.v_codes_x = c->vx.p;
    }
    kvqb::DecodeArgs probe = a;
    probe.v_codes_t = reinterpret_cast<const uint8_t*>(1);  // shape check only
    const bool umma_ok = plain && c->dim == 128 && c->word_bits == 8 && kvqb::decode_umma_supported(probe);
    // Long fp32 tails leave the in-kernel tail of the tensor-core decode for the tail pass
    // (k2_tail.cu), which streams them at HBM rate and merges by log-sum-exp.
    if (plain && c->tail_cap > kvqb::kTcTailMax && kvqb::decode_tail_supported(a)) {
        if (c->lse.n < c->units * c->group) c->lse.alloc(c->units * c->group);
        a.tail_lse = c->lse.p;
    }
    bool tc_ok = kvqb::decode_tc_supported(a) && plain;
    // Probability-row / violation export (decode_step_detailed) is a generic-path feature:
    // an explicit tensor-core path selection applies to plain decodes only.
    if (c->path == KVQ_PATH_UMMA && !umma_ok && plain)
        raise(KVQ_ERR_CONFIG, "tcgen05 decode path needs dim 128, 8-bit words, a quantized "
                              "prefill and no weight/violation export");
    if (c->path == KVQ_PATH_TC && !tc_ok && plain)
        raise(KVQ_ERR_CONFIG, "tensor-core decode path needs dim 128, 8-bit words, a quantized "
                              "prefill and no weight/violation export");
    // AUTO prefers the mma.sync IMMA kernel: for this problem's N = G x digit planes = 16
    // it out-runs tcgen05 (a kind::i8 UTCIMMA costs ~100 cycles for any N <= 128,
    // profiles/r01_umma_rate.txt). The tcgen05 path remains selectable (KVQ_PATH_UMMA).
    if ((c->path == KVQ_PATH_UMMA || (c->path == KVQ_PATH_AUTO && !tc_ok)) && umma_ok) {
        ensure_vt(c, s);
        a.v_codes_t = c->vt.p;
        a.v_codes_x = c->vx.p;
        a.tail_lse = nullptr;
        const size_t need = kvqb::decode_tc_scratch_bytes(c->units);
        if (c->tc_scratch.n < need) c->tc_scratch.alloc(need);
        a.umma_qb = c->tc_scratch.p;
        a.tc_qconst = reinterpret_cast<float2*>(c->tc_scratch.p + c->units * 2 * 512 * sizeof(uint32_t));
        traced(c, a, s, [&] { ck(kvqb::launch_decode_umma(a, s), "decode (umma)"); });
        return;
    }
    if ((c->path == KVQ_PATH_AUTO || c->path == KVQ_PATH_TC) && tc_ok) {
        traced(c, a, s, [&] { ck(kvqb::launch_decode_tc(a, s), "decode (tc)"); });
        if (a.tail_lse) ck(kvqb::launch_decode_tail(a, true, s), "decode (tail)");
        return;
    }
    // A pure fp32 cache (build_full_precision): the tail pass is the whole decode.
    if (plain && c->n_vis == 0 && c->path != KVQ_PATH_GENERIC && kvqb::decode_tail_supported(a)) {
        ck(kvqb::launch_decode_tail(a, false, s), "decode (tail)");
        return;
    }
    size_t need = c->units * c->group * (c->n_vis + c->tail_cap);
    if (c->scratch.n < need) c->scratch.alloc(need);
    a.scratch = c->scratch.p;
    if (want_weights) {
        size_t wl = c->units * c->group * (c->n_vis + c->n_tail);
        if (c->weights.n < wl) c->weights.alloc(wl);
        a.weights = c->weights.p;
        a.weights_stride = c->n_vis + c->n_tail;
    }
    if (want_viol) {
        if (c->viol.n < c->units * c->group) c->viol.alloc(c->units * c->group);
        a.violations = c->viol.p;
    }
    ck(kvqb::launch_decode_generic(a, s), "decode (generic)");
}

kvq_cache* build_common(size_t batch, size_t kv_heads, size_t group, size_t n_vis, size_t dim,
                        int bitwidth, int mode, int word_bits, float tau1, float tau2) {
    require_device();
    const bool full = bitwidth == KVQ_FULL_PRECISION_BITS;
    if (!full) validate_config(bitwidth, word_bits);
    if (mode != KVQ_MODE_CHANNEL_WISE && mode != KVQ_MODE_GLOBAL) raise(KVQ_ERR_CONFIG, "unknown quant mode");
    // check_prefill (kvcache.hpp:224-236)
    if (batch == 0 || kv_heads == 0) raise(KVQ_ERR_DOMAIN, "cache build: need matching per-head key/value lists");
    if (group == 0) raise(KVQ_ERR_DOMAIN, "cache build: query group must be >= 1");
    if (dim == 0) raise(KVQ_ERR_DOMAIN, "cache build: head dim must be positive");
    auto* c = new kvq_cache;
    c->batch = batch;
    c->kv_heads = kv_heads;
    c->group = group;
    c->units = batch * kv_heads;
    c->dim = dim;
    c->bits = bitwidth;
    c->mode = mode;
    c->word_bits = full ? 8 : word_bits;
    c->tau1 = full ? 0.f : tau1;
    c->tau2 = full ? 0.f : tau2;
    c->n_vis = full ? 0 : n_vis;
    c->rb = row_bytes(dim, full ? 8 : bitwidth, c->word_bits);
    ck(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking), "stream");
    ck(cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&c->decoded, cudaEventDisableTiming), "event");
    c->stats.alloc(4 * c->units * dim);
    ck(cudaMemsetAsync(c->stats.p, 0, sizeof(float) * c->stats.n, c->stream), "memset");
    c->codes.alloc(2 * c->units * c->n_vis * c->rb);
    c->tail_len.alloc(batch);
    ck(cudaMemsetAsync(c->tail_len.p, 0, sizeof(int) * batch, c->stream), "memset");
    c->d_q.alloc(c->q_elems());
    c->d_out.alloc(c->q_elems());
    c->d_knew.alloc(c->units * dim);
    c->d_vnew.alloc(c->units * dim);
    grow_tail(c, full ? (n_vis > 16 ? n_vis : 16) : 16);
    return c;
}

// Quantize K and V prefill already on the device.
void quantize_prefill(kvq_cache* c, const float* dk, const float* dv, cudaStream_t s) {
    const size_t u = c->units, n = c->n_vis, d = c->dim;
    const float* srcs[2] = {dk, dv};
    for (int which = 0; which < 2; ++which) {
        uint8_t* codes = which == 0 ? c->k_codes() : c->v_codes();
        float* alpha = which == 0 ? c->k_alpha() : c->v_alpha();
        float* beta = which == 0 ? c->k_beta() : c->v_beta();
        if (kvqb::quantize_fused_supported(n, d, c->word_bits, c->mode)) {
            ck(kvqb::launch_quantize_fused(srcs[which], u, n, d, c->bits, c->mode, alpha, beta, codes, s), "quantize");
        } else {
            ck(kvqb::launch_compute_stats(srcs[which], u, n, d, c->mode, alpha, beta, s), "compute_stats");
            ck(kvqb::launch_quantize_pack(srcs[which], u, n, d, alpha, beta, c->bits, c->word_bits, codes, s),
               "quantize");
        }
    }
}

// Device layout for the tcgen05 decode: V codes re-packed along the token axis. Built on
// first use of that path (the default IMMA path reads the reference layout).
void ensure_vx(kvq_cache* c, cudaStream_t s) {
    if (c->vx.p || c->dim != 128 || c->n_vis == 0 || c->bits == KVQ_FULL_PRECISION_BITS) return;
    c->vx.alloc(kvqb::vx_bytes(c->units, c->n_vis, c->bits));
    ck(kvqb::launch_pack_vx(c->v_codes(), c->units, c->n_vis, c->bits, c->word_bits, c->vx.p, s), "pack vx");
}

void ensure_vt(kvq_cache* c, cudaStream_t s) {
    if (c->vt.p || c->dim != 128 || c->word_bits != 8 || c->n_vis == 0) return;
    c->vt.alloc(kvqb::vt_bytes(c->units, c->n_vis, c->bits));
    ck(kvqb::launch_pack_vt(c->v_codes(), c->units, c->n_vis, c->bits, c->vt.p, s), "pack vt");
}

void fill_full_precision_tail(kvq_cache* c, const float* k, const float* v, size_t n, cudaMemcpyKind kind) {
    const size_t d = c->dim;
    if (n) {
        ck(cudaMemcpy2DAsync(c->k_tail.p, c->tail_cap * d * sizeof(float), k, n * d * sizeof(float),
                             n * d * sizeof(float), c->units, kind, c->stream), "tail fill");
        ck(cudaMemcpy2DAsync(c->v_tail.p, c->tail_cap * d * sizeof(float), v, n * d * sizeof(float),
                             n * d * sizeof(float), c->units, kind, c->stream), "tail fill");
    }
    std::vector<int> lens(c->batch, (int)n);
    c->tail_len.upload(lens.data(), c->batch, c->stream);
    c->n_tail = n;
    sync(c->stream);
}

}  // namespace

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
            ck(kvqb::launch_quantize_fused(x, mats, rows, dim, bitwidth, mode, alpha, beta, codes, s), "quantize");
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

int kvq_cache_build(const float* k_vis, const float* v_vis, size_t batch, size_t kv_heads, size_t group,
                    size_t n_vis, size_t dim, int bitwidth, int mode, int word_bits, float tau1, float tau2,
                    kvq_cache** out) {
    return guarded([&] {
        *out = nullptr;
        kvq_cache* c = build_common(batch, kv_heads, group, n_vis, dim, bitwidth, mode, word_bits, tau1, tau2);
        try {
            const size_t elems = c->units * n_vis * dim;
            if (bitwidth == KVQ_FULL_PRECISION_BITS) {
                fill_full_precision_tail(c, k_vis, v_vis, n_vis, cudaMemcpyHostToDevice);
            } else if (n_vis > 0) {
                DevBuf<float> dk(elems), dv(elems);
                dk.upload(k_vis, elems, c->stream);
                dv.upload(v_vis, elems, c->stream);
                quantize_prefill(c, dk.p, dv.p, c->stream);
                sync(c->stream);
            }
            sync(c->stream);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

int kvq_cache_build_device(const float* k_vis, const float* v_vis, size_t batch, size_t kv_heads,
                           size_t group, size_t n_vis, size_t dim, int bitwidth, int mode, int word_bits,
                           float tau1, float tau2, void* stream, kvq_cache** out) {
    return guarded([&] {
        *out = nullptr;
        kvq_cache* c = build_common(batch, kv_heads, group, n_vis, dim, bitwidth, mode, word_bits, tau1, tau2);
        try {
            sync(c->stream);
            cudaStream_t s = (cudaStream_t)stream;
            if (bitwidth == KVQ_FULL_PRECISION_BITS) {
                ck(cudaStreamSynchronize(s), "sync");
                fill_full_precision_tail(c, k_vis, v_vis, n_vis, cudaMemcpyDeviceToDevice);
            } else if (n_vis > 0) {
                quantize_prefill(c, k_vis, v_vis, s);
                ck(cudaStreamSynchronize(s), "quantize");
            }
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

void kvq_cache_free(kvq_cache* c) { delete c; }

int kvq_cache_reserve_tail(kvq_cache* c, size_t rows) {
    return guarded([&] { grow_tail(c, rows); });
}

int kvq_cache_set_path(kvq_cache* c, int path) {
    return guarded([&] {
        if (path < KVQ_PATH_AUTO || path > KVQ_PATH_UMMA) raise(KVQ_ERR_CONFIG, "unknown decode path");
        c->path = path;
    });
}

int kvq_cache_append(kvq_cache* c, const float* k_new, const float* v_new) {
    return guarded([&] {
        grow_tail(c, c->n_tail + 1);
        c->d_knew.upload(k_new, c->units * c->dim, c->stream);
        c->d_vnew.upload(v_new, c->units * c->dim, c->stream);
        ck(kvqb::launch_append(c->d_knew.p, c->d_vnew.p, c->batch, c->kv_heads, c->dim, c->tail_cap,
                               c->k_tail.p, c->v_tail.p, c->tail_len.p, c->stream), "append");
        sync(c->stream);
        c->n_tail += 1;
    });
}

int kvq_cache_append_device(kvq_cache* c, const float* k_new, const float* v_new, void* stream) {
    return guarded([&] {
        if (c->n_tail + 1 > c->tail_cap) {
            ck(cudaStreamSynchronize((cudaStream_t)stream), "sync");
            grow_tail(c, c->n_tail + 1);
        }
        ck(kvqb::launch_append(k_new, v_new, c->batch, c->kv_heads, c->dim, c->tail_cap, c->k_tail.p,
                               c->v_tail.p, c->tail_len.p, (cudaStream_t)stream), "append");
        c->n_tail += 1;
    });
}

int kvq_cache_decode(kvq_cache* c, const float* queries, float* out, float* weights, size_t* slope_violations) {
    return guarded([&] {
        c->d_q.upload(queries, c->q_elems(), c->stream);
        run_decode(c, c->d_q.p, c->d_out.p, weights != nullptr, slope_violations != nullptr, c->stream);
        c->d_out.download(out, c->q_elems(), c->stream);
        std::vector<int> v;
        if (weights) {
            size_t wl = c->units * c->group * (c->n_vis + c->n_tail);
            c->weights.download(weights, wl, c->stream);
        }
        if (slope_violations) {
            v.resize(c->units * c->group);
            c->viol.download(v.data(), v.size(), c->stream);
        }
        sync(c->stream);
        if (slope_violations)
            for (int x : v) *slope_violations += (size_t)x;
    });
}

int kvq_cache_decode_device(kvq_cache* c, const float* queries, float* out, void* stream) {
    return guarded([&] { run_decode(c, queries, out, false, false, (cudaStream_t)stream); });
}

}  // extern "C"

namespace {

// Requests [b0, b1) of the cache as DecodeArgs: every per-unit array is unit-major and
// tail_len request-major, so a request range is a pointer offset.
kvqb::DecodeArgs range_args(const kvqb::DecodeArgs& a, const kvq_cache* c, size_t b0, size_t b1) {
    kvqb::DecodeArgs r = a;
    const size_t u0 = b0 * c->kv_heads, d = c->dim, G = c->group;
    r.k_codes += u0 * c->n_vis * c->rb;
    r.v_codes += u0 * c->n_vis * c->rb;
    if (r.v_codes_x) r.v_codes_x += kvqb::vx_bytes(u0, c->n_vis, c->bits);
    r.k_alpha += u0 * d;
    r.k_beta += u0 * d;
    r.v_alpha += u0 * d;
    r.v_beta += u0 * d;
    r.k_tail += u0 * c->tail_cap * d;
    r.v_tail += u0 * c->tail_cap * d;
    r.tail_len += b0;
    r.q += u0 * G * d;
    r.out += u0 * G * d;
    if (r.tail_lse) r.tail_lse += u0 * G;
    r.units = (b1 - b0) * c->kv_heads;
    r.plan_units = c->units;  // chunked results are bit-identical to the whole-batch decode
    return r;
}

// How many request chunks one host-buffer step is cut into: each chunk's query upload,
// decode and output download run on their own streams, so chunk i's decode overlaps chunk
// i+1's upload and chunk i-1's download. KVQ_STEP_CHUNKS overrides (tuning).
size_t step_chunks(const kvq_cache* c);

// The chunk count a step will actually use: chunking needs the tensor-core decode.
size_t step_chunks_for(kvq_cache* c) {
    size_t chunks = step_chunks(c);
    if (chunks <= 1 || c->path == KVQ_PATH_GENERIC || c->path == KVQ_PATH_UMMA) return 1;
    kvqb::DecodeArgs a = decode_args(c, c->d_q.p, c->d_out.p);
    ensure_vx(c, c->stream);
    a.v_codes_x = c->vx.p;
    if (c->tail_cap > kvqb::kTcTailMax && kvqb::decode_tail_supported(a)) {
        if (c->lse.n < c->units * c->group) c->lse.alloc(c->units * c->group);
        a.tail_lse = c->lse.p;
    }
    return kvqb::decode_tc_supported(a) ? chunks : 1;
}

// Streams and events of the host-buffer step, created before any graph capture.
void step_resources(kvq_cache* c, size_t chunks) {
    auto event = [](cudaEvent_t& e) {
        if (!e) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    };
    if (!c->d2h) ck(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking), "stream");
    event(c->ev_fork);
    event(c->ev_kv);
    event(c->ev_join);
    while (c->ev_q.size() < chunks) {
        cudaEvent_t e1 = nullptr, e2 = nullptr;
        cudaStream_t cs;
        event(e1);
        event(e2);
        ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream");
        c->ev_q.push_back(e1);
        c->ev_dec.push_back(e2);
        c->chunk_streams.push_back(cs);
    }
}

// One decode + append step from host buffers (kvq_main.cpp:313-321 order). Streams it
// forks from c->stream all rejoin it, so one wait on c->stream (or one graph launch)
// covers the step:
//   side    : query upload(s) ... new K/V rows upload (one copy-engine queue, queries first)
//   chunk i : decode of requests [b_i, b_{i+1}) as soon as their queries are on the device
//             (chunk decodes overlap: one chunk alone is latency-, not throughput-bound)
//   d2h     : output download of each chunk once it is decoded
//   stream  : the append, after every decode read the tail and the new rows are uploaded
void issue_step(kvq_cache* c, const float* queries, const float* k_new, const float* v_new, float* out,
                size_t chunks) {
    cudaStream_t s = c->stream, s2 = c->side, d2h = c->d2h;
    ck(cudaEventRecord(c->ev_fork, s), "event");
    ck(cudaStreamWaitEvent(s2, c->ev_fork, 0), "event");
    ck(cudaStreamWaitEvent(d2h, c->ev_fork, 0), "event");
    const size_t per_req = c->kv_heads * c->group * c->dim;
    auto bounds = [&](size_t i) { return c->batch * i / chunks; };
    for (size_t i = 0; i < chunks; ++i) {
        const size_t b0 = bounds(i), b1 = bounds(i + 1);
        ck(cudaMemcpyAsync(c->d_q.p + b0 * per_req, queries + b0 * per_req, (b1 - b0) * per_req * 4,
                           cudaMemcpyHostToDevice, s2), "H2D");
        ck(cudaEventRecord(c->ev_q[i], s2), "event");
    }
    c->d_knew.upload(k_new, c->units * c->dim, s2);
    c->d_vnew.upload(v_new, c->units * c->dim, s2);
    ck(cudaEventRecord(c->ev_kv, s2), "event");
    if (chunks == 1) {
        ck(cudaStreamWaitEvent(s, c->ev_q[0], 0), "event");
        run_decode(c, c->d_q.p, c->d_out.p, false, false, s);
        ck(cudaEventRecord(c->ev_dec[0], s), "event");
    } else {
        kvqb::DecodeArgs a = decode_args(c, c->d_q.p, c->d_out.p);
        a.v_codes_x = c->vx.p;
        if (c->tail_cap > kvqb::kTcTailMax && kvqb::decode_tail_supported(a)) a.tail_lse = c->lse.p;
        for (size_t i = 0; i < chunks; ++i) {
            cudaStream_t cs = c->chunk_streams[i];
            ck(cudaStreamWaitEvent(cs, c->ev_q[i], 0), "event");
            const kvqb::DecodeArgs r = range_args(a, c, bounds(i), bounds(i + 1));
            ck(kvqb::launch_decode_tc(r, cs), "decode (tc)");
            if (r.tail_lse) ck(kvqb::launch_decode_tail(r, true, cs), "decode (tail)");
            ck(cudaEventRecord(c->ev_dec[i], cs), "event");
            ck(cudaStreamWaitEvent(s, c->ev_dec[i], 0), "event");
        }
    }
    for (size_t i = 0; i < chunks; ++i) {
        const size_t b0 = bounds(i), b1 = bounds(i + 1);
        ck(cudaStreamWaitEvent(d2h, c->ev_dec[i], 0), "event");
        ck(cudaMemcpyAsync(out + b0 * per_req, c->d_out.p + b0 * per_req, (b1 - b0) * per_req * 4,
                           cudaMemcpyDeviceToHost, d2h), "D2H");
    }
    ck(cudaEventRecord(c->ev_join, d2h), "event");
    ck(cudaStreamWaitEvent(s, c->ev_kv, 0), "event");
    ck(kvqb::launch_append(c->d_knew.p, c->d_vnew.p, c->batch, c->kv_heads, c->dim, c->tail_cap, c->k_tail.p,
                           c->v_tail.p, c->tail_len.p, s), "append");
    ck(cudaStreamWaitEvent(s, c->ev_join, 0), "event");
}

// Records the step just issued for these host buffers as a CUDA graph (memcpy and kernel
// nodes on the same streams), replayed while the buffers, the tail capacity and the path
// stay the same. KVQ_STEP_GRAPH=0 disables (and debug tracing does).
void capture_step(kvq_cache* c, const StepKey& key) {
    static const bool off = (std::getenv("KVQ_STEP_GRAPH") && std::atoi(std::getenv("KVQ_STEP_GRAPH")) == 0) ||
                            std::getenv("KVQ_TRACE_FILE");
    if (off) return;
    if (c->step_exec) cudaGraphExecDestroy(c->step_exec);
    c->step_exec = nullptr;
    cudaGraph_t g = nullptr;
    cudaStream_t s = c->stream;
    if (cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
        cudaGetLastError();
        return;
    }
    try {
        issue_step(c, static_cast<const float*>(key.q), static_cast<const float*>(key.k),
                   static_cast<const float*>(key.v), static_cast<float*>(key.out), key.chunks);
    } catch (const Error&) {
        cudaStreamEndCapture(s, &g);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return;
    }
    if (cudaStreamEndCapture(s, &g) != cudaSuccess || !g) {
        cudaGetLastError();
        return;
    }
    cudaGraphExec_t exec = nullptr;
    if (cudaGraphInstantiate(&exec, g, 0) == cudaSuccess) {
        c->step_exec = exec;
        c->step_key = key;
    } else {
        cudaGetLastError();
    }
    cudaGraphDestroy(g);
}

size_t step_chunks(const kvq_cache* c) {
    static const char* env = std::getenv("KVQ_STEP_CHUNKS");
    // measured (profiles/r01_e2e_chunks.txt): c5 B=512 706 -> 519 us/step with 4 chunks,
    // c2 B=64 unchanged at 2 (its uploads are short next to the decode)
    size_t k = env ? (size_t)std::max(1, std::atoi(env)) : (c->batch >= 256 ? 4 : c->batch >= 32 ? 2 : 1);
    return std::min(k, c->batch);
}

}  // namespace

extern "C" {

int kvq_cache_step(kvq_cache* c, const float* queries, const float* k_new, const float* v_new, float* out) {
    return guarded([&] {
        grow_tail(c, c->n_tail + 1);
        cudaStream_t s = c->stream;
        const size_t chunks = step_chunks_for(c);
        step_resources(c, chunks);
        const StepKey key{queries, k_new, v_new, out, c->tail_cap, c->path, chunks};
        if (c->step_exec && c->step_key == key) {  // replay: one launch, one wait
            ck(cudaGraphLaunch(c->step_exec, s), "step graph");
            sync(s);
            c->n_tail += 1;
            return;
        }
        issue_step(c, queries, k_new, v_new, out, chunks);
        sync(s);
        c->n_tail += 1;
        capture_step(c, key);  // for the next call with the same buffers
    });
}

int kvq_cache_info(const kvq_cache* c, size_t info[10]) {
    info[0] = c->batch;
    info[1] = c->kv_heads;
    info[2] = c->group;
    info[3] = c->dim;
    info[4] = c->n_vis;
    info[5] = c->n_tail;
    info[6] = (size_t)c->bits;
    info[7] = (size_t)c->word_bits;
    info[8] = (size_t)c->mode;
    info[9] = c->tail_cap;
    return KVQ_OK;
}

int kvq_cache_calibration(const kvq_cache* c, float tau[2]) {
    tau[0] = c->tau1;
    tau[1] = c->tau2;
    return KVQ_OK;
}

int kvq_cache_memory(const kvq_cache* c, size_t mem[6]) {
    // HybridKVCache::memory (kvcache.hpp:123-135), summed over every unit.
    mem[0] = 2 * c->units * c->n_vis * c->rb;
    mem[1] = c->units * 4 * 4 * c->dim;
    mem[2] = mem[0] + mem[1];
    mem[3] = c->units * 2 * c->n_tail * c->dim * 4;
    mem[4] = c->units * 2 * c->n_vis * c->dim * 4;
    mem[5] = mem[2] + mem[3];
    return KVQ_OK;
}

int kvq_cache_read_segment(const kvq_cache* c, size_t unit, int which, uint8_t* bytes, float* alpha, float* beta) {
    return guarded([&] {
        if (unit >= c->units) raise(KVQ_ERR_DOMAIN, "segment index out of range");
        const size_t seg = c->n_vis * c->rb;
        const uint8_t* src = (which == 0 ? c->k_codes() : c->v_codes());
        if (seg && bytes) ck(cudaMemcpyAsync(bytes, src + unit * seg, seg, cudaMemcpyDeviceToHost, c->stream), "D2H");
        const float* a = (which == 0 ? c->k_alpha() : c->v_alpha()) + unit * c->dim;
        const float* b = (which == 0 ? c->k_beta() : c->v_beta()) + unit * c->dim;
        if (alpha) ck(cudaMemcpyAsync(alpha, a, c->dim * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (beta) ck(cudaMemcpyAsync(beta, b, c->dim * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        sync(c->stream);
    });
}

int kvq_cache_read_tail(const kvq_cache* c, size_t unit, int which, float* out) {
    return guarded([&] {
        if (unit >= c->units) raise(KVQ_ERR_DOMAIN, "tail index out of range");
        const float* src = (which == 0 ? c->k_tail.p : c->v_tail.p) + unit * c->tail_cap * c->dim;
        if (c->n_tail)
            ck(cudaMemcpyAsync(out, src, c->n_tail * c->dim * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        sync(c->stream);
    });
}

int kvq_cache_device_pointers(const kvq_cache* c, void* ptrs[9]) {
    ptrs[0] = c->k_codes();
    ptrs[1] = c->v_codes();
    ptrs[2] = c->k_alpha();
    ptrs[3] = c->k_beta();
    ptrs[4] = c->v_alpha();
    ptrs[5] = c->v_beta();
    ptrs[6] = c->k_tail.p;
    ptrs[7] = c->v_tail.p;
    ptrs[8] = c->tail_len.p;
    return KVQ_OK;
}

// ---- cache snapshots: KVQC (kvcache.hpp:137-218) over KVQP (quantize.hpp:148-230) and
// KVQT (tensor_io.hpp:11-128) records, byte-identical to HybridKVCache::save -------------
//
// Every unit of a device cache has the same shapes, so the image is a fixed-size header
// followed by `units` equal head records; payloads move with 2-D copies between the
// cache's device layout and their record slots (the copy engines do the gather), headers
// are composed on the host. `load` validates the whole image on the host first (the
// reference's checks, messages and byte offsets), then uploads it.

}  // extern "C"

namespace {

constexpr char kMagicCache[4] = {'K', 'V', 'Q', 'C'};
constexpr char kMagicPacked[4] = {'K', 'V', 'Q', 'P'};
constexpr char kMagicTensor[4] = {'K', 'V', 'Q', 'T'};
constexpr size_t kCacheHeader = 4 + 4 + 8 + 8 + 4 + 8 + 8 + 4 + 4;  // 52
constexpr size_t kSegHeader = 4 + 4 + 1 + 1 + 2 + 8;                 // 20, then words
constexpr size_t kTensorHeader = 4 + 4 + 8 + 8;                      // 24, then data

void put_le(uint8_t* p, uint64_t v, int n) {
    for (int i = 0; i < n; ++i) p[i] = (uint8_t)(v >> (8 * i));
}
void put_f32(uint8_t* p, float v) {
    uint32_t b;
    std::memcpy(&b, &v, 4);
    put_le(p, b, 4);
}

// Byte layout of one head record of cache `c` (n_txt tail rows).
struct Record {
    int seg_bits, seg_words;  // N, M stored in the segments
    size_t logical, code_bytes, seg_bytes, tensor_bytes, bytes;
    Record(const kvq_cache* c) {
        const bool full = c->bits == KVQ_FULL_PRECISION_BITS;
        seg_bits = full ? 8 : c->bits;
        seg_words = c->word_bits;
        logical = c->n_vis * codes_per_row(c->dim, seg_bits, seg_words);
        code_bytes = c->n_vis * c->rb;
        seg_bytes = kSegHeader + code_bytes + 8 + 8 * c->dim;
        tensor_bytes = kTensorHeader + 4 * c->n_tail * c->dim;
        bytes = 2 * seg_bytes + 2 * tensor_bytes;
    }
};

// Header bytes of the segment / tensor records of every unit (identical across units).
std::vector<uint8_t> record_headers(const kvq_cache* c, const Record& r) {
    std::vector<uint8_t> h(kSegHeader + 8 + kTensorHeader, 0);
    std::memcpy(h.data(), kMagicPacked, 4);
    put_le(h.data() + 4, 1, 4);
    h[8] = (uint8_t)r.seg_bits;
    h[9] = (uint8_t)r.seg_words;
    put_le(h.data() + 12, r.logical, 8);
    put_le(h.data() + kSegHeader, c->dim, 8);  // the segment's `d`, after its words
    uint8_t* t = h.data() + kSegHeader + 8;
    std::memcpy(t, kMagicTensor, 4);
    put_le(t + 4, 1, 4);
    put_le(t + 8, c->n_tail, 8);
    put_le(t + 16, c->dim, 8);
    return h;
}

// Sequential little-endian reader with the reference's truncation messages.
struct Reader {
    const uint8_t* p;
    size_t n, off = 0;
    void need(size_t k, const std::string& what) {
        if (n - off < k) raise_format("truncated while reading " + what, off);
    }
    uint64_t le(int k, const char* what) {
        need((size_t)k, what);
        uint64_t v = 0;
        for (int i = 0; i < k; ++i) v |= (uint64_t)p[off + i] << (8 * i);
        off += (size_t)k;
        return v;
    }
    float f32(const char* what) {
        uint32_t b = (uint32_t)le(4, what);
        float v;
        std::memcpy(&v, &b, 4);
        return v;
    }
    void magic(const char m[4], const std::string& name) {
        if (n - off < 4) raise_format("truncated before " + name + " magic", off);
        if (std::memcmp(p + off, m, 4) != 0) raise_format("bad " + name + " magic", off);
        off += 4;
    }
};

struct SegInfo {
    int bits, words;
    size_t logical, dim, tokens, codes_at, alpha_at;
};

// read_segment (quantize.hpp:178-223): validates and records where the payloads are.
SegInfo read_segment(Reader& r) {
    r.magic(kMagicPacked, "packed segment");
    const uint32_t version = (uint32_t)r.le(4, "version");
    if (version != 1) raise_format("unsupported segment version " + std::to_string(version), r.off - 4);
    if (r.n - r.off < 4) raise_format("truncated while reading width header", r.off);
    SegInfo s{};
    s.bits = r.p[r.off];
    s.words = r.p[r.off + 1];
    r.off += 4;
    try {
        validate_widths(s.bits, s.words);
    } catch (const Error& e) {  // garbage widths in a file are a format problem
        raise_format("stored widths invalid: " + e.msg, r.off - 4);
    }
    s.logical = (size_t)r.le(8, "logical_count");
    const size_t g = (size_t)(s.words / s.bits);
    const size_t nbytes = (s.logical + g - 1) / g * (size_t)(s.words / 8);
    if (r.n - r.off < nbytes) raise_format("truncated packed words", r.off);
    s.codes_at = r.off;
    r.off += nbytes;
    s.dim = (size_t)r.le(8, "dim");
    if ((r.n - r.off) / 8 < s.dim) {  // alpha then beta, f32 x dim each
        const size_t have = (r.n - r.off) / 4;  // whole floats present
        r.off += 4 * have;
        raise_format(std::string("truncated while reading ") + (have < s.dim ? "alpha" : "beta"), r.off);
    }
    s.alpha_at = r.off;
    r.off += 8 * s.dim;
    const size_t stride = (s.dim + g - 1) / g * g;
    if (stride == 0 ? s.logical != 0 : s.logical % stride != 0)
        raise_format("logical_count does not cover whole rows", r.off);
    s.tokens = stride == 0 ? 0 : s.logical / stride;
    return s;
}

struct TensorInfo {
    size_t rows, cols, data_at;
};

// read_tensor (tensor_io.hpp:84-107): shape, payload, finite values.
TensorInfo read_tensor(Reader& r) {
    r.magic(kMagicTensor, "tensor");
    const uint32_t version = (uint32_t)r.le(4, "version");
    if (version != 1) raise_format("unsupported tensor version " + std::to_string(version), r.off - 4);
    TensorInfo t{};
    t.rows = (size_t)r.le(8, "rows");
    t.cols = (size_t)r.le(8, "cols");
    const size_t count = t.rows * t.cols;
    if (t.cols && count / t.cols != t.rows) raise_format("truncated while reading tensor data", r.off);
    if ((r.n - r.off) / 4 < count) {
        r.off += (r.n - r.off) / 4 * 4;
        raise_format("truncated while reading tensor data", r.off);
    }
    t.data_at = r.off;
    for (size_t i = 0; i < count; ++i) {
        uint32_t b;
        std::memcpy(&b, r.p + r.off + 4 * i, 4);
        if ((b & 0x7f800000u) == 0x7f800000u) {
            r.off += 4 * count;
            raise_format("tensor contains non-finite values", r.off);
        }
    }
    r.off += 4 * count;
    return t;
}

}  // namespace

extern "C" {

int kvq_cache_image_bytes(const kvq_cache* c, size_t* bytes) {
    return guarded([&] { *bytes = kCacheHeader + c->units * Record(c).bytes; });
}

int kvq_cache_save_image(const kvq_cache* c, void* image, size_t capacity, int image_on_device, void* stream) {
    return guarded([&] {
        const Record r(c);
        const size_t total = kCacheHeader + c->units * r.bytes;
        if (capacity < total) raise(KVQ_ERR_DOMAIN, "cache save: image buffer too small");
        require_device();
        cudaStream_t s = stream ? (cudaStream_t)stream : c->stream;
        uint8_t* img = static_cast<uint8_t*>(image);
        // manifest (kvcache.hpp:137-146)
        uint8_t head[kCacheHeader];
        std::memcpy(head, kMagicCache, 4);
        put_le(head + 4, 1, 4);
        put_le(head + 8, c->units, 8);
        put_le(head + 16, c->dim, 8);
        put_le(head + 24, (uint64_t)c->bits, 4);
        put_le(head + 28, c->n_vis, 8);
        put_le(head + 36, c->n_tail, 8);
        put_f32(head + 44, c->tau1);
        put_f32(head + 48, c->tau2);
        const std::vector<uint8_t> hdr = record_headers(c, r);
        // per-unit header pieces: seg header x2, dim x2, tensor header x2 (offsets in a record)
        const size_t seg_at[2] = {0, r.seg_bytes};
        const size_t ten_at[2] = {2 * r.seg_bytes, 2 * r.seg_bytes + r.tensor_bytes};
        const size_t d = c->dim, U = c->units, pitch = r.bytes;
        uint8_t* rec0 = img + kCacheHeader;
        const cudaMemcpyKind to = image_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
        std::vector<uint8_t> rep;  // headers replicated per unit (device images: one H2D each)
        auto put_headers = [&](size_t at, const uint8_t* src, size_t len) {
            if (!image_on_device) {
                for (size_t u = 0; u < U; ++u) std::memcpy(rec0 + u * pitch + at, src, len);
                return;
            }
            rep.resize(U * len);
            for (size_t u = 0; u < U; ++u) std::memcpy(rep.data() + u * len, src, len);
            ck(cudaMemcpy2DAsync(rec0 + at, pitch, rep.data(), len, len, U, cudaMemcpyHostToDevice, s), "save");
            sync(s);  // `rep` is reused
        };
        if (image_on_device) {
            ck(cudaMemcpyAsync(img, head, kCacheHeader, cudaMemcpyHostToDevice, s), "save");
            sync(s);
        } else {
            std::memcpy(img, head, kCacheHeader);
        }
        for (int w = 0; w < 2; ++w) {
            put_headers(seg_at[w], hdr.data(), kSegHeader);
            put_headers(seg_at[w] + kSegHeader + r.code_bytes, hdr.data() + kSegHeader, 8);
            put_headers(ten_at[w], hdr.data() + kSegHeader + 8, kTensorHeader);
            const uint8_t* codes = w == 0 ? c->k_codes() : c->v_codes();
            if (r.code_bytes)
                ck(cudaMemcpy2DAsync(rec0 + seg_at[w] + kSegHeader, pitch, codes, r.code_bytes, r.code_bytes, U, to, s),
                   "save");
            const float* alpha = w == 0 ? c->k_alpha() : c->v_alpha();
            const float* beta = w == 0 ? c->k_beta() : c->v_beta();
            const size_t st = seg_at[w] + kSegHeader + r.code_bytes + 8;
            ck(cudaMemcpy2DAsync(rec0 + st, pitch, alpha, 4 * d, 4 * d, U, to, s), "save");
            ck(cudaMemcpy2DAsync(rec0 + st + 4 * d, pitch, beta, 4 * d, 4 * d, U, to, s), "save");
            const float* tail = w == 0 ? c->k_tail.p : c->v_tail.p;
            if (c->n_tail)
                ck(cudaMemcpy2DAsync(rec0 + ten_at[w] + kTensorHeader, pitch, tail, 4 * c->tail_cap * d,
                                     4 * c->n_tail * d, U, to, s),
                   "save");
        }
        sync(s);
    });
}

int kvq_cache_load_image(const void* image, size_t bytes, size_t batch, size_t group, size_t* consumed,
                         kvq_cache** out) {
    return guarded([&] {
        *out = nullptr;
        Reader r{static_cast<const uint8_t*>(image), bytes};
        // HybridKVCache::load (kvcache.hpp:163-211)
        r.magic(kMagicCache, "cache");
        const uint32_t version = (uint32_t)r.le(4, "version");
        if (version != 1) raise_format("unsupported cache version " + std::to_string(version), r.off - 4);
        const size_t heads = (size_t)r.le(8, "heads");
        const size_t dim = (size_t)r.le(8, "dim");
        const int bitwidth = (int)(uint32_t)r.le(4, "bitwidth");
        const size_t n_vis = (size_t)r.le(8, "vis tokens");
        const size_t n_txt = (size_t)r.le(8, "tail tokens");
        const float tau1 = r.f32("tau1"), tau2 = r.f32("tau2");
        if (bitwidth != KVQ_FULL_PRECISION_BITS && bitwidth != 1 && bitwidth != 2 && bitwidth != 4 && bitwidth != 8)
            raise_format("invalid cache bitwidth " + std::to_string(bitwidth), r.off);
        std::vector<SegInfo> segs;
        std::vector<TensorInfo> tails;
        for (size_t h = 0; h < heads; ++h) {
            SegInfo k = read_segment(r), v = read_segment(r);
            TensorInfo kt = read_tensor(r), vt = read_tensor(r);
            const char* bad = nullptr;
            if (k.dim != dim || v.dim != dim) bad = "segment dim";
            else if (k.tokens != n_vis || v.tokens != n_vis) bad = "segment token count";
            else if (kt.cols != dim || vt.cols != dim) bad = "tail cols";
            else if (kt.rows != n_txt || vt.rows != n_txt) bad = "tail token count";
            else if (n_vis > 0 && (k.bits != bitwidth || v.bits != bitwidth)) bad = "segment bitwidth";
            if (bad)
                raise_format("cache head " + std::to_string(h) + " does not match manifest: " + std::string(bad), r.off);
            segs.push_back(k);
            segs.push_back(v);
            tails.push_back(kt);
            tails.push_back(vt);
        }
        // What the reference accepts but one device cache cannot represent.
        if (heads == 0) raise(KVQ_ERR_DOMAIN, "cache load: a device cache needs at least one head");
        if (batch == 0 || heads % batch) raise(KVQ_ERR_DOMAIN, "cache load: heads not divisible by batch");
        const int words = segs[0].words;
        for (const SegInfo& sg : segs)
            if (sg.words != words || (n_vis > 0 && sg.bits != segs[0].bits))
                raise_format("cache load: mixed pack widths across heads are not supported by the device cache", 0);
        if (bitwidth == KVQ_FULL_PRECISION_BITS && n_vis > 0)
            raise_format("cache load: a full-precision cache cannot hold a packed segment", 0);
        if (consumed) *consumed = r.off;
        kvq_cache* c = build_common(batch, heads / batch, group, n_vis, dim, bitwidth, KVQ_MODE_CHANNEL_WISE,
                                    bitwidth == KVQ_FULL_PRECISION_BITS ? 8 : words, tau1, tau2);
        try {
            grow_tail(c, n_txt);
            const uint8_t* img = r.p;
            const size_t U = c->units;
            // records are equal-sized, so each payload is one strided copy
            const size_t pitch = heads > 1 ? segs[2].codes_at - segs[0].codes_at : 0;
            const size_t rb_bytes = n_vis * c->rb;
            for (int w = 0; w < 2; ++w) {
                const SegInfo& s0 = segs[w];
                uint8_t* codes = w == 0 ? c->k_codes() : c->v_codes();
                if (rb_bytes)
                    ck(cudaMemcpy2DAsync(codes, rb_bytes, img + s0.codes_at, pitch ? pitch : rb_bytes, rb_bytes, U,
                                         cudaMemcpyHostToDevice, c->stream), "load");
                float* alpha = w == 0 ? c->k_alpha() : c->v_alpha();
                float* beta = w == 0 ? c->k_beta() : c->v_beta();
                ck(cudaMemcpy2DAsync(alpha, 4 * dim, img + s0.alpha_at, pitch ? pitch : 4 * dim, 4 * dim, U,
                                     cudaMemcpyHostToDevice, c->stream), "load");
                ck(cudaMemcpy2DAsync(beta, 4 * dim, img + s0.alpha_at + 4 * dim, pitch ? pitch : 4 * dim, 4 * dim, U,
                                     cudaMemcpyHostToDevice, c->stream), "load");
                float* tail = w == 0 ? c->k_tail.p : c->v_tail.p;
                if (n_txt)
                    ck(cudaMemcpy2DAsync(tail, 4 * c->tail_cap * dim, img + tails[w].data_at,
                                         pitch ? pitch : 4 * n_txt * dim, 4 * n_txt * dim, U, cudaMemcpyHostToDevice,
                                         c->stream), "load");
            }
            std::vector<int> lens(c->batch, (int)n_txt);
            c->tail_len.upload(lens.data(), c->batch, c->stream);
            c->n_tail = n_txt;
            sync(c->stream);
        } catch (...) {
            delete c;
            throw;
        }
        *out = c;
    });
}

}  // extern "C"
