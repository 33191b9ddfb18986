// capi_internal.cuh — shared internals of the C-ABI translation units (kvq_capi.cu,
// kvq_cache.cu, kvq_snapshot.cu): the error plumbing that maps onto the reference's
// exception classes, device buffers, and the hybrid cache object behind `kvq_cache*`.
#pragma once

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "kvq_capi.h"
#include "kvq_internal.cuh"

namespace kvqb::capi {

using kvqb::codes_per_row;
using kvqb::row_bytes;


using kvqb::codes_per_row;
using kvqb::row_bytes;

inline thread_local std::string g_err;
inline thread_local unsigned long long g_err_offset = 0;

struct Error {
    int code;
    std::string msg;
    unsigned long long offset = 0;  // byte offset of a FORMAT error (format_error::offset)
};

[[noreturn]] inline void raise(int code, const std::string& msg) { throw Error{code, msg}; }
[[noreturn]] inline void raise_format(const std::string& msg, unsigned long long off) {
    throw Error{KVQ_ERR_FORMAT, msg, off};
}

inline void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) raise(KVQ_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

inline void require_device() {
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
inline void validate_widths(int code_bits, int word_bits) {
    if (code_bits < 1 || word_bits < 8 || word_bits > 32 || word_bits % 8 != 0)
        raise(KVQ_ERR_CONFIG, "word bits must be 8, 16, or 32 and code bits >= 1");
    if (word_bits % code_bits != 0)
        raise(KVQ_ERR_CONFIG, "code bits " + std::to_string(code_bits) + " must divide word bits " +
                                  std::to_string(word_bits));
}

// QuantizationConfig::validate (quantize.hpp:38-43).
inline void validate_config(int bitwidth, int word_bits) {
    if (bitwidth != 1 && bitwidth != 2 && bitwidth != 4 && bitwidth != 8)
        raise(KVQ_ERR_CONFIG, "bitwidth must be 1, 2, 4, or 8");
    validate_widths(bitwidth, word_bits);
}

// Codes wider than 16 bits have no defined level count in the reference
// ((1u << 32) - 1 is UB at quantize.hpp:98); the quantizer entry points reject them.
inline void validate_quant_bits(int bits, int word_bits) {
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

inline void sync(cudaStream_t s) { ck(cudaStreamSynchronize(s), "kernel execution"); }


}  // namespace kvqb::capi

using kvqb::capi::DevBuf;

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
    // K codes in the reference layout. V codes: a tensor-core-eligible cache (d = 128, G <= 8)
    // holds them ONLY as the decode's operand layout (vx) - one resident copy; the reference
    // rows are rebuilt on demand (v_ref / read-back / snapshots). Others keep [2][...] rows.
    DevBuf<uint8_t> codes;   // [1 or 2][units][n_vis][rb]  (K, then V unless v_operand_only)
    bool v_operand_only = false;
    DevBuf<uint8_t> vt;      // token-packed V codes for the tcgen05 decode (d = 128, M = 8)
    DevBuf<uint8_t> vx;      // V codes pre-arranged as IMMA operands for the default decode
    DevBuf<uint8_t> vref;    // reference-layout V rebuilt from vx for the generic / tcgen05 paths
    DevBuf<float> stats;     // [2 (K,V)][2 (alpha,beta)][units][dim]
    DevBuf<float> vtok;      // token-wise V (KVQ_MODE_V_TOKEN_WISE): [2 (alpha,beta)][units][n_vis]
    DevBuf<float2> vtok_so;  //   and the decode's (step, alpha / step) per token [units][n_vis]
    DevBuf<float> k_tail, v_tail;  // [units][tail_cap][dim]
    DevBuf<float> lse;             // [units][group] decode log-sum-exp for the tail pass
    DevBuf<float> tail_part;       // [units][group][130] tail-pass partials (concurrent schedule)
    cudaStream_t tstream = nullptr;  // the tail pass, concurrent with the decode
    cudaEvent_t ev_tfork = nullptr, ev_tjoin = nullptr;
    DevBuf<int> tail_len;    // [2 batch + 1]: rows per request, the append overflow flag, the
                             // fused-append counters per request (self-resetting)
    DevBuf<float> d_q, d_out, d_knew, d_vnew, scratch, weights;
    DevBuf<uint8_t> tc_scratch;  // prep-kernel outputs of the tcgen05 decode path
    DevBuf<int> viol;

    uint8_t* k_codes() const { return codes.p; }
    uint8_t* v_codes() const { return codes.p && !v_operand_only ? codes.p + units * n_vis * rb : nullptr; }
    float* k_alpha() const { return stats.p; }
    float* k_beta() const { return stats.p + units * dim; }
    float* v_alpha() const { return stats.p + 2 * units * dim; }
    float* v_beta() const { return stats.p + 3 * units * dim; }
    size_t q_elems() const { return units * group * dim; }
    bool v_token_wise() const { return mode == KVQ_MODE_V_TOKEN_WISE; }
    int* overflow_flag() const { return tail_len.p ? tail_len.p + batch : nullptr; }
    int* append_counters() const { return tail_len.p ? tail_len.p + batch + 1 : nullptr; }  // fused append
    ~kvq_cache() {
        if (stream) cudaStreamDestroy(stream);
        if (side) cudaStreamDestroy(side);
        if (decoded) cudaEventDestroy(decoded);
        if (d2h) cudaStreamDestroy(d2h);
        if (tstream) cudaStreamDestroy(tstream);
        if (ev_tfork) cudaEventDestroy(ev_tfork);
        if (ev_tjoin) cudaEventDestroy(ev_tjoin);
        for (cudaEvent_t e : ev_q) cudaEventDestroy(e);
        for (cudaEvent_t e : ev_dec) cudaEventDestroy(e);
        for (cudaStream_t x : chunk_streams) cudaStreamDestroy(x);
        for (cudaEvent_t e : {ev_fork, ev_kv, ev_join})
            if (e) cudaEventDestroy(e);
        if (step_exec) cudaGraphExecDestroy(step_exec);
    }
};


namespace kvqb::capi {

// Cache internals shared by the cache and snapshot translation units (kvq_cache.cu).
void grow_tail(kvq_cache* c, size_t need);
void ensure_tail_room(kvq_cache* c, size_t extra);
void sync_tail(kvq_cache* c);
kvqb::DecodeArgs decode_args(kvq_cache* c, const float* q, float* out);
void run_decode(kvq_cache* c, const float* q, float* out, bool want_weights, bool want_viol, cudaStream_t s,
                const float* k_new = nullptr, const float* v_new = nullptr);
kvq_cache* build_common(size_t batch, size_t kv_heads, size_t group, size_t n_vis, size_t dim, int bitwidth,
                        int mode, int word_bits, float tau1, float tau2);
void ensure_vx(kvq_cache* c, cudaStream_t s);
void ensure_vt(kvq_cache* c, cudaStream_t s);
// Reference-layout V rows: the resident copy, or rebuilt from vx into c->vref (kept).
const uint8_t* v_ref(kvq_cache* c, cudaStream_t s);
// Reference-layout V rows into `tmp` when V is held only as vx (one-off read-backs).
const uint8_t* v_ref_tmp(kvq_cache* c, DevBuf<uint8_t>& tmp, cudaStream_t s);
// Store reference-layout V rows (build / load): into the cache, or packed into vx.
void store_v_rows(kvq_cache* c, const uint8_t* rows, cudaStream_t s);

}  // namespace kvqb::capi
