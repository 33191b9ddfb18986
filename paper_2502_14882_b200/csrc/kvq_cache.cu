// kvq_cache.cu — the hybrid cache behind `kvq_cache*` (kvcache.hpp:43-319): build
// (K1), decode path selection and launch (K2 + the tail pass), append (K3), the
// pipelined host-buffer step, accessors.
#include <chrono>

#include "capi_internal.cuh"

namespace kvqb::capi {


// The host tail counter from the device (after any stream / graph work on the cache):
// appends issued on user streams or replayed from captured graphs advance tail_len on the
// device only. A set overflow flag means appends were dropped at a full tail (k3_append.cu):
// reported once as a domain_error.
void sync_tail(kvq_cache* c) {
    if (!c->tail_len.p) return;
    ck(cudaDeviceSynchronize(), "kernel execution");
    std::vector<int> h(c->batch + 1);
    ck(cudaMemcpy(h.data(), c->tail_len.p, sizeof(int) * (c->batch + 1), cudaMemcpyDeviceToHost), "D2H");
    c->n_tail = (size_t)h[0];  // every request holds the same number of tail rows
    if (h[c->batch]) {
        ck(cudaMemset(c->overflow_flag(), 0, sizeof(int)), "memset");
        raise(KVQ_ERR_DOMAIN, "append: fp32 tail full (tail_cap rows); appends issued past it on the device "
                              "(e.g. a captured decode + append graph replayed beyond reserve_tail) were dropped");
    }
}

// Room for `extra` more tail rows. The host counter runs ahead of the device after graph
// captures (a captured append counts, runs later or never) and behind it after replays, so
// a shortfall is first checked against the device's own count (sync_tail) before the tail
// is reallocated - a spurious growth would change tail_cap (the host-step graph key, and
// past 64 rows the decode path).
void ensure_tail_room(kvq_cache* c, size_t extra) {
    if (c->n_tail + extra <= c->tail_cap) return;
    sync_tail(c);
    if (c->n_tail + extra <= c->tail_cap) return;
    grow_tail(c, c->n_tail + extra);
}

void grow_tail(kvq_cache* c, size_t need) {
    if (need <= c->tail_cap) return;
    sync_tail(c);  // rows appended on the device only must move too
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
    a.v_alpha = c->v_token_wise() ? c->vtok.p : c->v_alpha();
    a.v_beta = c->v_token_wise() ? c->vtok.p + c->units * c->n_vis : c->v_beta();
    a.v_token_wise = c->v_token_wise() ? 1 : 0;
    a.v_tok_so = c->vtok_so.p;
    a.k_tail = c->k_tail.p;
    a.v_tail = c->v_tail.p;
    a.tail_len = c->tail_len.p;
    a.append_cnt = c->append_counters();
    a.overflow = c->overflow_flag();
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
// tensor-core decode (tools/trace_decode.py reads it). KVQ_TRACE_CHAIN=k keeps one buffer
// for k consecutive decodes (slot i = call i, no synchronisation in between) and dumps it
// after the k-th, so back-to-back launches can be compared. Off the measured path.
template <typename F>
void traced(kvq_cache* c, kvqb::DecodeArgs& a, cudaStream_t s, F&& launch) {
    static const char* trace_file = std::getenv("KVQ_TRACE_FILE");
    if (!trace_file) {
        launch();
        return;
    }
    static const int chain = std::getenv("KVQ_TRACE_CHAIN") ? std::max(1, std::atoi(std::getenv("KVQ_TRACE_CHAIN"))) : 1;
    static int call = 0;
    static DevBuf<unsigned long long>* buf = nullptr;
    const size_t trace_n = c->units * 256 * 16;
    if (call == 0) {
        buf = new DevBuf<unsigned long long>(trace_n * chain);
        ck(cudaMemsetAsync(buf->p, 0, trace_n * chain * 8, s), "trace");
    }
    a.trace = buf->p + trace_n * call;
    launch();
    a.trace = nullptr;
    if (++call < chain) return;
    call = 0;
    std::vector<unsigned long long> h(trace_n * chain);
    buf->download(h.data(), h.size(), s);
    sync(s);
    delete buf;
    buf = nullptr;
    if (FILE* f = std::fopen(trace_file, "wb")) {
        std::fwrite(h.data(), 8, h.size(), f);
        std::fclose(f);
    }
}

void ensure_vt(kvq_cache* c, cudaStream_t s);
void ensure_vx(kvq_cache* c, cudaStream_t s);

// Long tails: the tail pass chained behind the decode (programmatic dependent launch) is
// the default; KVQ_TAIL_CONCURRENT=1 runs it on its own stream beside the decode with a
// separate merge - measured 3-4 us slower per step (the decode's CTAs already fill the SMs,
// profiles/r01_tail_concurrent.txt), kept as an option.
static bool tail_concurrent() {
    static const char* env = std::getenv("KVQ_TAIL_CONCURRENT");
    return env ? std::atoi(env) != 0 : false;
}

// Step = decode + append as ONE kernel when the tensor-core decode owns the tail in-kernel
// (one dependency hop per step instead of two); KVQ_FUSED_APPEND=0 issues the append
// kernel behind the decode instead (same results).
static bool fused_append() {
    static const char* env = std::getenv("KVQ_FUSED_APPEND");
    return env ? std::atoi(env) != 0 : true;
}

// The tensor-core decode a plain decode of this cache runs: KVQ_PATH_TC (the IMMA kernel,
// k2_decode_tc.cu), or -1 (the shape needs another path). Builds the V operand layout it
// reads (vx) on first use. (Round 2 measured three alternative schedules of the same
// kernel - channel-split 8-warp CTAs, persistent warp-specialized, persistent with dynamic
// chunk queues - all slower at every BASELINE shape: profiles/r02_decode_variants.md.)
int pick_tensor_decode(kvq_cache* c, kvqb::DecodeArgs& a, cudaStream_t s) {
    if (c->path == KVQ_PATH_AUTO || c->path == KVQ_PATH_TC) {
        kvqb::DecodeArgs probe = a;
        probe.v_codes_x = reinterpret_cast<const uint8_t*>(1);  // shape check only
        if (kvqb::decode_tc_supported(probe)) {
            ensure_vx(c, s);
            a.v_codes_x = c->vx.p;
            return KVQ_PATH_TC;
        }
    }
    return -1;
}

void launch_tensor_decode(int kind, const kvqb::DecodeArgs& a, cudaStream_t s) {
    (void)kind;
    ck(kvqb::launch_decode_tc(a, s), "decode (tc)");
}

// k_new / v_new (device, nullable): the step's append, fused into the tensor-core decode
// when it owns the fp32 tail in-kernel, else issued as the append kernel right behind.
void run_decode(kvq_cache* c, const float* q, float* out, bool want_weights, bool want_viol,
                cudaStream_t s, const float* k_new, const float* v_new) {
    kvqb::DecodeArgs a = decode_args(c, q, out);
    bool appended = false;
    auto append_rest = [&] {
        if (k_new && !appended)
            ck(kvqb::launch_append(k_new, v_new, c->batch, c->kv_heads, c->dim, c->tail_cap, c->k_tail.p,
                                   c->v_tail.p, c->tail_len.p, c->overflow_flag(), s), "append");
    };
    const bool plain = !want_weights && !want_viol;
    kvqb::DecodeArgs probe = a;
    probe.v_codes_t = reinterpret_cast<const uint8_t*>(1);  // shape check only
    const bool umma_ok = plain && c->dim == 128 && c->word_bits == 8 && kvqb::decode_umma_supported(probe);
    // Long fp32 tails leave the in-kernel tail of the tensor-core decode for the tail pass
    // (k2_tail.cu), which streams them at HBM rate and merges by log-sum-exp.
    if (plain && c->tail_cap > kvqb::kTcTailMax && kvqb::decode_tail_supported(a)) {
        if (c->lse.n < c->units * c->group) c->lse.alloc(c->units * c->group);
        if (c->tail_part.n < c->units * c->group * 130) c->tail_part.alloc(c->units * c->group * 130);
        a.tail_lse = c->lse.p;
    }
    const bool generic_only = c->path == KVQ_PATH_GENERIC || c->path == KVQ_PATH_UMMA || c->path == KVQ_PATH_DEQUANT;
    if (c->v_token_wise() && (!plain || generic_only))
        raise(KVQ_ERR_CONFIG, "token-wise V decodes on the tensor-core path only (no probability / violation "
                              "export, no generic / tcgen05 / dequant path)");
    const int tc_kind = plain && !generic_only ? pick_tensor_decode(c, a, s) : -1;
    if (c->v_token_wise() && tc_kind < 0)
        raise(KVQ_ERR_CONFIG, "token-wise V: this shape has no tensor-core decode");
    a.dequant_dot = c->path == KVQ_PATH_DEQUANT ? 1 : 0;
    // Probability-row / violation export (decode_step_detailed) is a generic-path feature:
    // an explicit tensor-core path selection applies to plain decodes only.
    if (c->path == KVQ_PATH_UMMA && !umma_ok && plain)
        raise(KVQ_ERR_CONFIG, "tcgen05 decode path needs dim 128, 8-bit words, a quantized "
                              "prefill and no weight/violation export");
    if (c->path == KVQ_PATH_TC && tc_kind < 0 && plain)
        raise(KVQ_ERR_CONFIG, "tensor-core decode path needs dim 128, 8-bit words, a quantized "
                              "prefill and no weight/violation export");
    // AUTO prefers the mma.sync IMMA kernels: for this problem's N = G x digit planes = 16 a
    // tcgen05 MMA costs 35-47 cycles (profiles/r02_umma_rate2.txt) on the same tensor
    // datapath (r02_mma_mix.txt). The tcgen05 path remains selectable (KVQ_PATH_UMMA).
    if ((c->path == KVQ_PATH_UMMA || (c->path == KVQ_PATH_AUTO && tc_kind < 0)) && umma_ok) {
        ensure_vx(c, s);
        ensure_vt(c, s);
        a.v_codes_t = c->vt.p;
        a.v_codes_x = c->vx.p;
        a.tail_lse = nullptr;
        const size_t need = kvqb::decode_tc_scratch_bytes(c->units);
        if (c->tc_scratch.n < need) c->tc_scratch.alloc(need);
        a.umma_qb = c->tc_scratch.p;
        a.tc_qconst = reinterpret_cast<float2*>(c->tc_scratch.p + c->units * 2 * 512 * sizeof(uint32_t));
        traced(c, a, s, [&] { ck(kvqb::launch_decode_umma(a, s), "decode (umma)"); });
        append_rest();
        return;
    }
    if (tc_kind >= 0) {
        if (a.tail_lse && tail_concurrent()) {
            // the HBM-bound tail pass runs beside the issue-bound decode (its own stream,
            // partials to scratch), then one merge - instead of queueing behind it
            ck(cudaEventRecord(c->ev_tfork, s), "event");
            ck(cudaStreamWaitEvent(c->tstream, c->ev_tfork, 0), "event");
            ck(kvqb::launch_decode_tail_partials(a, c->tail_part.p, c->tstream), "decode (tail)");
            ck(cudaEventRecord(c->ev_tjoin, c->tstream), "event");
            traced(c, a, s, [&] { launch_tensor_decode(tc_kind, a, s); });
            ck(cudaStreamWaitEvent(s, c->ev_tjoin, 0), "event");
            ck(kvqb::launch_tail_merge(a, c->tail_part.p, s), "decode (tail merge)");
            append_rest();
            return;
        }
        if (k_new && !a.tail_lse && fused_append()) {  // in-kernel tail: the decode appends
            a.k_new = k_new, a.v_new = v_new;
            appended = true;
        }
        traced(c, a, s, [&] { launch_tensor_decode(tc_kind, a, s); });
        if (a.tail_lse) ck(kvqb::launch_decode_tail(a, true, s), "decode (tail)");
        append_rest();
        return;
    }
    // A pure fp32 cache (build_full_precision): the tail pass is the whole decode.
    if (plain && c->n_vis == 0 && c->path != KVQ_PATH_GENERIC && c->path != KVQ_PATH_DEQUANT &&
        kvqb::decode_tail_supported(a)) {
        ck(kvqb::launch_decode_tail(a, false, s), "decode (tail)");
        append_rest();
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
    a.v_codes = v_ref(c, s);
    ck(kvqb::launch_decode_generic(a, s), "decode (generic)");
    append_rest();
}

kvq_cache* build_common(size_t batch, size_t kv_heads, size_t group, size_t n_vis, size_t dim,
                        int bitwidth, int mode, int word_bits, float tau1, float tau2) {
    require_device();
    const bool full = bitwidth == KVQ_FULL_PRECISION_BITS;
    if (!full) validate_config(bitwidth, word_bits);
    if (mode != KVQ_MODE_CHANNEL_WISE && mode != KVQ_MODE_GLOBAL && mode != KVQ_MODE_V_TOKEN_WISE)
        raise(KVQ_ERR_CONFIG, "unknown quant mode");
    if (mode == KVQ_MODE_V_TOKEN_WISE && (full || dim != 128 || n_vis == 0 || group > 8 || std::getenv("KVQ_KEEP_V_ROWS")))
        raise(KVQ_ERR_CONFIG, "token-wise V needs head dim 128, a quantized prefill and query groups <= 8 "
                              "(tensor-core decode)");
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
    ck(cudaStreamCreateWithFlags(&c->tstream, cudaStreamNonBlocking), "stream");
    ck(cudaEventCreateWithFlags(&c->ev_tfork, cudaEventDisableTiming), "event");
    ck(cudaEventCreateWithFlags(&c->ev_tjoin, cudaEventDisableTiming), "event");
    c->stats.alloc(4 * c->units * dim);
    ck(cudaMemsetAsync(c->stats.p, 0, sizeof(float) * c->stats.n, c->stream), "memset");
    // one resident V copy: eligible caches keep V only in the tensor-core operand layout
    static const bool keep_rows = std::getenv("KVQ_KEEP_V_ROWS") != nullptr;  // (debug)
    c->v_operand_only = !full && dim == 128 && c->n_vis > 0 && group <= 8 && !keep_rows;
    c->codes.alloc((c->v_operand_only ? 1 : 2) * c->units * c->n_vis * c->rb);
    if (c->v_operand_only) c->vx.alloc(kvqb::vx_bytes(c->units, c->n_vis, c->bits));
    if (c->v_token_wise()) c->vtok.alloc(2 * c->units * c->n_vis), c->vtok_so.alloc(c->units * c->n_vis);
    c->tail_len.alloc(2 * batch + 1);  // + the append overflow flag + fused-append counters
    ck(cudaMemsetAsync(c->tail_len.p, 0, sizeof(int) * (2 * batch + 1), c->stream), "memset");
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
    DevBuf<uint8_t> vrows;  // V rows staged for the operand layout (v_operand_only)
    if (c->v_operand_only) vrows.alloc(u * n * c->rb);
    for (int which = 0; which < 2; ++which) {
        uint8_t* codes = which == 0 ? c->k_codes() : (c->v_operand_only ? vrows.p : c->v_codes());
        float* alpha = which == 0 ? c->k_alpha() : c->v_alpha();
        float* beta = which == 0 ? c->k_beta() : c->v_beta();
        if (which == 1 && c->v_token_wise()) {  // opt-in: V stats per token (one pass)
            ck(kvqb::launch_quantize_tokenwise(srcs[1], u, n, c->bits, c->word_bits, c->vtok.p, c->vtok.p + u * n,
                                               c->vtok_so.p, codes, s),
               "quantize (token-wise V)");
            continue;
        }
        const int mode = c->v_token_wise() ? KVQ_MODE_CHANNEL_WISE : c->mode;  // K stays channel-wise
        if (kvqb::quantize_fused_supported(n, d, c->word_bits, mode)) {
            ck(kvqb::launch_quantize_fused(srcs[which], u, n, d, c->bits, c->word_bits, mode, alpha, beta, codes, s),
               "quantize");
        } else {
            ck(kvqb::launch_compute_stats(srcs[which], u, n, d, mode, alpha, beta, s), "compute_stats");
            ck(kvqb::launch_quantize_pack(srcs[which], u, n, d, alpha, beta, c->bits, c->word_bits, codes, s),
               "quantize");
        }
    }
    if (c->v_operand_only) {
        store_v_rows(c, vrows.p, s);
        sync(s);  // the staged rows are released on return
    }
}

// V operand layout of the IMMA decode (vx). An eligible cache built it at build / load time
// and holds V only there; a cache that keeps reference rows (KVQ_KEEP_V_ROWS) builds it on
// first use.
void ensure_vx(kvq_cache* c, cudaStream_t s) {
    if (c->v_operand_only || c->vx.p || c->dim != 128 || c->n_vis == 0 || c->bits == KVQ_FULL_PRECISION_BITS) return;
    c->vx.alloc(kvqb::vx_bytes(c->units, c->n_vis, c->bits));
    ck(kvqb::launch_pack_vx(c->v_codes(), c->units, c->n_vis, c->bits, c->word_bits, c->vx.p, s), "pack vx");
}

void store_v_rows(kvq_cache* c, const uint8_t* rows, cudaStream_t s) {
    if (c->n_vis == 0) return;
    if (c->v_operand_only)
        ck(kvqb::launch_pack_vx(rows, c->units, c->n_vis, c->bits, c->word_bits, c->vx.p, s), "pack vx");
    else if (rows != c->v_codes())
        ck(cudaMemcpyAsync(c->v_codes(), rows, c->units * c->n_vis * c->rb, cudaMemcpyDeviceToDevice, s), "V rows");
}

const uint8_t* v_ref_tmp(kvq_cache* c, DevBuf<uint8_t>& tmp, cudaStream_t s) {
    if (!c->v_operand_only) return c->v_codes();
    if (c->vref.p) return c->vref.p;
    tmp.alloc(c->units * c->n_vis * c->rb);
    ck(kvqb::launch_unpack_vx(c->vx.p, c->units, c->n_vis, c->bits, c->word_bits, tmp.p, s), "unpack vx");
    return tmp.p;
}

const uint8_t* v_ref(kvq_cache* c, cudaStream_t s) {
    if (!c->v_operand_only) return c->v_codes();
    if (!c->vref.p) {
        c->vref.alloc(c->units * c->n_vis * c->rb);
        ck(kvqb::launch_unpack_vx(c->vx.p, c->units, c->n_vis, c->bits, c->word_bits, c->vref.p, s), "unpack vx");
    }
    return c->vref.p;
}

void ensure_vt(kvq_cache* c, cudaStream_t s) {
    if (c->vt.p || c->dim != 128 || c->word_bits != 8 || c->n_vis == 0) return;
    c->vt.alloc(kvqb::vt_bytes(c->units, c->n_vis, c->bits));
    ck(kvqb::launch_pack_vt(v_ref(c, s), c->units, c->n_vis, c->bits, c->vt.p, s), "pack vt");
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


}  // namespace kvqb::capi

using namespace kvqb::capi;

namespace {


// Requests [b0, b1) of the cache as DecodeArgs: every per-unit array is unit-major and
// tail_len request-major, so a request range is a pointer offset.
kvqb::DecodeArgs range_args(const kvqb::DecodeArgs& a, const kvq_cache* c, size_t b0, size_t b1) {
    kvqb::DecodeArgs r = a;
    const size_t u0 = b0 * c->kv_heads, d = c->dim, G = c->group;
    r.k_codes += u0 * c->n_vis * c->rb;
    if (r.v_codes) r.v_codes += u0 * c->n_vis * c->rb;
    if (r.v_codes_x) r.v_codes_x += kvqb::vx_bytes(u0, c->n_vis, c->bits);
    r.k_alpha += u0 * d;
    r.k_beta += u0 * d;
    const size_t vs = r.v_token_wise ? c->n_vis : d;  // V stats per unit: per channel or per token
    r.v_alpha += u0 * vs;
    r.v_beta += u0 * vs;
    if (r.v_tok_so) r.v_tok_so += u0 * c->n_vis;
    r.k_tail += u0 * c->tail_cap * d;
    r.v_tail += u0 * c->tail_cap * d;
    r.tail_len += b0;
    if (r.append_cnt) r.append_cnt += b0;
    if (r.k_new) r.k_new += u0 * d, r.v_new += u0 * d;
    r.q += u0 * G * d;
    r.out += u0 * G * d;
    if (r.tail_lse) r.tail_lse += u0 * G;
    r.units = (b1 - b0) * c->kv_heads;
    r.plan_units = c->units;  // chunked results are bit-identical to the whole-batch decode
    r.unit_base = u0;
    return r;
}

// How many request chunks one host-buffer step is cut into: each chunk's query upload,
// decode and output download run on their own streams, so chunk i's decode overlaps chunk
// i+1's upload and chunk i-1's download. KVQ_STEP_CHUNKS overrides (tuning).
size_t step_chunks(const kvq_cache* c);

// The chunk count a step will actually use: chunking needs the tensor-core decode.
size_t step_chunks_for(kvq_cache* c) {
    size_t chunks = step_chunks(c);
    if (chunks <= 1 || c->path == KVQ_PATH_GENERIC || c->path == KVQ_PATH_UMMA || c->path == KVQ_PATH_DEQUANT)
        return 1;
    kvqb::DecodeArgs a = decode_args(c, c->d_q.p, c->d_out.p);
    if (c->tail_cap > kvqb::kTcTailMax && kvqb::decode_tail_supported(a)) {
        if (c->lse.n < c->units * c->group) c->lse.alloc(c->units * c->group);
        a.tail_lse = c->lse.p;
    }
    return pick_tensor_decode(c, a, c->stream) >= 0 ? chunks : 1;
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
    // (Tried: the decode writing `out` straight into pinned host memory, and reading the
    // queries from it - zero-copy, one chunk: C2 e2e 619 k -> 589 k / 386 k tok/s, C5 B=512
    // 1.39 M -> 1.18 M; the staged, chunked copies stay.)
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
        if (c->tail_cap > kvqb::kTcTailMax && kvqb::decode_tail_supported(a)) a.tail_lse = c->lse.p;
        const int kind = pick_tensor_decode(c, a, s);
        for (size_t i = 0; i < chunks; ++i) {
            cudaStream_t cs = c->chunk_streams[i];
            ck(cudaStreamWaitEvent(cs, c->ev_q[i], 0), "event");
            const kvqb::DecodeArgs r = range_args(a, c, bounds(i), bounds(i + 1));
            launch_tensor_decode(kind, r, cs);
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
                           c->v_tail.p, c->tail_len.p, c->overflow_flag(), s), "append");
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
    // measured (profiles/r02_e2e_chunks.txt, 1/2/3/4/8 chunks per config): C5 B=512 best at 4,
    // C2 / C3 at 2, long rows (C4, 32 k tokens, B=16) at 3 (174 -> 163 us per step)
    size_t k = env ? (size_t)std::max(1, std::atoi(env))
                   : (c->batch >= 256 ? 4 : c->batch >= 32 ? 2 : (c->n_vis >= 16384 && c->batch >= 3) ? 3 : 1);
    return std::min(k, c->batch);
}


}  // namespace

extern "C" {

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

int kvq_cache_sync_tail(kvq_cache* c) {
    return guarded([&] { sync_tail(c); });
}

int kvq_cache_reserve_tail(kvq_cache* c, size_t rows) {
    return guarded([&] { grow_tail(c, rows); });
}

int kvq_cache_set_path(kvq_cache* c, int path) {
    return guarded([&] {
        if (path < KVQ_PATH_AUTO || path > KVQ_PATH_DEQUANT) raise(KVQ_ERR_CONFIG, "unknown decode path");
        c->path = path;
    });
}

int kvq_cache_append(kvq_cache* c, const float* k_new, const float* v_new) {
    return guarded([&] {
        sync_tail(c);
        ensure_tail_room(c, 1);
        c->d_knew.upload(k_new, c->units * c->dim, c->stream);
        c->d_vnew.upload(v_new, c->units * c->dim, c->stream);
        ck(kvqb::launch_append(c->d_knew.p, c->d_vnew.p, c->batch, c->kv_heads, c->dim, c->tail_cap,
                               c->k_tail.p, c->v_tail.p, c->tail_len.p, c->overflow_flag(), c->stream), "append");
        sync(c->stream);
        c->n_tail += 1;
    });
}

int kvq_cache_append_device(kvq_cache* c, const float* k_new, const float* v_new, void* stream) {
    return guarded([&] {
        if (c->n_tail + 1 > c->tail_cap) {
            ck(cudaStreamSynchronize((cudaStream_t)stream), "sync");
            ensure_tail_room(c, 1);
        }
        ck(kvqb::launch_append(k_new, v_new, c->batch, c->kv_heads, c->dim, c->tail_cap, c->k_tail.p,
                               c->v_tail.p, c->tail_len.p, c->overflow_flag(), (cudaStream_t)stream), "append");
        c->n_tail += 1;
    });
}

int kvq_cache_decode(kvq_cache* c, const float* queries, float* out, float* weights, size_t* slope_violations) {
    return guarded([&] {
        if (weights) sync_tail(c);  // the probability rows are n_vis + n_tail long
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

int kvq_cache_step_device(kvq_cache* c, const float* queries, const float* k_new, const float* v_new, float* out,
                          void* stream) {
    return guarded([&] {
        if (c->n_tail + 1 > c->tail_cap) {
            ck(cudaStreamSynchronize((cudaStream_t)stream), "sync");
            ensure_tail_room(c, 1);
        }
        run_decode(c, queries, out, false, false, (cudaStream_t)stream, k_new, v_new);
        c->n_tail += 1;
    });
}



int kvq_cache_step(kvq_cache* c, const float* queries, const float* k_new, const float* v_new, float* out) {
    return guarded([&] {
        ensure_tail_room(c, 1);
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

int kvq_cache_info(const kvq_cache* cc, size_t info[10]) {
    kvq_cache* c = const_cast<kvq_cache*>(cc);  // the tail counter is a host mirror of device state
    const int st = guarded([&] { sync_tail(c); });
    if (st != KVQ_OK) return st;
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

int kvq_cache_memory(const kvq_cache* cc, size_t mem[6]) {
    // HybridKVCache::memory (kvcache.hpp:123-135), summed over every unit.
    kvq_cache* c = const_cast<kvq_cache*>(cc);
    const int st = guarded([&] { sync_tail(c); });
    if (st != KVQ_OK) return st;
    mem[0] = 2 * c->units * c->n_vis * c->rb;
    mem[1] = c->units * 4 * 4 * c->dim;
    if (c->v_token_wise()) mem[1] = c->units * (2 * 4 * c->dim + 4 * 4 * c->n_vis);  // K per channel; V per token (+ decode pair)
    mem[2] = mem[0] + mem[1];
    mem[3] = c->units * 2 * c->n_tail * c->dim * 4;
    mem[4] = c->units * 2 * c->n_vis * c->dim * 4;
    mem[5] = mem[2] + mem[3];
    return KVQ_OK;
}

int kvq_cache_resident_bytes(const kvq_cache* c, size_t bytes[4]) {
    const size_t seg = c->units * c->n_vis * c->rb;
    bytes[0] = seg;
    bytes[1] = c->v_operand_only ? 0 : seg;
    bytes[2] = c->vx.n;
    bytes[3] = c->vt.n + c->vref.n;
    return KVQ_OK;
}

int kvq_cache_read_segment(const kvq_cache* c, size_t unit, int which, uint8_t* bytes, float* alpha, float* beta) {
    return guarded([&] {
        if (unit >= c->units) raise(KVQ_ERR_DOMAIN, "segment index out of range");
        const size_t seg = c->n_vis * c->rb;
        DevBuf<uint8_t> tmp;
        const uint8_t* src = which == 0 ? c->k_codes() : v_ref_tmp(const_cast<kvq_cache*>(c), tmp, c->stream);
        if (seg && bytes) ck(cudaMemcpyAsync(bytes, src + unit * seg, seg, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (which == 1 && c->v_token_wise() && (alpha || beta))
            raise(KVQ_ERR_CONFIG, "token-wise V: per-channel stats do not exist (kvq_cache_read_value_token_stats)");
        const float* a = (which == 0 ? c->k_alpha() : c->v_alpha()) + unit * c->dim;
        const float* b = (which == 0 ? c->k_beta() : c->v_beta()) + unit * c->dim;
        if (alpha) ck(cudaMemcpyAsync(alpha, a, c->dim * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (beta) ck(cudaMemcpyAsync(beta, b, c->dim * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        sync(c->stream);
    });
}

int kvq_cache_read_value_token_stats(const kvq_cache* c, size_t unit, float* alpha, float* beta) {
    return guarded([&] {
        if (!c->v_token_wise()) raise(KVQ_ERR_CONFIG, "not a token-wise V cache");
        if (unit >= c->units) raise(KVQ_ERR_DOMAIN, "segment index out of range");
        const size_t n = c->n_vis;
        if (alpha) ck(cudaMemcpyAsync(alpha, c->vtok.p + unit * n, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        if (beta)
            ck(cudaMemcpyAsync(beta, c->vtok.p + (c->units + unit) * n, n * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        sync(c->stream);
    });
}

int kvq_cache_read_tail(const kvq_cache* cc, size_t unit, int which, float* out) {
    kvq_cache* c = const_cast<kvq_cache*>(cc);
    return guarded([&] {
        sync_tail(c);
        if (unit >= c->units) raise(KVQ_ERR_DOMAIN, "tail index out of range");
        const float* src = (which == 0 ? c->k_tail.p : c->v_tail.p) + unit * c->tail_cap * c->dim;
        if (c->n_tail)
            ck(cudaMemcpyAsync(out, src, c->n_tail * c->dim * 4, cudaMemcpyDeviceToHost, c->stream), "D2H");
        sync(c->stream);
    });
}

int kvq_cache_device_pointers(const kvq_cache* c, void* ptrs[9]) {
    ptrs[0] = c->k_codes();
    // V reference rows: rebuilt from the operand layout (and kept) for an eligible cache
    const int st = guarded([&] {
        ptrs[1] = const_cast<uint8_t*>(v_ref(const_cast<kvq_cache*>(c), c->stream));
        sync(c->stream);
    });
    if (st != KVQ_OK) return st;
    ptrs[2] = c->k_alpha();
    ptrs[3] = c->k_beta();
    ptrs[4] = c->v_alpha();
    ptrs[5] = c->v_beta();
    ptrs[6] = c->k_tail.p;
    ptrs[7] = c->v_tail.p;
    ptrs[8] = c->tail_len.p;
    return KVQ_OK;
}

}  // extern "C"
