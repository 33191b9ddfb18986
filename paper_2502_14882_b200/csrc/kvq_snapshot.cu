// kvq_snapshot.cu — cache snapshots (HybridKVCache::save / load, kvcache.hpp:137-218):
// the reference's KVQC / KVQP / KVQT byte stream, validated like the reference.
#include "capi_internal.cuh"

using namespace kvqb::capi;

// ---- cache snapshots: KVQC (kvcache.hpp:137-218) over KVQP (quantize.hpp:148-230) and
// KVQT (tensor_io.hpp:11-128) records, byte-identical to HybridKVCache::save -------------
//
// Every unit of a device cache has the same shapes, so the image is a fixed-size header
// followed by `units` equal head records; payloads move with 2-D copies between the
// cache's device layout and their record slots (the copy engines do the gather), headers
// are composed on the host. `load` validates the whole image on the host first (the
// reference's checks, messages and byte offsets), then uploads it.

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
    return guarded([&] {
        sync_tail(const_cast<kvq_cache*>(c));  // tail rows appended on the device count too
        *bytes = kCacheHeader + c->units * Record(c).bytes;
    });
}

int kvq_cache_save_image(const kvq_cache* c, void* image, size_t capacity, int image_on_device, void* stream) {
    return guarded([&] {
        sync_tail(const_cast<kvq_cache*>(c));
        if (c->v_token_wise()) raise(KVQ_ERR_CONFIG, "cache save: KVQC has no token-wise V stats");
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
        DevBuf<uint8_t> vtmp;  // V rows rebuilt from the operand layout (v_operand_only)
        for (int w = 0; w < 2; ++w) {
            put_headers(seg_at[w], hdr.data(), kSegHeader);
            put_headers(seg_at[w] + kSegHeader + r.code_bytes, hdr.data() + kSegHeader, 8);
            put_headers(ten_at[w], hdr.data() + kSegHeader + 8, kTensorHeader);
            const uint8_t* codes = w == 0 ? c->k_codes() : v_ref_tmp(const_cast<kvq_cache*>(c), vtmp, s);
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
            DevBuf<uint8_t> vtmp;  // V rows staged for the operand layout (v_operand_only)
            for (int w = 0; w < 2; ++w) {
                const SegInfo& s0 = segs[w];
                if (w == 1 && c->v_operand_only && rb_bytes) vtmp.alloc(U * rb_bytes);
                uint8_t* codes = w == 0 ? c->k_codes() : (c->v_operand_only ? vtmp.p : c->v_codes());
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
            if (c->v_operand_only) store_v_rows(c, vtmp.p, c->stream);
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

