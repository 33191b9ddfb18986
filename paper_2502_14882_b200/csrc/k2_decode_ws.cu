// k2_decode_ws.cu — K2 throughput path for many units: a persistent, warp-specialized
// version of the exact-integer IMMA decode (k2_decode_tc.cu), d = 128, b in {1, 2, 4},
// G <= 4 query heads per KV head, n <= 8192 visual tokens.
//
// Math (reference: kernels.hpp:14-26, 183-194, 277-283; calibrate.hpp:62-114;
// kvcache.hpp:263-311), per (unit, query head h):
//   score_j = (sum_c qs_c code_jc + q.alpha) / sqrt(d),  qs_c = q_c (beta_c - alpha_c) / L
//   row     = [g(score_vis) | score_tail],  g affine from (gamma, delta) of the vis part
//   out_c   = (s_c sum_j p_j code_jc + alpha_c sum_j p_j + sum_t p_t v_tc) / sum p
//
// One CTA per SM walks its units (u = blockIdx.x + k gridDim.x) with two warp roles:
//   * 8 "score" warps (phase A, q.K): per unit they fold the K scales into four balanced
//     int8 digit planes of the query (exact int32 scores, as k2_decode_tc.cu), stream their
//     eighth of the unit's K rows through a private cp.async.bulk ring (the ring runs on
//     into the next unit), and park the scores in tensor memory bank k & 1;
//   * 8 "value" warps (phase B, p.V): for the unit whose scores are complete, each turns
//     its eighth of the scores into 22-bit p (three u8 planes) and accumulates p.V over all
//     128 channels (IMMA u8 x u8, 64 accumulator registers) from the vx operand layout,
//     then the eight reduce exactly in shared memory and write the outputs.
// Score warps of unit k + 1 overlap value warps of unit k; two mbarriers per tensor-memory
// bank hand it over ("scores ready", count 8) and back ("bank free", count 8). The CTA-wide
// reductions of the per-CTA kernels become a 4-byte exchange per warp.
//
// Why (profiles/r02_*): the per-CTA IMMA kernels run one unit's phases back to back in
// every CTA; here each warp does one phase with registers sized for it (value warps hold
// all channels, so no probability work is duplicated and no pairing barrier is needed),
// the per-unit fixed costs of one role overlap the other role's streaming, and the
// tensor pipe sees both phases' IMMAs continuously.
#include <cstdlib>

#include "kvq_internal.cuh"
#include "kvq_ptx.cuh"

namespace kvqb {

namespace {

using namespace ptx;

constexpr int kDim = 128;
constexpr int kWA = 8, kWB = 8;          // score warps, value warps
constexpr int kThreads = 32 * (kWA + kWB);
constexpr int kStagesA = 4, kStageBytesA = 2048;
constexpr int kStagesB = 3, kStageBytesB = 4096;
constexpr int kTailMax = 64;             // fp32 tail tokens kept in-kernel
constexpr int kMaxN = 8192;              // two tensor-memory banks of <= 256 columns
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kMagic = 12582912.0f;    // 1.5 * 2^23: float -> int rounding trick
constexpr float kPScale = 4190000.0f;    // p in [0, 1(+eps)] -> integer < 2^22
constexpr float kLog2PScale = 21.9985188f;
constexpr int kPRow = 12;                // words per p-plane smem row (bank-conflict free)
constexpr int kBarA = 1, kBarB = 2;      // named barriers of the two roles

struct WsParams {
    DecodeArgs a;
    int T8;       // tokens per warp per unit (multiple of 32): ceil(n / 256) * 32
    int nk_max;   // units per CTA, at most
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
__device__ __forceinline__ void imma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void imma_u8u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, float a, float b, float c, float d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d)));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]));
    v[0] = __uint_as_float(r[0]), v[1] = __uint_as_float(r[1]), v[2] = __uint_as_float(r[2]), v[3] = __uint_as_float(r[3]);
}
__device__ __forceinline__ void red_add_u32(uint32_t* p, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

template <int BITS>
struct Geo {
    static constexpr int kRowBytes = 16 * BITS;                     // reference K row (M = 8)
    static constexpr int kKTok = kStageBytesA / kRowBytes;          // K tokens per stage (>= 32)
    static constexpr int kVBlk = 512 * BITS;                        // vx bytes per 32-token block
    static constexpr int kVBlkPerStage = kStageBytesB / kVBlk;      // >= 2
    static constexpr uint32_t kMask = 0x01010101u * ((1u << BITS) - 1u);
    static constexpr int kCpb = 8 / BITS;
};

// K side of phase A (k2_decode_tc.cu): channel c sits in byte j of register rho of lane
// group tt, shifted by sh (the code-slot position; undone in the query digits).
template <int BITS>
__device__ __forceinline__ int k_rho(int c, int word_bits, int& tt, int& j, int& sh) {
    constexpr int cpb = Geo<BITS>::kCpb;
    const int s_slot = cpb - 1 - c % cpb, qidx = (c / cpb) ^ (word_bits / 8 - 1);
    j = qidx & 3;
    const int tb = qidx >> 2;
    tt = tb / BITS;
    const int u = tb % BITS;
    sh = s_slot * BITS;
    return u * cpb + s_slot;
}

struct Smem {
    uint8_t* ringA;     // [kWA][kStagesA][kStageBytesA]
    uint8_t* ringB;     // [kWB][kStagesB][kStageBytesB]
    uint32_t* acc;      // [2 banks][16 nc][4 r][32 lanes] exact p.V sums of the value warps
    uint32_t* pw;       // [kWB][2][12][kPRow] p digit planes of a warp's block
    float* part;        // [2 banks][kWA][12]: per score warp min[4], max[4], tail max[4]
    float* tail_s;      // [2 banks][4 heads][kTailMax] fp32 tail scores
    float* mh;          // [2 banks][4 heads] softmax offset -m log2(e)
    uint32_t* wsum;     // [2 banks][kWB][4] u22 weight sums
    uint64_t* fullA;    // [kWA][kStagesA]
    uint64_t* fullB;    // [kWB][kStagesB]
    uint64_t* ready;    // [2 banks] scores complete (8 score-warp arrivals)
    uint64_t* freed;    // [2 banks] bank read (8 value-warp arrivals)
    uint32_t* tmem_slot;
};

__host__ __device__ inline size_t ws_smem_bytes(Smem* out = nullptr, uint8_t* base = nullptr) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 127) & ~size_t(127);
        return base + o;
    };
    uint8_t* ringA = take((size_t)kWA * kStagesA * kStageBytesA);
    uint8_t* ringB = take((size_t)kWB * kStagesB * kStageBytesB);
    uint8_t* acc = take((size_t)2 * 16 * 4 * 32 * 4);
    uint8_t* pw = take((size_t)kWB * 2 * 12 * kPRow * 4);
    uint8_t* part = take((size_t)2 * kWA * 12 * 4);
    uint8_t* tail_s = take((size_t)2 * 4 * kTailMax * 4);
    uint8_t* mh = take(2 * 4 * 4);
    uint8_t* wsum = take((size_t)2 * kWB * 4 * 4);
    uint8_t* fullA = take((size_t)kWA * kStagesA * 8);
    uint8_t* fullB = take((size_t)kWB * kStagesB * 8);
    uint8_t* ready = take(2 * 8);
    uint8_t* freed = take(2 * 8);
    uint8_t* slot = take(16);
    if (out) {
        out->ringA = ringA;
        out->ringB = ringB;
        out->acc = reinterpret_cast<uint32_t*>(acc);
        out->pw = reinterpret_cast<uint32_t*>(pw);
        out->part = reinterpret_cast<float*>(part);
        out->tail_s = reinterpret_cast<float*>(tail_s);
        out->mh = reinterpret_cast<float*>(mh);
        out->wsum = reinterpret_cast<uint32_t*>(wsum);
        out->fullA = reinterpret_cast<uint64_t*>(fullA);
        out->fullB = reinterpret_cast<uint64_t*>(fullB);
        out->ready = reinterpret_cast<uint64_t*>(ready);
        out->freed = reinterpret_cast<uint64_t*>(freed);
        out->tmem_slot = reinterpret_cast<uint32_t*>(slot);
    }
    return off;
}

// Tensor-memory columns: bank = 2 warps per lane quarter x T8/32 steps x 4 columns.
__host__ __device__ inline uint32_t bank_cols(int T8) { return (uint32_t)(T8 / 4); }
__host__ __device__ inline uint32_t alloc_cols(int T8) {
    uint32_t c = 32;
    while (c < 2 * bank_cols(T8)) c <<= 1;
    return c;
}

#define WSTRACE(k)                                                                         \
    do {                                                                                   \
        if (a.trace) a.trace[(size_t)blockIdx.x * 256 + (k)] = gtimer();                   \
    } while (0)

// ---- query prep (scale_query, kernels.hpp:183-194), one CTA of 128 channel threads per unit ----
// Q'_c = round(S_h qs_c / 2^sh_c) in 4 balanced int8 digit planes, S_h bounding the int32
// score so the IMMA accumulation is exact (as k2_decode_tc.cu's prologue), written as the
// phase-A B fragments [(pp, kb, r)][lane]; q_const[h] = (isd / S_h, q.alpha isd).
template <int BITS>
__global__ void __launch_bounds__(kDim) prep_q_kernel(const DecodeArgs a) {
    __shared__ float red[2][4][4];
    __shared__ uint32_t frag[512];
    const int unit = blockIdx.x, c = threadIdx.x, lane = c & 31, warp = c >> 5;
    const int G = (int)a.group;
    const float levels = (float)((1u << BITS) - 1u);
    for (int e = c; e < 512; e += kDim) frag[e] = 0u;
    const float ka = __ldg(a.k_alpha + (size_t)unit * kDim + c);
    const float kbeta = __ldg(a.k_beta + (size_t)unit * kDim + c);
    griddep_wait();  // q comes from the preceding kernel
    griddep_launch();
    const float range = __fsub_rn(kbeta, ka);
    const float stp = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
    float qsv[4], ab[4], sa[4];
#pragma unroll
    for (int h = 0; h < 4; ++h) {
        const float qv = h < G ? a.q[((size_t)unit * G + h) * kDim + c] : 0.0f;
        qsv[h] = range > 0.0f ? __fmul_rn(qv, stp) : 0.0f;
        ab[h] = fabsf(qsv[h]);
        sa[h] = __fmul_rn(qv, ka);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1)
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            ab[h] += __shfl_xor_sync(0xffffffffu, ab[h], o);
            sa[h] += __shfl_xor_sync(0xffffffffu, sa[h], o);
        }
    if (lane < 4) {
        float x = ab[0], y = sa[0];
#pragma unroll
        for (int h = 1; h < 4; ++h)
            if (lane == h) x = ab[h], y = sa[h];
        red[0][lane][warp] = x;
        red[1][lane][warp] = y;
    }
    __syncthreads();
    auto scale_of = [&](int h) {
        const float sum_abs = (red[0][h][0] + red[0][h][1]) + (red[0][h][2] + red[0][h][3]);
        return sum_abs > 0.0f ? 1073741824.0f * __frcp_rn(levels * sum_abs) : 0.0f;
    };
    {
        int tt, j, sh;
        const int rho = k_rho<BITS>(c, a.word_bits, tt, j, sh);
        const int kb = rho >> 1, r = rho & 1;
        uint8_t* fb = reinterpret_cast<uint8_t*>(frag);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (h >= G) break;
            const int Q = __float2int_rn(__fmul_rn(qsv[h], scale_of(h)) * __int_as_float((127 - sh) << 23));
            const int d0 = ((Q + 128) & 255) - 128;
            const int q1 = (Q - d0) >> 8;
            const int d1 = ((q1 + 128) & 255) - 128;
            const int q2 = (q1 - d1) >> 8;
            const int d2 = ((q2 + 128) & 255) - 128;
            const int d3 = (q2 - d2) >> 8;
            const int dg[4] = {d0, d1, d2, d3};
#pragma unroll
            for (int plane = 0; plane < 4; ++plane) {
                const int gg = 2 * h + (plane & 1), pp = plane >> 1;
                fb[4 * (((pp * 4 + kb) * 2 + r) * 32 + gg * 4 + tt) + j] = (uint8_t)(dg[plane] & 255);
            }
        }
    }
    __syncthreads();
    for (int e = c; e < 512; e += kDim) a.q_frag[(size_t)unit * 512 + e] = frag[e];
    if (c < 4) {
        const float isd0 = __fdiv_rn(1.0f, sqrtf((float)kDim));
        float cA = 0.f, cB = 0.f;
        if (c < G) {
            const float S_h = scale_of(c);
            const float qdota = (red[1][c][0] + red[1][c][1]) + (red[1][c][2] + red[1][c][3]);
            cA = S_h > 0.0f ? isd0 / S_h : 0.0f;
            cB = qdota * isd0;
        }
        a.q_const[(size_t)unit * 4 + c] = make_float2(cA, cB);
    }
}

template <int BITS>
__global__ void __launch_bounds__(kThreads, 1) decode_ws_kernel(const WsParams p) {
    using Gm = Geo<BITS>;
    const DecodeArgs& a = p.a;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int G = (int)a.group;  // <= 4
    const int n = (int)a.n_vis;
    const int T8 = p.T8;
    const int units = (int)a.units;
    const int nk = ((units - (int)blockIdx.x) + (int)gridDim.x - 1) / (int)gridDim.x;  // this CTA's units

    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem sm;
    ws_smem_bytes(&sm, smem_raw);
    if (threadIdx.x == 0) WSTRACE(0);

    if (threadIdx.x == 0) {
        for (int i = 0; i < kWA * kStagesA; ++i) mbar_init(&sm.fullA[i], 1);
        for (int i = 0; i < kWB * kStagesB; ++i) mbar_init(&sm.fullB[i], 1);
        for (int b = 0; b < 2; ++b) mbar_init(&sm.ready[b], kWA), mbar_init(&sm.freed[b], kWB);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < 2 * 16 * 4 * 32; i += kThreads) sm.acc[i] = 0u;
    const uint32_t tcols = alloc_cols(T8);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sm.tmem_slot)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *sm.tmem_slot;

    const int role_w = warp < kWA ? warp : warp - kWA;  // index within the role
    const int tok_lo = role_w * T8;                     // this warp's tokens of every unit
    const int nv = max(0, min(T8, n - tok_lo));          // valid ones
    // lane quarter role_w & 3; warps q and q + 4 take column halves of a bank
    const uint32_t tq = tbase + ((uint32_t)(32 * (role_w & 3)) << 16) + (uint32_t)((role_w >> 2) * (T8 / 8));
    auto unit_of = [&](int k) { return (int)blockIdx.x + k * (int)gridDim.x; };

    if (warp < kWA) {
        // ======================= score warps (phase A) =======================
        const int nsa = (nv + Gm::kKTok - 1) / Gm::kKTok;  // stages per unit
        uint8_t* ring = sm.ringA + warp * kStagesA * kStageBytesA;
        uint64_t* full = sm.fullA + warp * kStagesA;
        const int total = nsa * nk;
        auto issue = [&](int i) {  // lane 0: global stage i = (unit k, stage s)
            const int k = i / nsa, s = i - k * nsa;
            const int slot = i % kStagesA;
            const uint32_t bytes = (uint32_t)min(Gm::kKTok, nv - s * Gm::kKTok) * (uint32_t)Gm::kRowBytes;
            const uint8_t* src = a.k_codes + ((size_t)unit_of(k) * n + tok_lo + s * Gm::kKTok) * Gm::kRowBytes;
            mbar_expect_tx(&full[slot], bytes);
            bulk_g2s(ring + slot * kStageBytesA, src, bytes, &full[slot]);
        };
        if (lane == 0)
            for (int i = 0; i < min(kStagesA, total); ++i) issue(i);
        // the query fragments (prep kernel) and the tail come from the preceding kernels;
        // the codes streaming above are the cache's own
        griddep_wait();
        griddep_launch();
        if (threadIdx.x == 0) WSTRACE(3);
        // this lane's phase-A B fragments and (score scale, offset) of head t, one unit ahead
        auto load_q = [&](int k, uint32_t (&bq)[2][4][2], float2& cq) {
            const uint32_t* fr = a.q_frag + (size_t)unit_of(k) * 512 + lane;
#pragma unroll
            for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                    for (int r = 0; r < 2; ++r) bq[pp][kb][r] = __ldcg(fr + ((pp * 4 + kb) * 2 + r) * 32);
            cq = __ldcg(a.q_const + (size_t)unit_of(k) * 4 + t);
        };
        uint32_t bq[2][4][2], bqn[2][4][2];
        float2 cq, cqn;
        load_q(0, bq, cq);
        int gs = 0;  // global stage counter
        for (int k = 0; k < nk; ++k) {
            const int unit = unit_of(k);
            const int bank = k & 1;
            if (lane == 0 && warp == 0 && k < 8) WSTRACE(40 + 4 * k);
            if (k + 1 < nk) load_q(k + 1, bqn, cqn);  // in flight during this unit
            const float cA = cq.x, cB = cq.y;
            if (lane == 0 && warp == 0 && k < 8) WSTRACE(41 + 4 * k);
            // the bank is free once the value warps have read it (unit k - 2)
            if (k >= 2) mbar_wait(&sm.freed[bank], ((k >> 1) - 1) & 1);
            if (lane == 0 && warp == 0 && k < 8) WSTRACE(42 + 4 * k);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t tcol0 = tq + (uint32_t)bank * bank_cols(T8);
            float lo = INFINITY, hi = -INFINITY;
            // ---- phase A: D[16 tok x 8 (head, plane)] += K[16 tok x 32 ch] * Q[32 ch x 8] ----
            for (int s = 0; s < nsa; ++s, ++gs) {
                const int slot = gs % kStagesA;
                mbar_wait(&full[slot], (gs / kStagesA) & 1);
                const uint8_t* buf = ring + slot * kStageBytesA + g * Gm::kRowBytes + t * 4 * BITS;
                const int tok_st = s * Gm::kKTok;
                const int nsteps = min(Gm::kKTok / 32, (nv - tok_st + 31) / 32);
#pragma unroll
                for (int ks = 0; ks < Gm::kKTok / 32; ++ks) {
                    if (ks >= nsteps) break;
                    uint32_t w[4][BITS];  // row words of tokens g + 8 i
#pragma unroll
                    for (int i = 0; i < 4; ++i) {
                        const uint8_t* rowp = buf + (32 * ks + 8 * i) * Gm::kRowBytes;
                        if (BITS == 1) {
                            w[i][0] = *reinterpret_cast<const uint32_t*>(rowp);
                        } else if (BITS == 2) {
                            const uint2 v = *reinterpret_cast<const uint2*>(rowp);
                            w[i][0] = v.x, w[i][1 % BITS] = v.y;
                        } else {
                            const uint4 v = *reinterpret_cast<const uint4*>(rowp);
                            w[i][0] = v.x, w[i][1 % BITS] = v.y, w[i][2 % BITS] = v.z, w[i][3 % BITS] = v.w;
                        }
                    }
                    int acc[2][2][4];
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int pp = 0; pp < 2; ++pp) acc[u][pp][0] = acc[u][pp][1] = acc[u][pp][2] = acc[u][pp][3] = 0;
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
                        for (int u = 0; u < 2; ++u) {
                            uint32_t ar[4];
#pragma unroll
                            for (int q = 0; q < 2; ++q)
#pragma unroll
                                for (int hh = 0; hh < 2; ++hh) {
                                    const int rho = 2 * kb + q;
                                    ar[2 * q + hh] =
                                        w[2 * u + hh][rho / Gm::kCpb] & (Gm::kMask << ((rho % Gm::kCpb) * BITS));
                                }
#pragma unroll
                            for (int pp = 0; pp < 2; ++pp)
                                imma_u8s8(acc[u][pp], ar[0], ar[1], ar[2], ar[3], bq[pp][kb][0], bq[pp][kb][1]);
                        }
                    }
                    float sc[4];
#pragma unroll
                    for (int u = 0; u < 2; ++u)
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const uint32_t tot = (uint32_t)acc[u][0][2 * hh] + ((uint32_t)acc[u][0][2 * hh + 1] << 8) +
                                                 ((uint32_t)acc[u][1][2 * hh] << 16) +
                                                 ((uint32_t)acc[u][1][2 * hh + 1] << 24);
                            sc[2 * u + hh] = __fmaf_rn((float)(int)tot, cA, cB);
                        }
                    const int tok0 = tok_st + 32 * ks;
                    if (tok0 + 32 <= nv) {
                        lo = fminf(lo, fminf(fminf(sc[0], sc[1]), fminf(sc[2], sc[3])));
                        hi = fmaxf(hi, fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3])));
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (tok0 + g + 8 * i < nv) lo = fminf(lo, sc[i]), hi = fmaxf(hi, sc[i]);
                    }
                    tmem_st4(tcol0 + (uint32_t)(4 * (s * (Gm::kKTok / 32) + ks)), sc[0], sc[1], sc[2], sc[3]);
                }
                __syncwarp();
                if (lane == 0 && gs + kStagesA < total) issue(gs + kStagesA);
            }
            // fp32 tail rows (unless the tail pass owns them): warp w takes rows w, w + 8, ...
            float tmax = -INFINITY;  // head lane & 3
            const int ntl = a.tail_lse == nullptr ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
            if (ntl > warp) {
                const float isd = __fdiv_rn(1.0f, sqrtf((float)kDim));
                float4 qv[4];
#pragma unroll
                for (int h = 0; h < 4; ++h)
                    qv[h] = h < G ? *reinterpret_cast<const float4*>(a.q + ((size_t)unit * G + h) * kDim + 4 * lane)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
                for (int j = warp; j < ntl; j += kWA) {
                    const float4 kv =
                        *reinterpret_cast<const float4*>(a.k_tail + ((size_t)unit * a.tail_cap + j) * kDim + 4 * lane);
#pragma unroll
                    for (int h = 0; h < 4; ++h) {
                        if (h < G) {
                            float d = kv.x * qv[h].x + kv.y * qv[h].y + kv.z * qv[h].z + kv.w * qv[h].w;
#pragma unroll
                            for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                            d *= isd;
                            if (lane == 0) sm.tail_s[(bank * 4 + h) * kTailMax + j] = d;
                            if ((lane & 3) == h) tmax = fmaxf(tmax, d);
                        }
                    }
                }
            }
            // per-warp partial: min / max over lanes of the same head, tail max
#pragma unroll
            for (int o : {4, 8, 16}) {
                lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
                hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
            }
            float* pr = sm.part + (bank * kWA + warp) * 12;
            if (lane < 4) pr[lane] = lo, pr[4 + lane] = hi, pr[8 + lane] = tmax;
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.ready[bank]);
            if (lane == 0 && warp == 0) WSTRACE(8 + 2 * min(k, 7));
            if (lane == 0 && warp == 0 && k < 8) WSTRACE(43 + 4 * k);
            if (k + 1 < nk) {
#pragma unroll
                for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                    for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                        for (int r = 0; r < 2; ++r) bq[pp][kb][r] = bqn[pp][kb][r];
                cq = cqn;
            }
        }
    } else {
        // ======================= value warps (phase B) =======================
        const int vw = warp - kWA;
        const int nb_w = (nv + 31) / 32;                          // 32-token blocks per unit
        const int nsb = (nb_w + Gm::kVBlkPerStage - 1) / Gm::kVBlkPerStage;
        uint8_t* ring = sm.ringB + vw * kStagesB * kStageBytesB;
        uint64_t* full = sm.fullB + vw * kStagesB;
        const int total = nsb * nk;
        const size_t nb32 = (size_t)(n + 31) / 32;
        auto issue = [&](int i) {
            const int k = i / nsb, s = i - k * nsb;
            const int slot = i % kStagesB;
            const uint32_t bytes = (uint32_t)min(Gm::kVBlkPerStage, nb_w - s * Gm::kVBlkPerStage) * (uint32_t)Gm::kVBlk;
            const uint8_t* src = a.v_codes_x + ((size_t)unit_of(k) * nb32 + (size_t)(tok_lo / 32) + (size_t)s * Gm::kVBlkPerStage) *
                                                   (size_t)Gm::kVBlk;
            mbar_expect_tx(&full[slot], bytes);
            bulk_g2s(ring + slot * kStageBytesB, src, bytes, &full[slot]);
        };
        if (lane == 0)
            for (int i = 0; i < min(kStagesB, total); ++i) issue(i);
        griddep_wait();  // the tail (previous append) and, through the score warps, q
        griddep_launch();
        uint32_t* pw = sm.pw + vw * 2 * 12 * kPRow;
        const int btid = threadIdx.x - kWA * 32;  // 0..255
        int gs = 0;
        for (int k = 0; k < nk; ++k) {
            const int unit = unit_of(k);
            const int bank = k & 1;
            mbar_wait(&sm.ready[bank], (k >> 1) & 1);
            if (lane == 0 && vw == 0 && k < 8) WSTRACE(80 + 4 * k);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            // softmax parameters of head t (calibrate.hpp:62-114): gamma, delta over every
            // score warp's partial, the calibrated row max at an endpoint or in the tail
            float pa, pb, mexp;
            {
                const float* pr = sm.part + bank * kWA * 12;
                float gamma = INFINITY, delta = -INFINITY, tm = -INFINITY;
#pragma unroll
                for (int w2 = 0; w2 < kWA; ++w2) {
                    gamma = fminf(gamma, pr[w2 * 12 + t]);
                    delta = fmaxf(delta, pr[w2 * 12 + 4 + t]);
                    tm = fmaxf(tm, pr[w2 * 12 + 8 + t]);
                }
                const float width = __fsub_rn(delta, gamma);
                float A = 1.0f, B = -a.tau1, m = tm;
                if (width > 0.0f) {
                    const float r = __fdiv_rn(__fsub_rn(a.tau2, a.tau1), width);
                    A = 1.0f - r;
                    B = __fmaf_rn(r, gamma, -a.tau1);
                    m = fmaxf(m, fmaxf(__fsub_rn(gamma, a.tau1), __fsub_rn(delta, a.tau2)));
                } else {
                    m = fmaxf(m, __fsub_rn(gamma, a.tau1));
                }
                const bool live = t < G;
                pa = live ? A * kLog2e : 0.0f;
                pb = live ? (B - m) * kLog2e : -INFINITY;
                mexp = -m * kLog2e;
            }
            if (vw == 0 && lane < 4) sm.mh[bank * 4 + lane] = mexp;
            // the epilogue's operands, fetched while phase B streams: this thread's output
            // channel's V stats (its channel is fixed: btid mod 128) and the tail rows (L2)
            const int ntl = a.tail_lse == nullptr ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
            const float v_a = __ldg(a.v_alpha + (size_t)unit * kDim + (btid & (kDim - 1)));
            const float v_b = __ldg(a.v_beta + (size_t)unit * kDim + (btid & (kDim - 1)));
            if (btid < 4 * ntl)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(a.v_tail + ((size_t)unit * a.tail_cap + (btid >> 2)) * kDim +
                                                                32 * (btid & 3)));
            const uint32_t tcol0 = tq + (uint32_t)bank * bank_cols(T8);
            int vacc[16][4];
#pragma unroll
            for (int nc = 0; nc < 16; ++nc) vacc[nc][0] = vacc[nc][1] = vacc[nc][2] = vacc[nc][3] = 0;
            uint32_t wacc = 0;
            auto p_write = [&](int blk, uint32_t* tile) {
                float sc[4];
                tmem_ld4(tcol0 + (uint32_t)(4 * blk), sc);
                uint32_t v[4];
                if (blk * 32 + 32 <= nv) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float pr = ex2(__fmaf_rn(sc[j], pa, pb));
                        v[j] = __float_as_uint(__fmaf_rn(pr, kPScale, kMagic));
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const float pr = blk * 32 + g + 8 * j < nv ? ex2(__fmaf_rn(sc[j], pa, pb)) : 0.0f;
                        v[j] = __float_as_uint(__fmaf_rn(pr, kPScale, kMagic));
                    }
                }
                wacc += (v[0] + v[1]) + (v[2] + v[3]) - 4u * 0x4B400000u;
                const uint32_t p01 = prmt(v[0], v[1], 0x5140), p23 = prmt(v[2], v[3], 0x5140);
                const uint32_t q01 = prmt(v[0], v[1], 0x7362), q23 = prmt(v[2], v[3], 0x7362);
                uint32_t* rowp = tile + t * kPRow + g;
                rowp[0 * 4 * kPRow] = prmt(p01, p23, 0x5410);
                rowp[1 * 4 * kPRow] = prmt(p01, p23, 0x7632);
                rowp[2 * 4 * kPRow] = prmt(q01, q23, 0x5410) & 0x3F3F3F3Fu;
            };
            if (nb_w > 0) p_write(0, pw);
            __syncwarp();
            const uint32_t* arow = pw + g * kPRow + t;
            for (int s = 0; s < nsb; ++s, ++gs) {
                const int slot = gs % kStagesB;
                mbar_wait(&full[slot], (gs / kStagesB) & 1);
                const uint8_t* buf = ring + slot * kStageBytesB + lane * (16 * BITS);
                const int nb = min(Gm::kVBlkPerStage, nb_w - s * Gm::kVBlkPerStage);
#pragma unroll
                for (int blk = 0; blk < Gm::kVBlkPerStage; ++blk) {
                    if (blk >= nb) break;
                    const int b = s * Gm::kVBlkPerStage + blk;
                    const uint32_t* r0 = arow + (b & 1) * 12 * kPRow;
                    const uint32_t af0 = r0[0], af2 = r0[4];
                    const uint32_t af1 = g < 4 ? r0[8 * kPRow] : 0u;
                    const uint32_t af3 = g < 4 ? r0[8 * kPRow + 4] : 0u;
                    if (b + 1 < nb_w) p_write(b + 1, pw + ((b + 1) & 1) * 12 * kPRow);
                    uint32_t X[2][2 * BITS];
                    {
                        const uint4* xp = reinterpret_cast<const uint4*>(buf + blk * 32 * (16 * BITS));
#pragma unroll
                        for (int u = 0; u < BITS; ++u) {
                            const uint4 v4 = xp[u];
                            const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                const int idx = 4 * u + kk;
                                X[idx / (2 * BITS)][idx % (2 * BITS)] = w4[kk];
                            }
                        }
                    }
#pragma unroll
                    for (int nc = 0; nc < 16; ++nc) {
                        constexpr int cpb = Gm::kCpb;
                        const uint32_t m = Gm::kMask << ((nc % cpb) * BITS);
                        imma_u8u8(vacc[nc], af0, af1, af2, af3, X[0][nc / cpb] & m, X[1][nc / cpb] & m);
                    }
                    __syncwarp();
                }
                __syncwarp();
                if (lane == 0 && gs + kStagesB < total) issue(gs + kStagesB);
            }
            if (lane == 0 && vw == 0 && k < 8) WSTRACE(81 + 4 * k);
            // exact integer CTA reduction of this unit ([nc][r][lane] image, bank k & 1)
            uint32_t* accb = sm.acc + bank * 16 * 4 * 32;
#pragma unroll
            for (int nc = 0; nc < 16; ++nc)
#pragma unroll
                for (int r = 0; r < 4; ++r) red_add_u32(accb + (nc * 4 + r) * 32 + lane, (uint32_t)vacc[nc][r]);
            {
                uint32_t w = wacc;
                w += __shfl_xor_sync(0xffffffffu, w, 4);
                w += __shfl_xor_sync(0xffffffffu, w, 8);
                w += __shfl_xor_sync(0xffffffffu, w, 16);
                if (lane < 4) sm.wsum[(bank * kWB + vw) * 4 + lane] = w;
            }
            named_bar(kBarB, kWB * 32);
            if (lane == 0 && vw == 0 && k < 8) WSTRACE(82 + 4 * k);
            // output, thread per (head, channel); reads (and re-zeroes) its 3 image words
            for (int idx = btid; idx < G * kDim; idx += kWB * 32) {
                const int h = idx / kDim, ch = idx % kDim;
                constexpr int cpb = Gm::kCpb;
                const int s_slot = cpb - 1 - ch % cpb, rem = ch / cpb;
                const int gcol = rem / (2 * BITS), qq = rem % (2 * BITS);
                const int nc = qq * cpb + s_slot, tt = gcol >> 1, rlo = gcol & 1;
                uint32_t pl[3];
#pragma unroll
                for (int plane = 0; plane < 3; ++plane) {
                    const int row = plane * 4 + h;
                    const int gg = row & 7, r = ((row >> 3) << 1) | rlo;
                    uint32_t* wp = accb + (nc * 4 + r) * 32 + gg * 4 + tt;
                    pl[plane] = *wp;
                    *wp = 0u;
                }
                const float V = __fmaf_rn((float)pl[2], 65536.0f, __fmaf_rn((float)pl[1], 256.0f, (float)pl[0])) *
                                __int_as_float((127 - s_slot * BITS) << 23);
                unsigned long long ws = 0;
#pragma unroll
                for (int w2 = 0; w2 < kWB; ++w2) ws += sm.wsum[(bank * kWB + w2) * 4 + h];
                const float wv = (float)ws;
                constexpr float kInvLevelsV = 1.0f / (float)((1u << BITS) - 1u);
                const float v_step = fmaxf(__fsub_rn(v_b, v_a) * kInvLevelsV, 0.0f);
                float num = __fmaf_rn(v_step, V, v_a * wv), den = wv;
                const float mh = sm.mh[bank * 4 + h];  // the head's softmax offset (value warp 0)
                const float* vt = a.v_tail + (size_t)unit * a.tail_cap * kDim + ch;
                const float* ts = sm.tail_s + (bank * 4 + h) * kTailMax;
                int j = 0;
                for (; j + 8 <= ntl; j += 8) {  // 8 independent loads in flight, j ascending
                    float vv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) vv[u] = __ldg(vt + (size_t)(j + u) * kDim);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float pt = ex2(__fmaf_rn(ts[j + u], kLog2e, mh)) * kPScale;
                        den += pt;
                        num = __fmaf_rn(pt, vv[u], num);
                    }
                }
                if (j < ntl) {  // the last < 8 rows, loads still issued together
                    float vv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) vv[u] = j + u < ntl ? __ldg(vt + (size_t)(j + u) * kDim) : 0.0f;
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (j + u < ntl) {
                            const float pt = ex2(__fmaf_rn(ts[j + u], kLog2e, mh)) * kPScale;
                            den += pt;
                            num = __fmaf_rn(pt, vv[u], num);
                        }
                    }
                }
                a.out[((size_t)unit * G + h) * kDim + ch] = num / den;
                if (a.tail_lse && ch == 0) a.tail_lse[(size_t)unit * G + h] = log2f(den) - kLog2PScale - mh;
            }
            // this warp is done with the bank (its scores, partials and tail scores): hand it
            // back to the score warps
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.freed[bank]);
            if (lane == 0 && vw == 0) WSTRACE(24 + min(k, 7));
        }
    }
    // all roles done: release tensor memory
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(tcols));
    }
    if (threadIdx.x == 0) WSTRACE(5);
}

template <int BITS>
cudaError_t launch_bits(const DecodeArgs& a, int T8, cudaStream_t s) {
    {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)a.units);
        cfg.blockDim = dim3(kDim);
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        const cudaError_t e = cudaLaunchKernelEx(&cfg, prep_q_kernel<BITS>, a);
        note_launch();
        if (e != cudaSuccess) return e;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<size_t>(a.units, (size_t)sms);
    WsParams p{a, T8, (int)((a.units + grid - 1) / grid)};
    const size_t smem = ws_smem_bytes();
    auto kern = decode_ws_kernel<BITS>;
    static unsigned attr_done = 0;  // per instantiation, bit per device
    const cudaError_t ea = once_per_device(
        attr_done, [&] { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    if (ea != cudaSuccess) return ea;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[1];
    attrs[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    note_launch();
    return e;
}

int ws_t8(size_t n) { return (int)((n + 255) / 256 * 32); }

}  // namespace

// The persistent kernel pays off when every SM gets at least two units to pipeline; fewer
// or longer units stay on the per-CTA kernels (which split a unit over a cluster).
size_t decode_ws_scratch_bytes(size_t units) { return units * (512 * sizeof(uint32_t) + 4 * sizeof(float2)); }

bool decode_ws_supported(const DecodeArgs& a) {
    static const char* env = std::getenv("KVQ_WS_MIN_UNITS");  // tuning
    const size_t min_units = env ? (size_t)std::atoi(env) : 2 * 148;
    if (a.dim != (size_t)kDim || a.n_vis == 0 || a.units < min_units || !a.v_codes_x) return false;
    if (a.word_bits != 8 && a.word_bits != 16 && a.word_bits != 32) return false;
    if (a.bits != 1 && a.bits != 2 && a.bits != 4) return false;
    if (a.group < 1 || a.group > 4) return false;
    if (a.n_vis > (size_t)kMaxN) return false;
    if (a.tail_cap > (size_t)kTailMax && a.tail_lse == nullptr) return false;
    if (a.plan_units && a.plan_units != a.units) return false;  // chunked steps: per-CTA kernels
    return ws_smem_bytes() <= 227 * 1024;
}

cudaError_t launch_decode_ws(const DecodeArgs& a, cudaStream_t s) {
    const int T8 = ws_t8(a.n_vis);
    switch (a.bits) {
        case 1: return launch_bits<1>(a, T8, s);
        case 2: return launch_bits<2>(a, T8, s);
        case 4: return launch_bits<4>(a, T8, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace kvqb
