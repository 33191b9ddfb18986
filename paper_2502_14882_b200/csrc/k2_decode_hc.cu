// k2_decode_hc.cu — K2 throughput path, second generation: fused, calibrated, post-scaled
// quantized decode attention on the sm_100a integer tensor cores (mma.sync m16n8k32 IMMA),
// d = 128, b in {1, 2, 4}, G <= 4 query heads per KV head, 8-warp CTAs with the p.V phase
// split in channel halves ("hc").
//
// Math (reference: kernels.hpp:14-26, 183-194, 277-283; calibrate.hpp:62-114;
// kvcache.hpp:263-311), per (unit, query head h):
//   score_j = (sum_c qs_c code_jc + q.alpha) / sqrt(d),  qs_c = q_c (beta_c - alpha_c) / L
//   row     = [g(score_vis) | score_tail],  g affine from (gamma, delta) of the vis part
//   out_c   = (s_c sum_j p_j code_jc + alpha_c sum_j p_j + sum_t p_t v_tc) / sum p
//
// Why a second kernel (profiles/r01_ncu_decode_tc_c2.json, r02_*): the first IMMA kernel
// (k2_decode_tc.cu) is latency bound - 126 registers per thread cap it at 16 warps per SM
// (four 4-warp CTAs), every unit is resident at once, and its tensor pipe is 40 % busy.
// The tensor work itself cannot shrink: with G = 4 only 16 columns share an operand, which
// is below what tcgen05 needs (~35-47 cycles per M128 N16 instruction, the same tensor
// datapath as mma.sync: profiles/r02_umma_rate2.txt, r02_mma_mix.txt), and FP8 mma.sync is
// emulated on sm_100a (F2FP unpack + 2 HMMA). So this kernel attacks latency: the same
// exact-integer phases with half the registers, twice the warps:
//  * phase A (q.K) as in k2_decode_tc.cu (raw code bytes as A, one LOP3 per 4 codes, four
//    balanced int8 digit planes of the scaled query as B, exact int32 scores), with one
//    accumulator slot and the A registers built per k-block;
//  * phase B (p.V, 22-bit p in three u8 planes x V codes): a warp owns HALF the channels
//    of its token group - 32 accumulator registers instead of 64 - so every thread fits in
//    64 registers: 8-warp CTAs, four per SM, 32 warps per SM.
//
// CTA = 8 warps over one unit's token chunk T (<= 4096; a cluster of S CTAs when a unit is
// split): token group tg = warp & 3 (= its tensor-memory lane quarter) covers T/4 tokens;
// warps tg and tg + 4 split its phase A (T/8 tokens each) and its phase B channels (64
// each). Scores wait in tensor memory, lane-private columns of the shared lane quarter,
// so both warps of a group read every score of the group after the softmax-parameter
// barrier. Every warp streams its own operands (its K rows, then its V half) through a
// private cp.async.bulk ring.
#include <cooperative_groups.h>

#include <cstdlib>

#include "kvq_internal.cuh"
#include "kvq_ptx.cuh"

namespace cg = cooperative_groups;

namespace kvqb {

namespace {

using namespace ptx;

constexpr int kDim = 128;
constexpr int kW = 8;                  // warps per CTA
constexpr int kOcc = 4;                // CTAs per SM
constexpr int kStages = 2;             // per-warp ring depth
constexpr int kStageBytes = 2048;      // per-warp ring stage
constexpr int kTailMax = 64;           // fp32 tail tokens per CTA (rank 0)
constexpr int kMaxCluster = 16;
constexpr int kMaxT = 4096;            // tokens per CTA: 128 TMEM columns
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: float -> int rounding trick
constexpr float kPScale = 4190000.0f;  // p in [0, 1(+eps)] -> integer < 2^22 (22-bit digits)
constexpr float kLog2PScale = 21.9985188f;
constexpr int kPRow = 12;              // words per p-plane smem row (bank-conflict free)
struct HcParams {
    DecodeArgs a;
    int S, T;  // cluster size, tokens per CTA (multiple of 512)
};

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
// D += A(16x32, u8) * B(32x8, s8)
__device__ __forceinline__ void imma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D += A(16x32, u8) * B(32x8, u8)
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

template <int BITS>
struct Geo {
    static constexpr int kRowBytes = 16 * BITS;                 // reference K row (M = 8 layout)
    static constexpr int kKTokPerStage = kStageBytes / kRowBytes;  // >= 32
    static constexpr int kVBlk = 256 * BITS;                    // bytes per 32-token block per V half
    static constexpr int kVBlkPerStage = kStageBytes / kVBlk;   // >= 2
    static constexpr uint32_t kMask = 0x01010101u * ((1u << BITS) - 1u);
    static constexpr int kCpb = 8 / BITS;
};

// K side: channel held by byte j of B-register rho of lane-group t (a row's words
// t*BITS .. t*BITS+BITS-1; register rho = u*cpb + s extracts code slot s of word u) -
// the same operand arrangement as k2_decode_tc.cu.
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
    uint8_t* ring;     // [kW][kStages][kStageBytes]; after the V stream: cluster receive buffer
    uint32_t* acc;     // [16 nc][4 r][32 lanes]: CTA sum of the warps' p.V accumulators
    uint32_t* pw;      // [kW][2][12][kPRow] p digit planes; prologue scratch before phase B
    float* tail_s;     // [8][kTailMax] fp32 tail scores (rank 0)
    float* wpart;      // [kW][24] per-warp (min, max, tail max) per head
    float* allpart;    // [S][24] per-CTA partials
    float* gpar;       // [8][4] softmax parameters per head
    uint32_t* wsum;    // [kW][8] per-warp u22 weight sums per head
    uint64_t* full;    // [kW][kStages] TMA completion barriers
    uint32_t* tmem_slot;
};

__host__ __device__ inline size_t hc_smem_bytes(int S, Smem* out = nullptr, uint8_t* base = nullptr) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 127) & ~size_t(127);
        return base + o;
    };
    const size_t recv_bytes = S > 1 ? (size_t)S * (8 * kDim + 8) * 4 : 0;
    const size_t ring_bytes = (size_t)kW * kStages * kStageBytes;
    uint8_t* ring = take(ring_bytes > recv_bytes ? ring_bytes : recv_bytes);
    uint8_t* acc = take((size_t)16 * 4 * 32 * 4);
    uint8_t* pw = take((size_t)kW * 2 * 12 * kPRow * 4);
    uint8_t* tail_s = take((size_t)8 * kTailMax * 4);
    uint8_t* wpart = take((size_t)kW * 24 * 4);
    uint8_t* allpart = take((size_t)(S > 0 ? S : 1) * 24 * 4);
    uint8_t* gpar = take(32 * 4);
    uint8_t* wsum = take((size_t)kW * 8 * 4);
    uint8_t* full = take((size_t)kW * kStages * 8);
    uint8_t* slot = take(16);
    if (out) {
        out->ring = ring;
        out->acc = reinterpret_cast<uint32_t*>(acc);
        out->pw = reinterpret_cast<uint32_t*>(pw);
        out->tail_s = reinterpret_cast<float*>(tail_s);
        out->wpart = reinterpret_cast<float*>(wpart);
        out->allpart = reinterpret_cast<float*>(allpart);
        out->gpar = reinterpret_cast<float*>(gpar);
        out->wsum = reinterpret_cast<uint32_t*>(wsum);
        out->full = reinterpret_cast<uint64_t*>(full);
        out->tmem_slot = reinterpret_cast<uint32_t*>(slot);
    }
    return off;
}

// Tensor-memory columns of a CTA of T tokens: 4 per 32-token step of a token group, rounded
// up to the power of two >= 32 tcgen05.alloc needs.
__host__ __device__ inline uint32_t tmem_cols(int T) {
    uint32_t c = 32;
    while (c < (uint32_t)(T / 32)) c <<= 1;
    return c;
}

#define HCTRACE(k)                                                                         \
    do {                                                                                   \
        if (a.trace) a.trace[(size_t)blockIdx.x * 256 + (k)] = gtimer();                   \
    } while (0)

template <int BITS>
__global__ void __launch_bounds__(kW * 32, kOcc) decode_hc_kernel(const HcParams p) {
    using Gm = Geo<BITS>;
    const DecodeArgs& a = p.a;
    const int S = p.S, T = p.T;
    const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int unit = blockIdx.x / S;
    const int G = (int)a.group;  // <= 4
    auto qrow = [&](int h) { return (size_t)unit * G + h; };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int tg = warp & 3, hf = warp >> 2;

    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem sm;
    hc_smem_bytes(S, &sm, smem_raw);
    if (threadIdx.x == 0) HCTRACE(0);
    uint8_t* ring = sm.ring + warp * kStages * kStageBytes;
    uint64_t* full = sm.full + warp * kStages;

    const int n = (int)a.n_vis;
    const int n_cta = n - rank * T;  // visual tokens from this CTA's first (may exceed T)
    // phase A: this warp's half of its token group; phase B: the whole group, half the channels
    const int tgt = T / 4;
    const int a0 = tg * tgt + hf * (tgt / 2);         // CTA-relative first phase-A token
    const int nva = max(0, min(tgt / 2, n_cta - a0));  // valid phase-A tokens
    const int b0 = tg * tgt;
    const int nvb = max(0, min(tgt, n_cta - b0));      // valid tokens of the group
    const int nstage_a = (nva + Gm::kKTokPerStage - 1) / Gm::kKTokPerStage;
    const int nblk_b = (nvb + 31) / 32;
    const int nstage_b = (nblk_b + Gm::kVBlkPerStage - 1) / Gm::kVBlkPerStage;
    const int total_stages = nstage_a + nstage_b;

    auto issue = [&](int i) {  // lane 0: stage i (K stages, then V stages) into slot i % kStages
        const int slot = i % kStages;
        uint32_t bytes;
        const uint8_t* src;
        if (i < nstage_a) {
            src = a.k_codes + ((size_t)unit * n + rank * T + a0 + i * Gm::kKTokPerStage) * Gm::kRowBytes;
            bytes = (uint32_t)min(Gm::kKTokPerStage, nva - i * Gm::kKTokPerStage) * (uint32_t)Gm::kRowBytes;
        } else {
            const int si = i - nstage_a;
            const size_t nb32 = (size_t)(n + 31) / 32;
            src = a.v_codes_x2 + ((((size_t)unit * 2 + hf) * nb32 + (size_t)(rank * T + b0) / 32) * Gm::kVBlk) +
                  (size_t)si * kStageBytes;
            bytes = (uint32_t)min(Gm::kVBlkPerStage, nblk_b - si * Gm::kVBlkPerStage) * (uint32_t)Gm::kVBlk;
        }
        mbar_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + slot * kStageBytes, src, bytes, &full[slot]);
    };
    if (lane == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < min(kStages, total_stages); ++i) issue(i);
    }
    const uint32_t tcols = tmem_cols(T);
    for (int i = threadIdx.x; i < 16 * 4 * 32; i += kW * 32) sm.acc[i] = 0u;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sm.tmem_slot)),
                     "r"(tcols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // #0

    // fp32 tail: rank 0, unless the tail pass owns it (a.tail_lse). tail_len is written by
    // the previous step's append: the pre-dependency read is an L2 prefetch hint only.
    const bool own_tail = rank == 0 && a.tail_lse == nullptr;
    const int ntl_hint = own_tail ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
    for (int l = threadIdx.x; l < 8 * min(ntl_hint, kTailMax); l += blockDim.x) {
        const float* base = (l & 4) ? a.v_tail : a.k_tail;
        const float* ptr = base + ((size_t)unit * a.tail_cap + (l >> 3)) * kDim + 32 * (l & 3);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
    }
    const float k_a = __ldg(a.k_alpha + unit * kDim + (threadIdx.x & (kDim - 1)));
    const float k_b = __ldg(a.k_beta + unit * kDim + (threadIdx.x & (kDim - 1)));
    // q and the tail come from the preceding kernel (see k2_decode_tc.cu for the balanced
    // sibling launch that waits at exit instead)
    if (!a.dep_wait_at_end) griddep_wait();
    const int ntl = own_tail ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
    griddep_launch();
    if (threadIdx.x == 0) HCTRACE(3);

    // ---- fold the K scales into the query (scale_query, kernels.hpp:183-194) ----
    // Q'_c = round(S_h qs_c / 2^sh_c) in 4 balanced int8 digit planes, S_h bounding the
    // int32 score so IMMA accumulation is exact (as k2_decode_tc.cu).
    float* s_red = reinterpret_cast<float*>(sm.pw);              // [2][4 heads][4 warps]: sum|qs|, q.alpha
    uint32_t* s_frag = reinterpret_cast<uint32_t*>(s_red + 32);  // [2 pp][4 kb][2 r][32 lanes]
    const float levels = (float)((1u << BITS) - 1u);
    const float isd0 = __fdiv_rn(1.0f, sqrtf((float)kDim));
    auto scale_of = [&](int h) {
        const float sum_abs = (s_red[h * 4 + 0] + s_red[h * 4 + 1]) + (s_red[h * 4 + 2] + s_red[h * 4 + 3]);
        return sum_abs > 0.0f ? 1073741824.0f * __frcp_rn(levels * sum_abs) : 0.0f;
    };
    for (int e = threadIdx.x; e < 512; e += kW * 32) s_frag[e] = 0u;  // heads >= G stay 0
    float qsv[4];
    if (threadIdx.x < kDim) {
        const int c = threadIdx.x;
        const float range = __fsub_rn(k_b, k_a);
        const float stp = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
        float ab[4], sa[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            const float qv = h < G ? a.q[qrow(h) * kDim + c] : 0.0f;
            qsv[h] = range > 0.0f ? __fmul_rn(qv, stp) : 0.0f;
            ab[h] = fabsf(qsv[h]);
            sa[h] = __fmul_rn(qv, k_a);
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
            s_red[(0 * 4 + lane) * 4 + warp] = x;
            s_red[(1 * 4 + lane) * 4 + warp] = y;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // also publishes the TMEM allocation
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *sm.tmem_slot;
    // B fragments: entry (pp, kb, r, lane(gg, tt)) byte j = digit plane 2 pp + gg % 2 of head
    // gg / 2 at the channel k_rho maps to register rho = 2 kb + r of lane group tt
    if (threadIdx.x < kDim) {
        const int c = threadIdx.x;
        int tt, j, sh;
        const int rho = k_rho<BITS>(c, a.word_bits, tt, j, sh);
        const int kb = rho >> 1, r = rho & 1;
        uint8_t* fb = reinterpret_cast<uint8_t*>(s_frag);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
            if (h >= G) break;
            const int Q = __float2int_rn(__fmul_rn(qsv[h], scale_of(h)) * __int_as_float((127 - sh) << 23));
            // balanced base-256 digits: Q = d0 + 2^8 d1 + 2^16 d2 + 2^24 d3
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
                const int e = ((((pp * 4 + kb) * 2 + r) * 32) + gg * 4 + tt);
                fb[4 * e + j] = (uint8_t)(dg[plane] & 255);
            }
        }
    }
    __syncthreads();
    uint32_t bq[2][4][2];  // [digit-plane pair][k-block][reg]
#pragma unroll
    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
            for (int r = 0; r < 2; ++r) bq[pp][kb][r] = s_frag[((pp * 4 + kb) * 2 + r) * 32 + lane];
    float cA = 0.f, cB = 0.f;  // lane's head t
    if (t < G) {
        const float S_h = scale_of(t);
        const float qdota = (s_red[(4 + t) * 4 + 0] + s_red[(4 + t) * 4 + 1]) +
                            (s_red[(4 + t) * 4 + 2] + s_red[(4 + t) * 4 + 3]);
        cA = S_h > 0.0f ? isd0 / S_h : 0.0f;
        cB = qdota * isd0;
    }
    float lo = INFINITY, hi = -INFINITY;
    if (threadIdx.x == 0) HCTRACE(2);

    // ---------------- phase A: scores of this warp's tokens ----------------
    // D[16 tokens x 8 (head, plane)] += K[16 tokens x 32 ch] * Q[32 ch x 8]: A = raw code
    // bytes (one LOP3 selects 4 codes x 2^sh), B = the q digit planes. Lane (g, t) ends with
    // all four digit planes of head t for tokens g, g+8 (m-tile 0) and g+16, g+24 (1).
    const uint32_t tmem_q = tbase + ((uint32_t)(32 * tg) << 16);
    const int step_base = hf * (tgt / 2) / 32;  // group-local step of this warp's first token
    constexpr int kStepsA = Gm::kKTokPerStage / 32;
    for (int st = 0; st < nstage_a; ++st) {
        const int slot = st % kStages;
        mbar_wait(&full[slot], (st / kStages) & 1);
        const uint8_t* buf = ring + slot * kStageBytes + g * Gm::kRowBytes + t * 4 * BITS;
        const int tok_st = st * Gm::kKTokPerStage;  // warp-relative first token of the stage
        const int nsteps = min(kStepsA, (nva - tok_st + 31) / 32);
        const uint32_t tcol = tmem_q + (uint32_t)(4 * (step_base + tok_st / 32));
#pragma unroll
        for (int ks = 0; ks < kStepsA; ++ks) {
            if (ks >= nsteps) break;
            // row words of tokens g + 8 i (i = 2 u + hh): this lane's 4 BITS bytes
            uint32_t w[4][BITS];
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
            int acc[2][2][4];  // [m-tile][digit-plane pair]
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int pp = 0; pp < 2; ++pp) acc[u][pp][0] = acc[u][pp][1] = acc[u][pp][2] = acc[u][pp][3] = 0;
#pragma unroll
            for (int kb = 0; kb < 4; ++kb) {
#pragma unroll
                for (int u = 0; u < 2; ++u) {
                    uint32_t ar[4];  // rows g / g+8 x registers 2 kb / 2 kb + 1
#pragma unroll
                    for (int q = 0; q < 2; ++q)
#pragma unroll
                        for (int hh = 0; hh < 2; ++hh) {
                            const int rho = 2 * kb + q;
                            ar[2 * q + hh] = w[2 * u + hh][rho / Gm::kCpb] & (Gm::kMask << ((rho % Gm::kCpb) * BITS));
                        }
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp)
                        imma_u8s8(acc[u][pp], ar[0], ar[1], ar[2], ar[3], bq[pp][kb][0], bq[pp][kb][1]);
                }
            }
            // epilogue: digit planes 0..3 -> exact int32 score (wrapping u32 sum), min/max, TMEM
            float sc[4];
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const uint32_t total = (uint32_t)acc[u][0][2 * hh] + ((uint32_t)acc[u][0][2 * hh + 1] << 8) +
                                           ((uint32_t)acc[u][1][2 * hh] << 16) + ((uint32_t)acc[u][1][2 * hh + 1] << 24);
                    sc[2 * u + hh] = __fmaf_rn((float)(int)total, cA, cB);
                }
            const int tok0 = tok_st + 32 * ks;  // warp-relative
            if (tok0 + 32 <= nva) {
                lo = fminf(lo, fminf(fminf(sc[0], sc[1]), fminf(sc[2], sc[3])));
                hi = fmaxf(hi, fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3])));
            } else {  // the last, partial step: padded rows leave min / max alone
#pragma unroll
                for (int i = 0; i < 4; ++i)
                    if (tok0 + g + 8 * i < nva) lo = fminf(lo, sc[i]), hi = fmaxf(hi, sc[i]);
            }
            tmem_st4(tcol + 4 * ks, sc[0], sc[1], sc[2], sc[3]);
        }
        __syncwarp();
        if (lane == 0 && st + kStages < total_stages) issue(st + kStages);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    if (lane == 0) HCTRACE(8 + warp);

    // fp32 tail rows (rank 0): warp w takes rows w, w + kW, ...; lanes split the channels
    const float isd = __fdiv_rn(1.0f, sqrtf((float)kDim));
    float tmax = -INFINITY;  // for head (lane & 7)
    if (ntl > warp) {
        float4 qv[4];
#pragma unroll
        for (int h = 0; h < 4; ++h)
            qv[h] = h < G ? *reinterpret_cast<const float4*>(a.q + qrow(h) * kDim + 4 * lane)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j = warp; j < ntl; j += kW) {
            const float4 kv = *reinterpret_cast<const float4*>(a.k_tail + ((size_t)unit * a.tail_cap + j) * kDim + 4 * lane);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                if (h < G) {
                    float d = kv.x * qv[h].x + kv.y * qv[h].y + kv.z * qv[h].z + kv.w * qv[h].w;
#pragma unroll
                    for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                    d *= isd;
                    if (lane == 0) sm.tail_s[h * kTailMax + j] = d;
                    if ((lane & 7) == h) tmax = fmaxf(tmax, d);
                }
            }
        }
    }
    // per-warp partial record (min[8], max[8], tail max[8]); lane k < 24 owns entry k
    {
#pragma unroll
        for (int o : {4, 8, 16}) {
            lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
            hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
        }
        const float l8 = __shfl_sync(0xffffffffu, lo, lane & 3);
        const float h8 = __shfl_sync(0xffffffffu, hi, lane & 3);
        float mine = INFINITY;
        if (lane < 4) mine = l8;
        if (lane >= 8 && lane < 12) mine = h8;
        if (lane >= 12 && lane < 16) mine = -INFINITY;
        const float tm8 = __shfl_sync(0xffffffffu, tmax, lane & 7);
        if (lane >= 16 && lane < 24) mine = tm8;
        if (lane < 24) sm.wpart[warp * 24 + lane] = mine;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (threadIdx.x < 24) {  // CTA partial
        const int kk = threadIdx.x;
        float v = sm.wpart[kk];
        for (int w2 = 1; w2 < kW; ++w2) v = kk < 8 ? fminf(v, sm.wpart[w2 * 24 + kk]) : fmaxf(v, sm.wpart[w2 * 24 + kk]);
        if (S > 1) {
            asm volatile("barrier.cluster.wait.acquire;" ::: "memory");  // #0 (one warp)
            for (int r = 0; r < S; ++r) st_cluster_f32(sm.allpart + rank * 24 + kk, r, v);
        } else {
            sm.allpart[kk] = v;
        }
    }
    if (S > 1) {
        if (threadIdx.x >= 24) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");  // #0, the rest
        __syncwarp();
        cluster_arrive();  // #1: partials pushed everywhere
        cluster_wait();
    } else {
        __syncthreads();
    }
    if (threadIdx.x < 8) {  // global softmax parameters per head (calibrate.hpp:62-114)
        const int h = threadIdx.x;
        float gamma = INFINITY, delta = -INFINITY, tm = -INFINITY;
        for (int r = 0; r < S; ++r) {
            gamma = fminf(gamma, sm.allpart[r * 24 + h]);
            delta = fmaxf(delta, sm.allpart[r * 24 + 8 + h]);
            tm = fmaxf(tm, sm.allpart[r * 24 + 16 + h]);
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
        const bool live = h < G;
        sm.gpar[h * 4 + 0] = live ? A * kLog2e : 0.0f;
        sm.gpar[h * 4 + 1] = live ? (B - m) * kLog2e : -INFINITY;
        sm.gpar[h * 4 + 2] = -m * kLog2e;
    }
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (threadIdx.x == 0) HCTRACE(1);

    // ---------------- phase B: p . V over the token group, half the channels ----------------
    // D[16 head-planes x 8 ch] += P[16 x 32 tok] * V[32 tok x 8 ch]; 8 channel tiles per
    // warp. The two warps of a token group alternate blocks for the probabilities: lane
    // (g, t) turns the four scores of head t it reads from tensor memory (tokens g, g+8,
    // g+16, g+24 of the block) into 22-bit p in three u8 planes (A rows plane * 4 + head) in
    // the group's 4-tile ring; one named barrier per block pair hands them over. V codes are
    // the B operand, slot-selected by LOP3 (x 2^sh).
    int vacc[8][4];
#pragma unroll
    for (int nc = 0; nc < 8; ++nc) vacc[nc][0] = vacc[nc][1] = vacc[nc][2] = vacc[nc][3] = 0;
    uint32_t wacc = 0;
    const float pa = sm.gpar[t * 4 + 0], pb = sm.gpar[t * 4 + 1];
    constexpr int kTile = 12 * kPRow;
    uint32_t* ptile = sm.pw + tg * 4 * kTile;
    auto p_write = [&](int blk) {
        float sc[4];
        tmem_ld4(tmem_q + (uint32_t)(4 * blk), sc);
        uint32_t v[4];
        if (blk * 32 + 32 <= nvb) {
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float pr = ex2(__fmaf_rn(sc[j], pa, pb));
                v[j] = __float_as_uint(__fmaf_rn(pr, kPScale, kMagic));
            }
        } else {  // the group's last, partial block: padded tokens get p = 0
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float pr = blk * 32 + g + 8 * j < nvb ? ex2(__fmaf_rn(sc[j], pa, pb)) : 0.0f;
                v[j] = __float_as_uint(__fmaf_rn(pr, kPScale, kMagic));
            }
        }
        wacc += (v[0] + v[1]) + (v[2] + v[3]) - 4u * 0x4B400000u;
        const uint32_t p01 = prmt(v[0], v[1], 0x5140), p23 = prmt(v[2], v[3], 0x5140);
        const uint32_t q01 = prmt(v[0], v[1], 0x7362), q23 = prmt(v[2], v[3], 0x7362);
        uint32_t* rowp = ptile + (blk & 3) * kTile + t * kPRow + g;
        rowp[0 * 4 * kPRow] = prmt(p01, p23, 0x5410);
        rowp[1 * 4 * kPRow] = prmt(p01, p23, 0x7632);
        rowp[2 * 4 * kPRow] = prmt(q01, q23, 0x5410) & 0x3F3F3F3Fu;
    };
    const uint32_t* arow = ptile + g * kPRow + t;
    if (hf < nblk_b) p_write(hf);
    for (int st = 0; st < nstage_b; ++st) {
        const int i = nstage_a + st;
        const int slot = i % kStages;
        mbar_wait(&full[slot], (i / kStages) & 1);
        const uint8_t* buf = ring + slot * kStageBytes + lane * (8 * BITS);
        const int nb = min(Gm::kVBlkPerStage, nblk_b - st * Gm::kVBlkPerStage);
#pragma unroll
        for (int blk = 0; blk < Gm::kVBlkPerStage; ++blk) {
            if (blk >= nb) break;
            const int b = st * Gm::kVBlkPerStage + blk;
            if ((blk & 1) == 0) asm volatile("bar.sync %0, 64;" ::"r"(1 + tg) : "memory");  // pair (b, b+1) ready
            const uint32_t* r0 = arow + (b & 3) * kTile;
            const uint32_t af0 = r0[0], af2 = r0[4];
            const uint32_t af1 = g < 4 ? r0[8 * kPRow] : 0u;
            const uint32_t af3 = g < 4 ? r0[8 * kPRow + 4] : 0u;
            // the next pair's block of this warp, written while this pair's MMAs run
            if ((blk & 1) == 0 && b + 2 + hf < nblk_b) p_write(b + 2 + hf);
            uint32_t X[2][BITS];
            {
                const uint8_t* xp = buf + blk * 32 * (8 * BITS);
                if (BITS == 1) {
                    const uint2 v2 = *reinterpret_cast<const uint2*>(xp);
                    X[0][0] = v2.x, X[1][0] = v2.y;
                } else {
#pragma unroll
                    for (int u = 0; u < BITS / 2; ++u) {
                        const uint4 v4 = reinterpret_cast<const uint4*>(xp)[u];
                        const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                        for (int k = 0; k < 4; ++k) {
                            const int idx = 4 * u + k;  // [grp][wi]
                            X[idx / BITS][idx % BITS] = w4[k];
                        }
                    }
                }
            }
#pragma unroll
            for (int nc = 0; nc < 8; ++nc) {
                constexpr int cpb = Gm::kCpb;
                const uint32_t m = Gm::kMask << ((nc % cpb) * BITS);
                imma_u8u8(vacc[nc], af0, af1, af2, af3, X[0][nc / cpb] & m, X[1][nc / cpb] & m);
            }
        }
        __syncwarp();
        if (lane == 0 && i + kStages < total_stages) issue(i + kStages);
    }
    if (lane == 0) HCTRACE(16 + warp);
    // ---------------- CTA reduction (exact integer sums in shared memory) ----------------
#pragma unroll
    for (int nc = 0; nc < 8; ++nc)
#pragma unroll
        for (int r = 0; r < 4; ++r)
            red_add_u32(sm.acc + ((8 * hf + nc) * 4 + r) * 32 + lane, (uint32_t)vacc[nc][r]);
    {
        uint32_t w = wacc;  // the two warps of a group weighed disjoint blocks
        w += __shfl_xor_sync(0xffffffffu, w, 4);
        w += __shfl_xor_sync(0xffffffffu, w, 8);
        w += __shfl_xor_sync(0xffffffffu, w, 16);
        if (lane < 8) sm.wsum[warp * 8 + lane] = lane < 4 ? w : 0u;
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    float* recv = reinterpret_cast<float*>(sm.ring);
    if (S > 1) {
        __syncwarp();
        cluster_arrive();  // #2a: every CTA's ring is drained
        cluster_wait();
    }
    for (int idx = threadIdx.x; idx < G * kDim; idx += kW * 32) {
        const int h = idx / kDim, ch = idx % kDim;
        constexpr int cpb = Gm::kCpb;
        // invert the V channel map: ch = (2 BITS g' + q) cpb + (cpb - 1 - s), nc = q cpb + s,
        // accumulator column g' = 2 tt + (r & 1), row = plane * 4 + head = gg + 8 (r >> 1)
        const int s_slot = cpb - 1 - ch % cpb, rem = ch / cpb;
        const int gcol = rem / (2 * BITS), qq = rem % (2 * BITS);
        const int nc = qq * cpb + s_slot, tt = gcol >> 1, rlo = gcol & 1;
        uint32_t pl[3];
#pragma unroll
        for (int plane = 0; plane < 3; ++plane) {
            const int row = plane * 4 + h;
            const int gg = row & 7, r = ((row >> 3) << 1) | rlo;
            pl[plane] = sm.acc[(nc * 4 + r) * 32 + gg * 4 + tt];
        }
        const float V = __fmaf_rn((float)pl[2], 65536.0f, __fmaf_rn((float)pl[1], 256.0f, (float)pl[0])) *
                        __int_as_float((127 - s_slot * BITS) << 23);
        unsigned long long ws = 0;
        for (int w2 = 0; w2 < kW; ++w2) ws += sm.wsum[w2 * 8 + h];
        const float wv = (float)ws;
        constexpr float kInvLevelsV = 1.0f / (float)((1u << BITS) - 1u);
        const float v_a = __ldg(a.v_alpha + unit * kDim + ch), v_b = __ldg(a.v_beta + unit * kDim + ch);
        const float v_step = fmaxf(__fsub_rn(v_b, v_a) * kInvLevelsV, 0.0f);
        float num = __fmaf_rn(v_step, V, v_a * wv), den = wv;
        const float* vt = a.v_tail + (size_t)unit * a.tail_cap * kDim + ch;
        int j = 0;
        for (; j + 8 <= ntl; j += 8) {
            float vv[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) vv[u] = __ldg(vt + (size_t)(j + u) * kDim);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const float pt = ex2(__fmaf_rn(sm.tail_s[h * kTailMax + j + u], kLog2e, sm.gpar[h * 4 + 2])) * kPScale;
                den += pt;
                num = __fmaf_rn(pt, vv[u], num);
            }
        }
        for (; j < ntl; ++j) {
            const float pt = ex2(__fmaf_rn(sm.tail_s[h * kTailMax + j], kLog2e, sm.gpar[h * 4 + 2])) * kPScale;
            den += pt;
            num = __fmaf_rn(pt, __ldg(vt + (size_t)j * kDim), num);
        }
        if (S == 1) {
            a.out[qrow(h) * kDim + ch] = num / den;
            if (a.tail_lse && ch == 0) a.tail_lse[qrow(h)] = log2f(den) - kLog2PScale - sm.gpar[h * 4 + 2];
        } else {
            st_cluster_f32(recv + rank * (8 * kDim + 8) + idx, 0, num);
            if (ch == 0) st_cluster_f32(recv + rank * (8 * kDim + 8) + 8 * kDim + h, 0, den);
        }
    }
    if (S > 1) {
        __syncwarp();
        cluster_arrive();  // #2b: partial numerators / denominators are in rank 0
        cluster_wait();
        if (rank == 0) {
            for (int idx = threadIdx.x; idx < G * kDim; idx += kW * 32) {
                const int h = idx / kDim;
                float num = 0.f, den = 0.f;
                for (int r = 0; r < S; ++r) {
                    num += recv[r * (8 * kDim + 8) + idx];
                    den += recv[r * (8 * kDim + 8) + 8 * kDim + h];
                }
                a.out[qrow(h) * kDim + (idx % kDim)] = num / den;
                if (a.tail_lse && idx % kDim == 0)
                    a.tail_lse[qrow(h)] = log2f(den) - kLog2PScale - sm.gpar[h * 4 + 2];
            }
        }
    }
    if (threadIdx.x == 0) HCTRACE(5);
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(tcols));
    }
    if (a.dep_wait_at_end) griddep_wait();
}

// Token split: T <= 4096 tokens per CTA (the score columns); small batches split a unit
// over a cluster so that units x S covers the SMs (about one CTA per SM, as measured for the
// IMMA kernel, profiles/r01_tc_split2.txt), never below 512 tokens per CTA.
void plan(const DecodeArgs& a, int& S, int& T) {
    const int n = (int)a.n_vis;
    const int s_min = std::max(1, (n + kMaxT - 1) / kMaxT);
    const size_t pu = a.plan_units ? a.plan_units : a.units;
    const int want = (int)((128 + pu - 1) / pu);
    int s = std::max(s_min, std::min(want, kMaxCluster));
    static const int force = std::getenv("KVQ_HC_SPLIT") ? std::atoi(std::getenv("KVQ_HC_SPLIT")) : 0;  // tuning
    if (force > 0) s = std::max(s_min, std::min(force, kMaxCluster));
    if (a.split_override > 0) s = std::max(s_min, std::min(a.split_override, kMaxCluster));
    s = std::min(s, std::max(1, (n + 511) / 512));
    T = ((n + s - 1) / s + 511) / 512 * 512;
    S = (n + T - 1) / T;
}

template <int BITS>
cudaError_t launch_bits(const DecodeArgs& a, cudaStream_t s) {
    int S, T;
    plan(a, S, T);
    HcParams p{a, S, T};
    size_t smem = hc_smem_bytes(S);
    // TMEM guard: never more CTAs per SM than the 512 columns serve
    const int max_ctas = std::min(kOcc, (int)(512 / tmem_cols(T)));
    const size_t floor_bytes = 232448 / (max_ctas + 1) + 1;
    if (smem < floor_bytes) smem = floor_bytes;
    auto kern = decode_hc_kernel<BITS>;
    static unsigned attr_done = 0;  // per instantiation, bit per device
    const cudaError_t ea = once_per_device(attr_done, [&] {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return r != cudaSuccess ? r : cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    });
    if (ea != cudaSuccess) return ea;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.units * S));
    cfg.blockDim = dim3(kW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = (unsigned)S;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, p);
    note_launch();
    return e;
}

// ---- device layouts ------------------------------------------------------------------
// vx2: [unit][half][32-token block][lane 32][2 grp][b words] = the IMMA kernel's vx words
// (k2_decode_tc.cu: X[grp][q] byte ii = row byte 2 b g + q of token 4 grp + t + 8 ii) split
// into channel halves (q in [half b, half b + b)).
// Reference rows: M-bit LE words, codes MSB-first (bitpack.hpp:85); M = 16 / 32 rows are
// M = 8 rows with the bytes of each word reversed: byte k is at k ^ (M/8 - 1).
__device__ __forceinline__ uint32_t ref_code(const uint8_t* row, int c, int bits, int bx) {
    const int cpb = 8 / bits;
    const uint32_t byte = row[(c / cpb) ^ bx];
    return (byte >> (8 - bits * (c % cpb + 1))) & ((1u << bits) - 1u);
}

template <int BITS>
__global__ void __launch_bounds__(32) pack_vx2_kernel(const uint8_t* __restrict__ rows, int n, int nb32, int bx,
                                                      uint8_t* __restrict__ vx2) {
    constexpr int rb = 16 * BITS;
    const size_t unit = blockIdx.y, blk = blockIdx.x;
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    uint32_t X[2][2 * BITS];
#pragma unroll
    for (int grp = 0; grp < 2; ++grp)
#pragma unroll
        for (int q = 0; q < 2 * BITS; ++q) {
            uint32_t w = 0;
#pragma unroll
            for (int ii = 0; ii < 4; ++ii) {
                const int tok = (int)blk * 32 + 4 * grp + t + 8 * ii;
                const uint32_t byte = tok < n ? rows[((size_t)unit * n + tok) * rb + ((2 * BITS * g + q) ^ bx)] : 0u;
                w |= byte << (8 * ii);
            }
            X[grp][q] = w;
        }
#pragma unroll
    for (int hf = 0; hf < 2; ++hf) {
        uint32_t* dst = reinterpret_cast<uint32_t*>(vx2 + ((((size_t)unit * 2 + hf) * nb32 + blk) * 32 + lane) * (8 * BITS));
#pragma unroll
        for (int grp = 0; grp < 2; ++grp)
#pragma unroll
            for (int wi = 0; wi < BITS; ++wi) dst[grp * BITS + wi] = X[grp][hf * BITS + wi];
    }
}

}  // namespace

size_t vx2_bytes(size_t units, size_t n_vis, int bits) { return units * 2 * ((n_vis + 31) / 32) * 256 * (size_t)bits; }

cudaError_t launch_pack_vx2(const uint8_t* rows, size_t units, size_t n_vis, int bits, int word_bits, uint8_t* vx2,
                            cudaStream_t s) {
    if (n_vis == 0 || units == 0) return cudaSuccess;
    const int nb32 = (int)((n_vis + 31) / 32);
    const dim3 grid((unsigned)nb32, (unsigned)units);
    const int bx = word_bits / 8 - 1;
    switch (bits) {
        case 1: pack_vx2_kernel<1><<<grid, 32, 0, s>>>(rows, (int)n_vis, nb32, bx, vx2); break;
        case 2: pack_vx2_kernel<2><<<grid, 32, 0, s>>>(rows, (int)n_vis, nb32, bx, vx2); break;
        case 4: pack_vx2_kernel<4><<<grid, 32, 0, s>>>(rows, (int)n_vis, nb32, bx, vx2); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

bool decode_hc_supported(const DecodeArgs& a) {
    if (a.dim != (size_t)kDim || a.n_vis == 0 || a.units == 0) return false;
    if (!a.v_codes_x2) return false;
    if (a.word_bits != 8 && a.word_bits != 16 && a.word_bits != 32) return false;
    if (a.bits != 1 && a.bits != 2 && a.bits != 4) return false;
    if (a.group < 1 || a.group > 4) return false;
    if (a.tail_cap > (size_t)kTailMax && a.tail_lse == nullptr) return false;
    int S, T;
    plan(a, S, T);
    if (S > kMaxCluster || T > kMaxT) return false;
    return hc_smem_bytes(S) <= 200 * 1024;
}

cudaError_t launch_decode_hc(const DecodeArgs& a, cudaStream_t s) {
    switch (a.bits) {
        case 1: return launch_bits<1>(a, s);
        case 2: return launch_bits<2>(a, s);
        case 4: return launch_bits<4>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace kvqb
