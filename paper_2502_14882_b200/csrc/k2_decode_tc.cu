// k2_decode_tc.cu — K2 throughput path: fused, calibrated, post-scaled quantized decode
// attention on the sm_100a integer tensor cores (mma.sync m16n8k32 IMMA), d = 128,
// reference M = 8 byte layout, b in {1,2,4,8}, G <= 8 query heads per KV head.
//
// Math (reference: kernels.hpp:14-26, 183-194, 277-283; calibrate.hpp:62-114;
// kvcache.hpp:263-311), per (unit, query head h):
//   score_j = (sum_c qs_c code_jc + q.alpha) / sqrt(d),  qs_c = q_c (beta_c-alpha_c)/L
//   row     = [g(score_vis) | score_tail],  g affine from (gamma, delta) of the vis part
//   out_c   = (s_c sum_j p_j code_jc + alpha_c sum_j p_j + sum_t p_t v_tc) / sum p
//
// One kernel, a cluster of S CTAs per unit and head group (each CTA a contiguous token
// chunk, 8 or 4 warps, each warp a contiguous slice streamed through its own cp.async.bulk
// ring):
//   prologue  : fold the K scale into the query: Q'_c = round(S_h qs_c / 2^sh_c) in 4
//               balanced int8 digit planes (S_h keeps the int32 score exact) -> the B
//               fragments of the q.K MMA, built in shared memory while the ring fills
//   phase A   : IMMA [16 tokens x 32 ch] x [32 ch x 8 (head, plane)]; A operand = the raw
//               code bytes, one LOP3 selects 4 codes (x 2^sh) per register; scores parked
//               in lane-private tensor-memory columns
//   cluster #1: DSMEM exchange of per-CTA (min, max, tail max) -> gamma, delta, m
//   phase B   : p = exp(g(s) - m) as a 22-bit integer (three u8 planes), computed by the
//               lane that owns the score -> IMMA [16 head-planes x 32 tok] x [32 tok x 8
//               ch]; V codes pre-arranged as B registers (vx layout), slot-selected by LOP3
//   epilogue  : exact integer CTA reduction (shared-memory atomics), DSMEM push of partial
//               numerators / denominators to rank 0 (cluster #2)
// Packed K/V are never dequantized; the only fp32 math per token is the softmax.
#include <cooperative_groups.h>

#include <cstdlib>
#include <type_traits>

#include "kvq_internal.cuh"
#include "kvq_ptx.cuh"

namespace cg = cooperative_groups;

namespace kvqb {

namespace {

constexpr int kDim = 128;
constexpr int kStages = 2;
#ifndef KVQ_TC_PAIR  // phase A: two 1-bit blocks' IMMAs interleaved (8 independent accumulator
#define KVQ_TC_PAIR 1  // chains between dependent IMMAs; C2 33.4 -> 33.0 us); 0 = one block at a time
#endif
#ifndef KVQ_TC_STAGE_BYTES  // (tuning builds)
#define KVQ_TC_STAGE_BYTES 4096
#endif
constexpr int kStageBytes = KVQ_TC_STAGE_BYTES;
constexpr int kTailMax = 64;   // fp32 tail tokens per CTA
constexpr int kMaxCluster = 16;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23: float -> int rounding trick
constexpr int kPxHead = 24;            // P transpose tile: words per head (2 planes x 8 + pad: no bank conflicts)
constexpr int kPxWords = 4 * kPxHead;  // one 32-token block of one head group

template <int BITS, int SB = kStageBytes>
struct Geo {
    static constexpr int kRowBytes = 16 * BITS;
    // >= 32 tokens per stage: a stage holds whole 32-token phase-B blocks
    static constexpr int kStageBytesB = SB / kRowBytes >= 32 ? SB : 32 * kRowBytes;
    static constexpr int kStageTokens = kStageBytesB / kRowBytes;
    static constexpr int kCpb = 8 / BITS;  // codes per byte
    static constexpr uint32_t kMask = 0x01010101u * ((1u << BITS) - 1u);
};

struct TcParams {
    DecodeArgs a;
    int S, T;    // cluster size, visual tokens per CTA (multiple of 256)
    int groups;  // head groups per unit handled by separate CTAs (1, or 2 for G > 4 at NT = 1)
    int whole;   // mixed launch: CTAs [0, whole) each own a whole unit alone (T1 tokens); the
    int T1;      // rest are S-CTA clusters of the remaining units (0: uniform launch)
    int split_first;  // mixed launch: the split units' CTAs come first in the grid
    int late_trigger; // dependents released: 0 after the dependency wait, 1 at exit, 2 after phase B, 3 at its start
};

// ---- PTX helpers (mbarriers, bulk copies, cluster barriers, PDL: kvq_ptx.cuh) ---------
using namespace ptx;
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}
// Debug timeline (KVQ_TRACE_FILE): slot k of this CTA's 256-entry record.
#define TTRACE(k)                                                                          \
    do {                                                                                   \
        if (a.trace) a.trace[(size_t)blockIdx.x * 256 + (k)] = gtimer();                   \
    } while (0)
// D += A(16x32, u8) * B(32x8, s8)
__device__ __forceinline__ void imma_u8s8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
// D += A(16x32, u8) * B(32x8, u8)
__device__ __forceinline__ void imma_u8u8(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                          uint32_t b0, uint32_t b1) {
    asm("mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
        : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
        : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// K side: channel held by byte j of B-register rho of lane-group t (a row's words
// t*BITS .. t*BITS+BITS-1; register rho = u*cpb + s extracts code slot s of word u).
template <int BITS>
__device__ __forceinline__ int k_channel(int t, int rho, int j, int& shift) {
    constexpr int cpb = Geo<BITS>::kCpb;
    const int u = rho / cpb, s = rho % cpb;
    shift = s * BITS;
    return (4 * (t * BITS + u) + j) * cpb + (cpb - 1 - s);
}
// V side: channel of A-register index iota (= q*cpb + s) of lane-group g.
template <int BITS>
__device__ __forceinline__ int v_channel(int g, int iota, int& shift) {
    constexpr int cpb = Geo<BITS>::kCpb;
    const int q = iota / cpb, s = iota % cpb;
    shift = s * BITS;
    return (2 * BITS * g + q) * cpb + (cpb - 1 - s);
}

// ---- decode ------------------------------------------------------------------------------
constexpr int kWarps = 8;             // consumer warps per CTA
// Visual tokens per warp (contiguous), at most: the warp's scores wait in TMEM (4 columns
// per 32-token step and head group): 256 columns per 8-warp CTA x 2 per SM, or 128 per
// 4-warp CTA x 4 per SM = all 512.
template <int NT>
constexpr int warp_tokens() { return NT == 1 ? 1024 : 512; }
#ifndef KVQ_TC_WARP_TOKENS_CAP  // (tuning builds: cap the per-warp token count)
#define KVQ_TC_WARP_TOKENS_CAP 1024
#endif
inline int cta_tokens(int NT, int W = kWarps) { return W * std::min(NT == 1 ? 1024 : 512, KVQ_TC_WARP_TOKENS_CAP); }

// Per-warp TMA ring: ~10 KB in flight per warp (80 KB per CTA, two CTAs per SM) covers
// the ~2 us bulk-copy latency measured under load (profiles/r01_trace_umma_c2.txt).
#ifndef KVQ_TC_STAGES  // (tuning builds; 0 = by stage size and occupancy)
#define KVQ_TC_STAGES 0
#endif
// Ring geometry: 4 KB stages two deep per warp, for both CTA shapes - fewer barrier rounds
// per token than 2 KB x 5 and still two (8-warp) or four (4-warp) CTAs per SM
// (profiles/r01_tc_stage.txt, r01_tc_stage8.txt: C2 50.0 -> 47.8 us, C3 48.0 -> 45.5 us,
// C4 164.5 -> 154.7 us; a third 4 KB stage would drop 8-warp CTAs to one per SM).
template <int W>
constexpr int stage_bytes() { return kStageBytes; }
template <int BITS, int OCC, int W = kWarps>
constexpr int ring_stages() {
    constexpr int sb = Geo<BITS, stage_bytes<W>()>::kStageBytesB;
    return KVQ_TC_STAGES > 0 ? KVQ_TC_STAGES
           : OCC >= 2        ? (sb >= 4096 ? 2 : (OCC == 2 ? 5 : 3))
                             : (sb >= 4096 ? 4 : 8);  // one CTA per SM (G > 4, NT = 2)
}

struct Smem {  // carve-up of the dynamic shared memory of one decode CTA
    uint8_t* ring;       // [kWarps][kStages][kStageBytes]: per-warp TMA landing zones;
                         // after the V stream: the cluster receive buffer
    float* acc;          // [kWarps][NT][16 channel rows][32 lanes]: the warps' p.V partials
    uint32_t* pw;        // [kWarps][4 blocks][NT][kPxWords] P transpose tiles (prologue scratch first)
    float* tail_s;       // [8][kTailMax] fp32 tail scores (rank 0)
    float* wpart;        // [kWarps][24] per-warp (min, max, tail max) per head
    float* allpart;      // [S][24] per-CTA partials (pushed by every CTA of the cluster)
    float* gpar;         // [8][4] softmax parameters per head
    float* wsum;         // [kWarps][16] per-warp weight sums per head (unit scale); [8..16):
                         // token-wise V: the per-head sums of weight x alpha_j
    uint64_t* full;      // [kWarps][kStages] TMA completion barriers
    float* arow;         // [2][kDim] the fused append's new K / V row (staged by cp.async)
    uint32_t* tmem_slot;
};

template <int BITS, int NT, int OCC, int W = kWarps>
__host__ __device__ inline size_t tc_smem_bytes(int S, Smem* out = nullptr, uint8_t* base = nullptr) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 127) & ~size_t(127);
        return base + o;
    };
    constexpr int stage = Geo<BITS, stage_bytes<W>()>::kStageBytesB;
    const size_t recv_bytes = S > 1 ? (size_t)S * (8 * kDim + 8) * 4 : 0;
    const size_t ring_bytes = (size_t)W * ring_stages<BITS, OCC, W>() * stage;
    const size_t tail_use = recv_bytes;
    uint8_t* ring = take(ring_bytes > tail_use ? ring_bytes : tail_use);
    uint8_t* acc = take((size_t)W * NT * 16 * 32 * 4);
    uint8_t* pw = take((size_t)W * 4 * NT * kPxWords * 4);
    uint8_t* tail_s = take((size_t)8 * kTailMax * 4);
    uint8_t* wpart = take((size_t)W * 24 * 4);
    uint8_t* allpart = take((size_t)(S > 0 ? S : 1) * 24 * 4);
    uint8_t* gpar = take(32 * 4);
    uint8_t* wsum = take((size_t)W * 16 * 4);
    uint8_t* full = take((size_t)W * ring_stages<BITS, OCC, W>() * 8);
    uint8_t* arow = take(2 * kDim * 4);
    uint8_t* slot = take(16);
    if (out) {
        out->ring = ring;
        out->acc = reinterpret_cast<float*>(acc);
        out->pw = reinterpret_cast<uint32_t*>(pw);
        out->tail_s = reinterpret_cast<float*>(tail_s);
        out->wpart = reinterpret_cast<float*>(wpart);
        out->allpart = reinterpret_cast<float*>(allpart);
        out->gpar = reinterpret_cast<float*>(gpar);
        out->wsum = reinterpret_cast<float*>(wsum);
        out->full = reinterpret_cast<uint64_t*>(full);
        out->arow = reinterpret_cast<float*>(arow);
        out->tmem_slot = reinterpret_cast<uint32_t*>(slot);
    }
    return off;
}

// Tensor-memory traffic here touches no generic memory: no "memory" clobbers, so the
// compiler may overlap shared-memory work with it; the wait carries the loaded registers
// as operands so no use of them can be scheduled above it.
__device__ __forceinline__ void tmem_st4(uint32_t taddr, float a, float b, float c, float d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(__float_as_uint(a)),
                 "r"(__float_as_uint(b)), "r"(__float_as_uint(c)), "r"(__float_as_uint(d)));
}
__device__ __forceinline__ void tmem_ld4_issue(uint32_t taddr, uint32_t (&r)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&r)[4]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, float (&v)[4]) {
    uint32_t r[4];
    tmem_ld4_issue(taddr, r);
    tmem_ld_wait(r);
    v[0] = __uint_as_float(r[0]), v[1] = __uint_as_float(r[1]), v[2] = __uint_as_float(r[2]), v[3] = __uint_as_float(r[3]);
}
// N consecutive lane-private columns (N = 16 or 32), one load + one wait.
template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t (&r)[N]) {
    static_assert(N == 16 || N == 32, "tmem_ld_cols: 16 or 32 columns");
    if constexpr (N == 16) {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
    } else {
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
            "tcgen05.wait::ld.sync.aligned;"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
              "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
              "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
            : "r"(taddr));
    }
}

// CTA = W warps (8, or 4 for many short units); warp w owns visual tokens [w T/W, (w+1) T/W)
// of the CTA's chunk (at most 1024) and streams them (K codes, then V codes) through its own
// TMA ring, re-armed by its lane 0. A unit of n visual tokens takes S CTAs (a cluster, see
// plan()); with S = 1 there is no cluster traffic at all.
//
// Token order inside a 32-token step: the phase-A accumulator gives lane (g, t) the
// scores of tokens {g, g+8, g+16, g+24} for head t. Phase B uses exactly those four
// tokens as its k-group g (k = 4g + j <-> token 8j' ... see v_row below), so every lane
// turns its own scores into probabilities: scores never leave the lane. They wait in
// tensor memory (lane-private columns, tcgen05.st/ld) between the phases.
// Cross-warp reductions of the p.V accumulators are exact integer shared-memory atomics
// (deterministic); cross-CTA traffic is push-only.
template <int BITS, int NT, int OCC, int W = kWarps, bool VTOK = false>
__global__ void __launch_bounds__(W * 32, OCC) decode_tc_kernel(const TcParams p) {
    using Gm = Geo<BITS, stage_bytes<W>()>;
    constexpr int kStagesW = ring_stages<BITS, OCC, W>();
    constexpr int kSteps = warp_tokens<NT>() / 32;                 // 32-token steps per warp, at most
    constexpr uint32_t kTmemCols = (W / 4) * kSteps * 4 * NT;        // lane-sharing warps; 256 / 128
    const DecodeArgs& a = p.a;
    // Grid: (unit, head group, rank). With two head groups a CTA serves query heads
    // [4 grp, 4 grp + G) of its unit (softmax rows are per head, so the split is exact).
    // A mixed launch (balanced batches) puts `whole` solo CTAs first: unit = CTA index.
    // Mixed launch order: the split units' clusters first (the block scheduler deals them
    // out one per SM), then the solo CTAs fill the remaining slots.
    const int nsplit_ctas = p.whole > 0 ? (int)gridDim.x - p.whole : 0;
    const int solo_base = p.split_first ? nsplit_ctas : 0;  // first solo CTA
    const int split_base = p.split_first ? 0 : p.whole;     // first split CTA
    const bool solo = p.whole > 0 && (int)blockIdx.x >= solo_base && (int)blockIdx.x < solo_base + p.whole;
    const int S = solo ? 1 : p.S;
    const int T = solo ? p.T1 : p.T;
    const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int unit_g = solo ? (int)blockIdx.x - solo_base : p.whole + ((int)blockIdx.x - split_base) / S;
    // the head groups of one unit (G > 4) are adjacent clusters: they stream the same code
    // bytes at about the same time, so the second stream is served from L2
    const int grp = unit_g % p.groups;
    const int unit = unit_g / p.groups;
    const int G_all = (int)a.group;
    const int h0 = 4 * grp;
    const int G = p.groups > 1 ? min(4, G_all - h0) : G_all;
    auto qrow = [&](int h) { return (size_t)unit * G_all + h0 + h; };  // row of head h in q / out
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;

    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem sm;
    tc_smem_bytes<BITS, NT, OCC, W>(S, &sm, smem_raw);
    if (threadIdx.x == 0) TTRACE(0);
    if (threadIdx.x == 0 && a.trace) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        a.trace[(size_t)blockIdx.x * 256 + 31] = smid + 1;
    }
    uint8_t* ring = sm.ring + warp * kStagesW * Gm::kStageBytesB;
    uint64_t* full = sm.full + warp * kStagesW;

    const int n = (int)a.n_vis;
    const int wt = T / W;                          // tokens per warp (multiple of 32, <= 1024)
    const int tok0 = rank * T + warp * wt;                // this warp's first token
    const int nv = max(0, min(wt, n - tok0));
    // fp32 tail: rank 0, unless a separate tail pass owns it (a.tail_lse). tail_len is written
    // by the previous step's append: the pre-dependency read is an L2 prefetch hint only.
    const bool own_tail = rank == 0 && a.tail_lse == nullptr;
    const int ntl_hint = own_tail ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
    const uint8_t* kcodes = a.k_codes + ((size_t)unit * n + tok0) * Gm::kRowBytes;
    const int nb32 = (n + 31) >> 5;  // 32-token blocks of the unit (vx_layout)
    const uint8_t* vcodes = a.v_codes_x + ((size_t)unit * nb32 + (tok0 >> 5)) * (size_t)(32 * Gm::kRowBytes);
    const int nstage = (nv + Gm::kStageTokens - 1) / Gm::kStageTokens;
    const int total_stages = 2 * nstage;

    auto issue = [&](int i) {  // lane 0: stage i (K stages, then V stages) into slot i % kStagesW
        const int slot = i % kStagesW;
        const int si = i < nstage ? i : i - nstage;
        const uint8_t* src = (i < nstage ? kcodes : vcodes) + (size_t)si * Gm::kStageBytesB;
        const int rows_left = min(Gm::kStageTokens, nv - si * Gm::kStageTokens);
        // K: exact rows; V (vx_layout): whole 32-token blocks (zero-padded past n)
        const uint32_t bytes = (uint32_t)((i < nstage ? rows_left : (rows_left + 31) / 32 * 32) * Gm::kRowBytes);
        mbar_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + slot * Gm::kStageBytesB, src, bytes, &full[slot]);
    };
    if (lane == 0) {
        for (int i = 0; i < kStagesW; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < min(kStagesW, total_stages); ++i) issue(i);
    }
    // allocate the lane-private score columns
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sm.tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // (the allocation is published by the first prologue barrier below)
    if (threadIdx.x == 0) TTRACE(6);
    if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // #0

    // Warm L2 with the fp32 tail rows (rank 0 reads them after phase A / in the epilogue).
    for (int l = threadIdx.x; l < 8 * min(ntl_hint, kTailMax); l += blockDim.x) {
        const float* base = (l & 4) ? a.v_tail : a.k_tail;
        const float* ptr = base + ((size_t)unit * a.tail_cap + (l >> 3)) * kDim + 32 * (l & 3);
        asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
    }
    // ... and with the unit's query rows (written by the preceding kernel: a prefetch is only
    // a hint - L2 is the point of coherence, the loads proper come after the dependency wait)
    if (threadIdx.x < 4 * G)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a.q + qrow(threadIdx.x >> 2) * kDim + 32 * (threadIdx.x & 3)));
    // Cache-build data (stats: stable since the build synchronized) is loaded before the
    // grid dependency resolves; only q and the tail come from the preceding kernel.
    // output channel's V stats (token-wise V: per-token stats, read in phase B instead)
    const float v_a = VTOK ? 0.0f : __ldg(a.v_alpha + unit * kDim + (threadIdx.x & (kDim - 1)));
    const float v_b = VTOK ? 0.0f : __ldg(a.v_beta + unit * kDim + (threadIdx.x & (kDim - 1)));
    // q fold: warp w < 4 NT folds head slot w (heads >= G fold to zero digits); lane l
    // owns channels l + 32 i. The K stats are loaded before the dependency wait.
    constexpr int kHeadSlots = 4 * NT;
    const bool folder = warp < kHeadSlots;
    const int fh = warp;  // head slot folded by this warp
    const float levels = (float)((1u << BITS) - 1u);
    float f_ka[4], f_stp[4];
    if (folder) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane + 32 * i;
            f_ka[i] = __ldg(a.k_alpha + unit * kDim + c);  // in flight across the dependency wait:
            f_stp[i] = __ldg(a.k_beta + unit * kDim + c);  // used only after it (no stall before it)
        }
    }
    if (threadIdx.x == 0) TTRACE(7);
    // The previous step's append (tail rows, tail_len) and q are visible from here on. A
    // balancing sibling launch (dep_wait_at_end) starts only once every CTA of the first
    // launch has passed this wait, so it may skip it; it waits at exit instead, keeping
    // "this grid done" = "both launches done" for the kernel that follows.
    if (!a.dep_wait_at_end) griddep_wait();
    // tail_len is read by ONE thread and broadcast through shared memory (after the prologue
    // barrier): with the fused append, that thread also counts this CTA in (relaxed atomic,
    // its operand data-dependent on the loaded length so it issues only after the read
    // returned - no fence; the barrier orders the broadcast); the request's last counter
    // moves tail_len on at exit.
    const bool fused_append = a.k_new != nullptr && own_tail;
    int cnt_old = -1;
    const int ntl_read = threadIdx.x == (W - 1) * 32 && own_tail ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
    // Dependents (the tail pass, or the append) may launch now: this grid is fully resident
    // once every CTA has passed here, and they wait for its completion before writing.
    if (!p.late_trigger) griddep_launch();
    if (threadIdx.x == 0) TTRACE(3);
    if (folder) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {  // the K grid step per channel (quantize.hpp:91-127)
            const float range = __fsub_rn(f_stp[i], f_ka[i]);
            f_stp[i] = range > 0.0f ? __fdiv_rn(range, levels) : -1.0f;  // < 0: degenerate channel
        }
    }

    // ---- fold the K scales into the query (scale_query, kernels.hpp:183-194) ----
    // Q'_c = round(S_h qs_c / 2^sh_c) in 4 balanced int8 digit planes, S_h bounding the
    // int32 score so IMMA accumulation is exact. One warp per head slot: warp-level sums,
    // digits scattered straight into the B-fragment tiles (the pw tiles are idle until
    // phase B); one barrier publishes tiles, per-head constants and the TMEM allocation.
    float* s_head = reinterpret_cast<float*>(sm.pw);               // [8][2]: S_h, q.alpha
    uint32_t* s_frag = reinterpret_cast<uint32_t*>(s_head + 16);   // [NT][512] B fragments
    const float isd0 = __fdiv_rn(1.0f, sqrtf((float)kDim));
    if (folder) {
        const bool live = fh < G;
        float qsv[4], ab = 0.0f, sa = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float qv = live ? a.q[qrow(fh) * kDim + lane + 32 * i] : 0.0f;
            qsv[i] = f_stp[i] > 0.0f ? __fmul_rn(qv, f_stp[i]) : 0.0f;
            ab += fabsf(qsv[i]);
            sa += __fmul_rn(qv, f_ka[i]);
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            ab += __shfl_xor_sync(0xffffffffu, ab, o);
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
        }
        // S_h: |score_int| <= (2^b - 1) * sum|Q_c| <= 2^30 (exact int32 accumulation). Any
        // S_h with that bound is exact; the same value scales Q and the score back (cA).
        const float S_h = ab > 0.0f ? 1073741824.0f * __frcp_rn(levels * ab) : 0.0f;
        if (lane == 0) s_head[2 * fh] = S_h, s_head[2 * fh + 1] = sa;
        // B fragments: entry (hg, pp, kb, r, lane(gg, tt)) byte j = digit plane 2pp + gg%2 of
        // head 4hg + gg/2 at channel k_channel(tt, 2kb + r, j): invert k_channel
        // (ch = (4 (t BITS + u) + j) cpb + cpb - 1 - s, rho = u cpb + s).
        constexpr int cpb = Gm::kCpb;
        uint8_t* fb = reinterpret_cast<uint8_t*>(s_frag);
        const int hg = fh >> 2;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int c = lane + 32 * i;
            // raw row byte of channel c: c / cpb for M = 8, the same byte of the reversed LE
            // word for M = 16 / 32 (bitpack.hpp:85)
            const int s_slot = cpb - 1 - c % cpb, qidx = (c / cpb) ^ (a.word_bits / 8 - 1);
            const int j = qidx & 3, tb = qidx >> 2;
            const int tt = tb / BITS, u = tb % BITS;
            const int rho = u * cpb + s_slot, kb = rho >> 1, r = rho & 1;
            const int sh = s_slot * BITS;
            const int Q = __float2int_rn(__fmul_rn(qsv[i], S_h) * __int_as_float((127 - sh) << 23));
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
                const int gg = 2 * (fh & 3) + (plane & 1), pp = plane >> 1;
                const int e = ((((hg * 2 + pp) * 4 + kb) * 2 + r) * 32) + gg * 4 + tt;
                fb[4 * e + j] = (uint8_t)(dg[plane] & 255);
            }
        }
    }
    if (threadIdx.x == (W - 1) * 32) {  // (the load has long returned: no stall here)
        reinterpret_cast<volatile int*>(sm.tmem_slot)[1] = ntl_read;
        if (fused_append) cnt_old = atomicAdd(a.append_cnt + unit / (int)a.kv_heads, 1 + min(ntl_read, 0));
    }
    if (threadIdx.x == 0) TTRACE(24);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // also publishes the TMEM allocation and the tail length
    if (threadIdx.x == 0) TTRACE(25);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tbase = *sm.tmem_slot;
    const int ntl = reinterpret_cast<volatile int*>(sm.tmem_slot)[1];
    const bool append_rows = fused_append && grp == 0 && ntl < (int)a.tail_cap;
    if (append_rows && warp == 0) {  // K row then V row, 16 B per lane each (no register staging)
        const size_t src = (size_t)unit * kDim + 4 * lane;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm.arow + 4 * lane)), "l"(a.k_new + src)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm.arow + kDim + 4 * lane)),
                     "l"(a.v_new + src)
                     : "memory");
        asm volatile("cp.async.commit_group;" ::: "memory");
    }
    // lanes of warp quarter (warp % 4); warps 4..7 use the upper half of the columns
    const uint32_t tmem_w = tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * kSteps * 4 * NT);
    if (threadIdx.x == 0) TTRACE(26);
    // Fused append (K3, kvcache.hpp:99-109; semantics of k3_append.cu): the new rows were
    // staged into shared memory by cp.async after the dependency wait and are written to slot
    // ntl at exit (the decode reads rows < ntl only); the request's last tail owner (cnt_old,
    // counted above) moves tail_len on at exit. The next decode sees both after its
    // dependency wait (this grid complete).
    uint32_t bq[NT][2][4][2];  // [head group][digit-plane pair][k-block][reg]
    float cA[NT], cB[NT], lo[NT], hi[NT];
#pragma unroll
    for (int hg = 0; hg < NT; ++hg)
#pragma unroll
        for (int pp = 0; pp < 2; ++pp)
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int r = 0; r < 2; ++r) bq[hg][pp][kb][r] = s_frag[(((hg * 2 + pp) * 4 + kb) * 2 + r) * 32 + lane];
#pragma unroll
    for (int hg = 0; hg < NT; ++hg) {
        const int h = 4 * hg + t;  // this lane's head in C columns 2t, 2t+1
        float ca = 0.f, cb = 0.f;
        if (h < G) {
            const float S_h = s_head[2 * h];
            ca = S_h > 0.0f ? isd0 / S_h : 0.0f;
            cb = s_head[2 * h + 1] * isd0;
        }
        cA[hg] = ca, cB[hg] = cb;
        lo[hg] = INFINITY, hi[hg] = -INFINITY;
    }

    if (threadIdx.x == 0) TTRACE(2);  // prologue done (q planes in registers)
    // ---------------- phase A: scores of this warp's tokens ----------------
    // D[16 tokens x 8 (head, plane)] += K[16 tokens x 32 ch] * Q[32 ch x 8]: A = raw code
    // bytes (one LOP3 selects 4 codes x 2^sh), B = the q digit planes (registers). Lane
    // (g, t) ends with all four digit planes of head t for tokens g and g + 8.
    for (int st = 0; st < nstage; ++st) {
        const int slot = st % kStagesW;
        mbar_wait(&full[slot], (st / kStagesW) & 1);
        const uint8_t* buf = ring + slot * Gm::kStageBytesB;
        const int ns = min(Gm::kStageTokens, nv - st * Gm::kStageTokens);
        int accA[NT][2][2][4], accB[NT][2][2][4];  // two pipeline slots: [head group][tile][plane pair]
        auto mma_step = [&](int tile, int (&ac)[NT][2][2][4]) {
            uint32_t areg[2][2][8];  // [tile][token g / g+8][slot register rho]
#pragma unroll
            for (int u2 = 0; u2 < 2; ++u2) {
#pragma unroll
                for (int hf = 0; hf < 2; ++hf) {
                    const uint8_t* rowp = buf + (tile + 16 * u2 + 8 * hf + g) * Gm::kRowBytes + t * 4 * BITS;
                    uint32_t w[BITS];
                    if (BITS == 1) {
                        w[0] = *reinterpret_cast<const uint32_t*>(rowp);
                    } else if (BITS == 2) {
                        const uint2 v = *reinterpret_cast<const uint2*>(rowp);
                        w[0] = v.x, w[1 % BITS] = v.y;
                    } else {
#pragma unroll
                        for (int u = 0; u < BITS; u += 4) {
                            const uint4 v = *reinterpret_cast<const uint4*>(rowp + 4 * u);
                            w[u] = v.x, w[(u + 1) % BITS] = v.y, w[(u + 2) % BITS] = v.z, w[(u + 3) % BITS] = v.w;
                        }
                    }
#pragma unroll
                    for (int rho = 0; rho < 8; ++rho)
                        areg[u2][hf][rho] = w[rho / Gm::kCpb] & (Gm::kMask << ((rho % Gm::kCpb) * BITS));
                }
            }
#pragma unroll
            for (int hg = 0; hg < NT; ++hg)
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2)
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp)
                        ac[hg][u2][pp][0] = ac[hg][u2][pp][1] = ac[hg][u2][pp][2] = ac[hg][u2][pp][3] = 0;
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int hg = 0; hg < NT; ++hg)
#pragma unroll
                    for (int u2 = 0; u2 < 2; ++u2)
#pragma unroll
                        for (int pp = 0; pp < 2; ++pp)
                            imma_u8s8(ac[hg][u2][pp], areg[u2][0][2 * kb], areg[u2][1][2 * kb], areg[u2][0][2 * kb + 1],
                                      areg[u2][1][2 * kb + 1], bq[hg][pp][kb][0], bq[hg][pp][kb][1]);
        };
        auto epilogue = [&](int tile, const int (&ac)[NT][2][2][4]) {
            const int step = (st * Gm::kStageTokens + tile) >> 5;  // warp-local 32-token step
            const int tbase_tok = st * Gm::kStageTokens + tile;
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) {
                float sc[4];
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2) {
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        // digit planes 0..3 of head t, token g (+8): the plane sums combine
                        // modulo 2^32 (unsigned: defined wrap-around); the total is exact in int32
                        const uint32_t total = (uint32_t)ac[hg][u2][0][2 * hf] +
                                               ((uint32_t)ac[hg][u2][0][2 * hf + 1] << 8) +
                                               ((uint32_t)ac[hg][u2][1][2 * hf] << 16) +
                                               ((uint32_t)ac[hg][u2][1][2 * hf + 1] << 24);
                        sc[2 * u2 + hf] = __fmaf_rn((float)(int)total, cA[hg], cB[hg]);
                    }
                }
                if (tbase_tok + 32 <= nv) {  // full step (warp-uniform): min/max trees, no checks
                    lo[hg] = fminf(lo[hg], fminf(fminf(sc[0], sc[1]), fminf(sc[2], sc[3])));
                    hi[hg] = fmaxf(hi[hg], fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3])));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int tok = tbase_tok + 16 * (j >> 1) + 8 * (j & 1) + g;
                        if (tok < nv) {
                            lo[hg] = fminf(lo[hg], sc[j]);
                            hi[hg] = fmaxf(hi[hg], sc[j]);
                        }
                    }
                }
                tmem_st4(tmem_w + (uint32_t)((step * NT + hg) * 4), sc[0], sc[1], sc[2], sc[3]);
            }
        };
        const int nsteps = (ns + 31) >> 5;  // >= 1
        if constexpr (KVQ_TC_PAIR != 0 && BITS == 1) {
        // two blocks' IMMAs interleaved per k-block: 8 independent accumulator chains instead
        // of 4 between dependent IMMAs (1-bit rows are one 32-bit word per lane and row half)
        auto mma_pair = [&](int t0, int (&a0)[NT][2][2][4], int t1, int (&a1)[NT][2][2][4]) {
            uint32_t w[2][2][2][BITS];  // [block][u2][hf][word]
#pragma unroll
            for (int bk = 0; bk < 2; ++bk)
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2)
#pragma unroll
                    for (int hf = 0; hf < 2; ++hf) {
                        const uint8_t* rowp =
                            buf + ((bk ? t1 : t0) + 16 * u2 + 8 * hf + g) * Gm::kRowBytes + t * 4 * BITS;
#pragma unroll
                        for (int u = 0; u < BITS; ++u) w[bk][u2][hf][u] = reinterpret_cast<const uint32_t*>(rowp)[u];
                    }
#pragma unroll
            for (int hg = 0; hg < NT; ++hg)
#pragma unroll
                for (int u2 = 0; u2 < 2; ++u2)
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                        for (int e = 0; e < 4; ++e) a0[hg][u2][pp][e] = a1[hg][u2][pp][e] = 0;
#pragma unroll
            for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                for (int bk = 0; bk < 2; ++bk) {
                    auto& ac = bk ? a1 : a0;
#pragma unroll
                    for (int u2 = 0; u2 < 2; ++u2) {
                        uint32_t r[2][2];  // [hf][rho - 2 kb]
#pragma unroll
                        for (int hf = 0; hf < 2; ++hf)
#pragma unroll
                            for (int i = 0; i < 2; ++i) {
                                const int rho = 2 * kb + i;
                                r[hf][i] = w[bk][u2][hf][rho / Gm::kCpb] & (Gm::kMask << ((rho % Gm::kCpb) * BITS));
                            }
#pragma unroll
                        for (int hg = 0; hg < NT; ++hg)
#pragma unroll
                            for (int pp = 0; pp < 2; ++pp)
                                imma_u8s8(ac[hg][u2][pp], r[0][0], r[1][0], r[0][1], r[1][1], bq[hg][pp][kb][0],
                                          bq[hg][pp][kb][1]);
                    }
                }
        };
        int k = 0;
        for (; k + 1 < nsteps; k += 2) {
            mma_pair(32 * k, accA, 32 * (k + 1), accB);
            epilogue(32 * k, accA);
            epilogue(32 * (k + 1), accB);
        }
        if (k < nsteps) {
            mma_step(32 * k, accA);
            epilogue(32 * k, accA);
        }
        } else {
        mma_step(0, accA);
        int k = 1;
        for (; k + 1 < nsteps; k += 2) {  // unrolled by two: register-resident pipeline slots
            mma_step(32 * k, accB);
            epilogue(32 * (k - 1), accA);
            mma_step(32 * (k + 1), accA);
            epilogue(32 * k, accB);
        }
        if (k < nsteps) {
            mma_step(32 * k, accB);
            epilogue(32 * (k - 1), accA);
            epilogue(32 * k, accB);
        } else {
            epilogue(32 * (k - 1), accA);
        }
        }
        __syncwarp();
        if (lane == 0 && st + kStagesW < total_stages) issue(st + kStagesW);
    }
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");  // scores are in tensor memory
    if (lane == 0) TTRACE(8 + warp);  // phase A done, per warp

    // fp32 tail rows (rank 0, naive_qk kernels.hpp:401-413): warp w takes rows w, w + W, ...
    // in batches of RB rows whose loads are all in flight at once; lane = 4 channels; the
    // RB x HB partial dots of a batch are reduced with one warp reduce-scatter (31 shuffles:
    // lane l ends with the full dot of row l / HB, head l % HB).
    const float isd = __fdiv_rn(1.0f, sqrtf((float)kDim));
    constexpr int HB = 4 * NT, RB = 32 / HB;
    float tmax = -INFINITY;  // head lane % HB
    if (ntl > warp) {
        float4 qv[HB];
#pragma unroll
        for (int h = 0; h < HB; ++h)
            qv[h] = h < G ? *reinterpret_cast<const float4*>(a.q + qrow(h) * kDim + 4 * lane)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        for (int j0 = warp; j0 < ntl; j0 += RB * W) {
            float4 kv[RB];
#pragma unroll
            for (int r = 0; r < RB; ++r) {
                const int j = j0 + r * W;
                kv[r] = j < ntl ? __ldcg(reinterpret_cast<const float4*>(a.k_tail + ((size_t)unit * a.tail_cap + j) * kDim) + lane)
                                : make_float4(0.f, 0.f, 0.f, 0.f);
            }
            float v[32];
#pragma unroll
            for (int r = 0; r < RB; ++r)
#pragma unroll
                for (int h = 0; h < HB; ++h)
                    v[r * HB + h] = kv[r].x * qv[h].x + kv[r].y * qv[h].y + kv[r].z * qv[h].z + kv[r].w * qv[h].w;
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const bool up = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < o; ++i) {
                    const float send = up ? v[i] : v[i + o], keep = up ? v[i + o] : v[i];
                    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            const int j = j0 + (lane / HB) * W, h = lane % HB;
            if (j < ntl && h < G) {
                const float d = v[0] * isd;
                sm.tail_s[h * kTailMax + j] = d;
                tmax = fmaxf(tmax, d);
            }
        }
    }
#pragma unroll
    for (int o = HB; o < 32; o <<= 1) tmax = fmaxf(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    if ((lane & 7) >= HB) tmax = -INFINITY;  // lane & 7 = head below (heads >= HB absent)
    if (threadIdx.x == 0) TTRACE(27);  // tail scores done (warp 0)
    // Per-warp partial record (min[8], max[8], tail max[8]); lane k < 24 owns entry k.
    float mine = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
#pragma unroll
        for (int o : {4, 8, 16}) {
            lo[nt] = fminf(lo[nt], __shfl_xor_sync(0xffffffffu, lo[nt], o));
            hi[nt] = fmaxf(hi[nt], __shfl_xor_sync(0xffffffffu, hi[nt], o));
        }
        // lane t (< 4) holds head 4nt + t
        const float l8 = __shfl_sync(0xffffffffu, lo[nt], lane & 3);
        const float h8 = __shfl_sync(0xffffffffu, hi[nt], lane & 3);
        if ((lane >> 2) == nt) mine = l8;              // lanes 4nt..4nt+3: min
        if (lane >= 8 && lane < 16 && ((lane - 8) >> 2) == nt) mine = h8;  // lanes 8+4nt..: max
    }
    if (lane >= 4 * NT && lane < 8) mine = INFINITY;  // absent heads
    const float tm8 = __shfl_sync(0xffffffffu, tmax, lane & 7);
    if (lane >= 16 && lane < 24) mine = tm8;
    if (lane < 24) sm.wpart[warp * 24 + lane] = mine;
    __syncthreads();
    if (threadIdx.x == 0) TTRACE(30);  // warp partials complete
    if (threadIdx.x < 24) {  // CTA partial
        const int kk = threadIdx.x;
        float v = sm.wpart[kk];
        for (int w2 = 1; w2 < W; ++w2) v = kk < 8 ? fminf(v, sm.wpart[w2 * 24 + kk]) : fmaxf(v, sm.wpart[w2 * 24 + kk]);
        if (S > 1) {
            asm volatile("barrier.cluster.wait.acquire;" ::: "memory");  // #0 (non-aligned: one warp)
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
    // Global softmax parameters per head.
    if (threadIdx.x < 8) {
        const int h = threadIdx.x;
        float gamma = INFINITY, delta = -INFINITY, tm = -INFINITY;
        for (int r = 0; r < S; ++r) {
            gamma = fminf(gamma, sm.allpart[r * 24 + h]);
            delta = fmaxf(delta, sm.allpart[r * 24 + 8 + h]);
            tm = fmaxf(tm, sm.allpart[r * 24 + 16 + h]);
        }
        // g(x) = A x + B (calibrate.hpp:62-67): g(gamma) = gamma - tau1, g(delta) =
        // delta - tau2; the calibrated row max is at an endpoint (or in the tail).
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
    // tail scores -> weights on the unit scale (read by the output pass after the next barrier)
    for (int e = threadIdx.x; e < G * ntl; e += W * 32) {
        const int h = e / ntl, j = e % ntl;
        sm.tail_s[h * kTailMax + j] = ex2(__fmaf_rn(sm.tail_s[h * kTailMax + j], kLog2e, sm.gpar[h * 4 + 2]));
    }

    if (threadIdx.x == 0) TTRACE(1);  // softmax parameters known
    if (p.late_trigger == 3) griddep_launch();  // release at the start of phase B (see launch_occ)
    // ---------------- phase B: p . V over this warp's tokens ----------------
    // D[16 channels x 8 (head, plane)] += V^T[16 ch x 32 tok] * P[32 tok x 8 (head, plane)]:
    // 8 channel tiles per 32-token block and head group (half the MMAs of a P-rows tile).
    // A operand = the V codes of 4 tokens of one channel row per register, x 2^sh (one LOP3
    // slot select on the vy layout; the per-channel 2^sh is divided out at the end). B = the
    // probabilities of the block as two u8 planes of a 16-bit integer, normalised per
    // 128-token group and head: P = round(2^(z - zmax_grp) (2^16 - 1)), so each group keeps
    // 16 bits relative to its own largest weight; the group's integer sums are folded into
    // fp32 accumulators with the group's exact scale 2^zmax_grp / (2^16 - 1).
    // Lane (g, t) owns the scores of head t for tokens {g + 8 j} of each block (phase A C
    // fragment); the P tile is transposed through shared memory so that B register 0 / 1 of
    // lane (g', t') holds the 4 tokens {2t' + 8 j} / {2t' + 1 + 8 j} of column g' - the
    // k-order the vy layout stores the V codes in.
    constexpr int cpb = Gm::kCpb;
    float fac[NT][16];  // channel rows rho = 2 mt + r (channel 16 mt + 8 r + g), head 4 hg + t
    float fw[NT];       // weight sum of head 4 hg + t (lane's tokens), unit scale
    float fa[NT];       // token-wise V: sum of weight x alpha_j (lane's tokens)
    float pa[NT], pb[NT];
#pragma unroll
    for (int hg = 0; hg < NT; ++hg) {
#pragma unroll
        for (int i = 0; i < 16; ++i) fac[hg][i] = 0.0f;
        fw[hg] = 0.0f;
        fa[hg] = 0.0f;
        pa[hg] = sm.gpar[(4 * hg + t) * 4 + 0];
        pb[hg] = sm.gpar[(4 * hg + t) * 4 + 1];
    }
    uint32_t* px = sm.pw + warp * (4 * NT * kPxWords);  // [4 blocks][NT][head 4][plane 2][8 (+pad)]
    constexpr int kBps = Gm::kStageTokens / 32;  // 32-token blocks per stage
    const int nblk_all = (nv + 31) >> 5;
    for (int b0 = 0; b0 < nblk_all; b0 += 4) {
        const int nbg = min(4, nblk_all - b0);
        // token-wise V: the group's per-token (step, offset) pairs, loaded once, under the
        // TMEM load and the exponentials
        float2 tso[4][VTOK ? 4 : 1];
        if constexpr (VTOK) {
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int tl = (b0 + bb) * 32 + 16 * (j >> 1) + 8 * (j & 1) + g;  // warp-local token
                    tso[bb][j] = __ldg(a.v_tok_so + (size_t)unit * n + tok0 + min(tl, max(nv - 1, 0)));
                }
        }
        // scores of the group (4 blocks x NT x 4, one TMEM load) -> z = log2 weight (<= 0)
        uint32_t zr[4 * NT * 4];
        tmem_ld_cols<4 * NT * 4>(tmem_w + (uint32_t)(b0 * NT * 4), zr);
        // e = 2^z issued at once; the group max zm (per head, over the 8 lanes of the head)
        // then scales e onto the 16-bit grid: P = round(e 2^-zm (2^16 - 2)). zm is clamped at
        // -100 (a group that far below the row max weighs < 2^-84 of it; also absent heads).
        const bool gfull = (b0 + 4) * 32 <= nv;  // warp-uniform: no per-token checks
        float e[4][NT][4], zm[NT];
#pragma unroll
        for (int hg = 0; hg < NT; ++hg) zm[hg] = -INFINITY;
        auto exps = [&](auto masked) {  // two instantiations: no per-token checks in full groups
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
#pragma unroll
                for (int hg = 0; hg < NT; ++hg)
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float zz = __fmaf_rn(__uint_as_float(zr[(bb * NT + hg) * 4 + j]), pa[hg], pb[hg]);
                        if constexpr (decltype(masked)::value) {
                            const int tok = (b0 + bb) * 32 + 16 * (j >> 1) + 8 * (j & 1) + g;
                            zz = tok < nv ? zz : -INFINITY;
                        }
                        zm[hg] = fmaxf(zm[hg], zz);
                        e[bb][hg][j] = ex2(zz);
                    }
        };
        if (gfull)
            exps(std::false_type{});
        else
            exps(std::true_type{});
        float sc[NT], up[NT];
        if constexpr (VTOK) {
            // token-wise V (out_c = sum_j p_j alpha_j + sum_j (p_j s_j) code_jc, s_j the token's
            // step): the IMMA weights are e_j s_j, normalised per group by their own maximum;
            // sum_j e_j and sum_j e_j alpha_j accumulate in fp32
            float gm[NT];
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) gm[hg] = 0.0f;
#pragma unroll
            for (int bb = 0; bb < 4; ++bb)
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float st = tso[bb][j].x;
#pragma unroll
                    for (int hg = 0; hg < NT; ++hg) {
                        const float ev = e[bb][hg][j];  // 0 for masked tokens
                        fw[hg] += ev;
                        if (st == 0.0f) fa[hg] = __fmaf_rn(ev, tso[bb][j].y, fa[hg]);  // a flat token: v = alpha
                        e[bb][hg][j] = ev * st;
                        gm[hg] = fmaxf(gm[hg], e[bb][hg][j]);
                    }
                }
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) {
                gm[hg] = fmaxf(gm[hg], __shfl_xor_sync(0xffffffffu, gm[hg], 4));
                gm[hg] = fmaxf(gm[hg], __shfl_xor_sync(0xffffffffu, gm[hg], 8));
                gm[hg] = fmaxf(gm[hg], __shfl_xor_sync(0xffffffffu, gm[hg], 16));
                up[hg] = gm[hg] > 0.0f ? __fdividef(65534.0f, gm[hg]) : 0.0f;
                sc[hg] = gm[hg] * (1.0f / 65534.0f);
            }
        } else {
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) {
                zm[hg] = fmaxf(zm[hg], __shfl_xor_sync(0xffffffffu, zm[hg], 4));
                zm[hg] = fmaxf(zm[hg], __shfl_xor_sync(0xffffffffu, zm[hg], 8));
                zm[hg] = fmaxf(zm[hg], __shfl_xor_sync(0xffffffffu, zm[hg], 16));
                zm[hg] = fmaxf(zm[hg], -100.0f);
                up[hg] = ex2(-zm[hg]) * 65534.0f;
                sc[hg] = ex2(zm[hg]) * (1.0f / 65534.0f);
            }
        }
        __syncwarp();  // the previous group's P tiles are consumed
        uint32_t wg[NT];
        float fo[NT];  // token-wise V: sum_j P_j o_j, o_j = alpha_j / s_j (the alpha term on the
                       // same integer weights as the codes: v_jc = s_j (code_jc + o_j))
#pragma unroll
        for (int hg = 0; hg < NT; ++hg) wg[hg] = 0u, fo[hg] = 0.0f;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            if (bb >= nbg) break;
            float oj[4];
            if constexpr (VTOK) {
#pragma unroll
                for (int j = 0; j < 4; ++j) oj[j] = tso[bb][j].x > 0.0f ? tso[bb][j].y : 0.0f;
            }
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) {
                uint32_t v[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)  // round(2^(z - zm) (2^16 - 2)) in the low mantissa bits
                    v[j] = __float_as_uint(__fmaf_rn(e[bb][hg][j], up[hg], kMagic));
                wg[hg] += (v[0] + v[1]) + (v[2] + v[3]) - 4u * 0x4B400000u;
                if constexpr (VTOK) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) fo[hg] = __fmaf_rn(__uint_as_float(v[j]) - kMagic, oj[j], fo[hg]);
                }
                const uint32_t p01 = prmt(v[0], v[1], 0x5140), p23 = prmt(v[2], v[3], 0x5140);
                uint32_t* tile = px + (bb * NT + hg) * kPxWords + t * kPxHead + g;
                tile[0] = prmt(p01, p23, 0x5410);  // plane 0: bits 0-7 of tokens g + 8 j
                tile[8] = prmt(p01, p23, 0x7632);  // plane 1: bits 8-15
            }
        }
        __syncwarp();
        int acc[NT][8][4];
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
            if (bb >= nbg) break;  // warp-uniform
            const int b = b0 + bb;
            const int i = nstage + b / kBps;  // V stage of this block
            const int slot = i % kStagesW;
            if (b % kBps == 0) mbar_wait(&full[slot], (i / kStagesW) & 1);
            const uint8_t* buf = ring + slot * Gm::kStageBytesB;
            uint32_t X[2][2 * BITS];  // [token half][word x]: channel rows x cpb + s, 4 tokens each
            {
                const uint4* xp = reinterpret_cast<const uint4*>(buf + (size_t)((b % kBps) * 32 + lane) * 16 * BITS);
#pragma unroll
                for (int u = 0; u < BITS; ++u) {
                    const uint4 v4 = xp[u];
                    const uint32_t w4[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) X[(4 * u + k) / (2 * BITS)][(4 * u + k) % (2 * BITS)] = w4[k];
                }
            }
            uint32_t bf[NT][2];
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) {
                const uint2 w2 = *reinterpret_cast<const uint2*>(px + (bb * NT + hg) * kPxWords + (g >> 1) * kPxHead +
                                                                 (g & 1) * 8 + 2 * t);
                bf[hg][0] = w2.x, bf[hg][1] = w2.y;
            }
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                const int rho0 = 2 * mt, rho1 = 2 * mt + 1;
                const uint32_t m0 = Gm::kMask << ((rho0 % cpb) * BITS), m1 = Gm::kMask << ((rho1 % cpb) * BITS);
                const uint32_t a0 = X[0][rho0 / cpb] & m0, a1 = X[0][rho1 / cpb] & m1;
                const uint32_t a2 = X[1][rho0 / cpb] & m0, a3 = X[1][rho1 / cpb] & m1;
#pragma unroll
                for (int hg = 0; hg < NT; ++hg) {
                    if (bb == 0) acc[hg][mt][0] = acc[hg][mt][1] = acc[hg][mt][2] = acc[hg][mt][3] = 0;
                    imma_u8u8(acc[hg][mt], a0, a1, a2, a3, bf[hg][0], bf[hg][1]);
                }
            }
            if (b % kBps == kBps - 1 || b == nblk_all - 1) {  // stage consumed: refill its slot
                __syncwarp();
                if (lane == 0 && i + kStagesW < total_stages) issue(i + kStagesW);
            }
        }
        // fold the group into fp32: column pair (2t, 2t+1) = planes 0 / 1 of head 4 hg + t
#pragma unroll
        for (int hg = 0; hg < NT; ++hg) {
#pragma unroll
            for (int mt = 0; mt < 8; ++mt) {
                const uint32_t c0 = (uint32_t)acc[hg][mt][0] + ((uint32_t)acc[hg][mt][1] << 8);
                const uint32_t c1 = (uint32_t)acc[hg][mt][2] + ((uint32_t)acc[hg][mt][3] << 8);
                fac[hg][2 * mt] = __fmaf_rn(__uint2float_rn(c0), sc[hg], fac[hg][2 * mt]);
                fac[hg][2 * mt + 1] = __fmaf_rn(__uint2float_rn(c1), sc[hg], fac[hg][2 * mt + 1]);
            }
            if constexpr (!VTOK) fw[hg] = __fmaf_rn(__uint2float_rn(wg[hg]), sc[hg], fw[hg]);
            if constexpr (VTOK) fa[hg] = __fmaf_rn(fo[hg], sc[hg], fa[hg]);
        }
    }

    if (lane == 0) TTRACE(16 + warp);  // phase B done, per warp
    if (p.late_trigger == 2) griddep_launch();
    // the output pass's first 16 fp32 tail V values of this thread's channel: loads go out
    // now, under the CTA reduction below
    constexpr int kTvv = 32;  // tail V rows in flight per thread (phase-B registers are free here)
    float tvv[kTvv];
    const float* vt = a.v_tail + (size_t)unit * a.tail_cap * kDim + (threadIdx.x & (kDim - 1));
#pragma unroll
    for (int u = 0; u < kTvv; ++u) tvv[u] = threadIdx.x < kDim && u < ntl ? __ldcg(vt + (size_t)u * kDim) : 0.0f;
    // ---------------- CTA reduction (fixed order, deterministic) ----------------
    // Image [warp][hg][rho][lane]: consecutive lanes hit consecutive banks.
#pragma unroll
    for (int hg = 0; hg < NT; ++hg) {
#pragma unroll
        for (int rho = 0; rho < 16; ++rho) sm.acc[((warp * NT + hg) * 16 + rho) * 32 + lane] = fac[hg][rho];
        float w = fw[hg];
        w += __shfl_xor_sync(0xffffffffu, w, 4);
        w += __shfl_xor_sync(0xffffffffu, w, 8);
        w += __shfl_xor_sync(0xffffffffu, w, 16);
        if (lane < 4) sm.wsum[warp * 16 + 4 * hg + lane] = w;
        if constexpr (VTOK) {
            float wa = fa[hg];
            wa += __shfl_xor_sync(0xffffffffu, wa, 4);
            wa += __shfl_xor_sync(0xffffffffu, wa, 8);
            wa += __shfl_xor_sync(0xffffffffu, wa, 16);
            if (lane < 4) sm.wsum[warp * 16 + 8 + 4 * hg + lane] = wa;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();  // (the V stream is drained: the ring is free from here on)
    if (threadIdx.x == 0) TTRACE(28);  // CTA image complete
    // Output, thread per (head, channel), from the per-warp images (unit weight scale):
    //   out = (s_c V / 2^sh + alpha_c W_vis + sum_t p_t v_tc) / (W_vis + sum_t p_t)
    // tail weights recomputed in fp32 (rank 0).
    float* recv = reinterpret_cast<float*>(sm.ring);
    if (S > 1) {  // every CTA's ring is drained before rank 0's becomes the receive buffer
        __syncwarp();
        cluster_arrive();  // #2a
        cluster_wait();
    }
    if (threadIdx.x < kDim) {  // thread = channel, all heads
        const int ch = threadIdx.x;
        const int mt = ch >> 4, r = (ch >> 3) & 1, gg = ch & 7, rho = 2 * mt + r;
        const float unshift = __int_as_float((127 - (rho % cpb) * BITS) << 23);  // divide out the slot's 2^sh
        constexpr float kInvLevelsV = 1.0f / (float)((1u << BITS) - 1u);
        const float v_step = fmaxf(__fsub_rn(v_b, v_a) * kInvLevelsV, 0.0f);
        float num[HB], den[HB];
#pragma unroll
        for (int h = 0; h < HB; ++h) {
            float V = 0.0f, wv = 0.0f, wa = 0.0f;
            if (h < G) {
                for (int w2 = 0; w2 < W; ++w2) {
                    V += sm.acc[((w2 * NT + (h >> 2)) * 16 + rho) * 32 + 4 * gg + (h & 3)];
                    wv += sm.wsum[w2 * 16 + h];
                    if constexpr (VTOK) wa += sm.wsum[w2 * 16 + 8 + h];
                }
            }
            // channel-wise V: s_c V / 2^sh + alpha_c W; token-wise V: the per-token steps are in
            // the weights (V / 2^sh) and the alphas in wa
            num[h] = VTOK ? V * unshift + wa : __fmaf_rn(v_step, V * unshift, v_a * wv);
            den[h] = wv;
        }
        // fp32 tail (naive_wv kernels.hpp:414-426): each row value loaded once for all heads,
        // 16 loads in flight; weights precomputed in tail_s
        for (int j0 = 0; j0 < ntl; j0 += kTvv) {
            float vv[kTvv];
#pragma unroll
            for (int u = 0; u < kTvv; ++u)
                vv[u] = j0 == 0 ? tvv[u] : j0 + u < ntl ? __ldcg(vt + (size_t)(j0 + u) * kDim) : 0.0f;
#pragma unroll
            for (int u = 0; u < kTvv; ++u) {
                if (j0 + u >= ntl) break;
#pragma unroll
                for (int h = 0; h < HB; ++h) {
                    if (h < G) {
                        const float pt = sm.tail_s[h * kTailMax + j0 + u];
                        den[h] += pt;
                        num[h] = __fmaf_rn(pt, vv[u], num[h]);
                    }
                }
            }
        }
        if (threadIdx.x == 0) TTRACE(29);  // output sums done (thread 0)
#pragma unroll
        for (int h = 0; h < HB; ++h) {
            if (h >= G) break;
            if (S == 1) {
                a.out[qrow(h) * kDim + ch] = num[h] / den[h];
                if (a.tail_lse && ch == 0) a.tail_lse[qrow(h)] = log2f(den[h]) - sm.gpar[h * 4 + 2];
            } else {
                st_cluster_f32(recv + rank * (8 * kDim + 8) + h * kDim + ch, 0, num[h]);
                if (ch == 0) st_cluster_f32(recv + rank * (8 * kDim + 8) + 8 * kDim + h, 0, den[h]);
            }
        }
    }
    if (S > 1) {
        __syncwarp();
        cluster_arrive();  // #2b: partial numerators / denominators are in rank 0
        cluster_wait();
        if (rank == 0) {
            for (int idx = threadIdx.x; idx < G * kDim; idx += W * 32) {
                const int h = idx / kDim;
                float num = 0.f, den = 0.f;
                for (int r = 0; r < S; ++r) {
                    num += recv[r * (8 * kDim + 8) + idx];
                    den += recv[r * (8 * kDim + 8) + 8 * kDim + h];
                }
                a.out[qrow(idx / kDim) * kDim + (idx % kDim)] = num / den;
                if (a.tail_lse && idx % kDim == 0)
                    a.tail_lse[qrow(h)] = log2f(den) - sm.gpar[h * 4 + 2];
            }
        }
    }
    if (threadIdx.x == 0) TTRACE(5);
    if (append_rows && warp == 0) {
        asm volatile("cp.async.wait_all;" ::: "memory");
        const size_t dst = ((size_t)unit * a.tail_cap + ntl) * kDim + 4 * lane;
        *reinterpret_cast<float4*>(const_cast<float*>(a.k_tail) + dst) = *reinterpret_cast<const float4*>(sm.arow + 4 * lane);
        *reinterpret_cast<float4*>(const_cast<float*>(a.v_tail) + dst) =
            *reinterpret_cast<const float4*>(sm.arow + kDim + 4 * lane);
    }
    if (cnt_old == (int)a.kv_heads * p.groups - 1) {  // the request's last tail owner
        const int req = unit / (int)a.kv_heads;
        a.append_cnt[req] = 0;
        if (ntl < (int)a.tail_cap)
            const_cast<int*>(a.tail_len)[req] = ntl + 1;
        else
            atomicOr(a.overflow, 1);
    }
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(kTmemCols));
    }
    if (a.dep_wait_at_end) griddep_wait();
}

// Token split: at most 8192 (NT = 1) / 4096 tokens per CTA; small batches split units further (down to
// 256 tokens per CTA) so that units x S covers the SMs - a single unit otherwise runs on
// one SM for its full latency.
void plan(const DecodeArgs& a, int NT, int& S, int& T, int W = kWarps) {
    const int n = (int)a.n_vis;
    const int ct = cta_tokens(NT, W);
    int s_min = std::max(1, (n + ct - 1) / ct);
    size_t pu = a.plan_units ? a.plan_units : a.units;  // a chunk plans as its whole batch
    if (NT == 1 && a.group > 4) pu *= 2;                 // two head-group CTAs per unit
    // split a unit only while the units leave CTA slots empty: fill the slots of one wave
    // (2 x 148 for 8-warp CTAs), never more (round 2, c5 B = 8 = 64 units: S = 4 12.6 us vs
    // S = 2 13.6 us vs S = 1 14.7 us; round 1 aimed at one CTA per SM,
    // profiles/r01_tc_split2.txt). (Also measured in round 2 and dropped: the fp32 tail scores
    // before phase A with their rows preloaded under the q fold, and every warp computing the
    // softmax parameters itself instead of two more CTA barriers - C2 32.96 -> 34.24 / 33.68 us.)
    const int slots = (W == 4 ? 4 : 2) * 148;
    const int want = std::max(1, (int)(slots / pu));
    int s = std::max(s_min, std::min(want, kMaxCluster));
    static const int force = std::getenv("KVQ_TC_SPLIT") ? std::atoi(std::getenv("KVQ_TC_SPLIT")) : 0;  // tuning
    if (force > 0) s = std::max(s_min, std::min(force, kMaxCluster));
    if (a.split_override > 0) s = std::max(s_min, std::min(a.split_override, kMaxCluster));
    s = std::min(s, std::max(1, (n + 255) / 256));
    T = ((n + s - 1) / s + 255) / 256 * 256;  // multiple of 8 warps x 32 tokens (and of 4 x 32)
    S = (n + T - 1) / T;
}

template <int BITS, int NT, int OCC, int W = kWarps, bool VTOK = false>
cudaError_t launch_occ(const DecodeArgs& a, cudaStream_t s, int groups = 1, int whole = 0) {
    int S, T, S1 = 1, T1 = 0;
    if (whole > 0) {  // mixed: solo whole units, then 2-CTA clusters of half units
        DecodeArgs a1 = a, a2 = a;
        a1.split_override = 1, a2.split_override = 2;
        plan(a1, NT, S1, T1, W);
        plan(a2, NT, S, T, W);
        if (S1 != 1 || S != 2) return cudaErrorInvalidValue;
    } else {
        plan(a, NT, S, T, W);
    }
    cudaError_t e = cudaSuccess;
    static const int split_first = std::getenv("KVQ_TC_SPLIT_FIRST") ? std::atoi(std::getenv("KVQ_TC_SPLIT_FIRST")) : 0;
    // Dependents are released late (phase B), so the next grid's CTAs are placed once this
    // grid's slots drain: released right after the dependency wait, they
    // land on the SMs that finish first and stack four whole units there (c2: 40 SMs with
    // 4.0 units instead of 3.5, profiles/r02_decode_c2.md). Early release (0) where a
    // dependent must overlap this grid: the fp32 tail pass, a sibling balancing grid.
    // Default: at the start of phase B (3) - the next grid's CTAs fill the slots of lightly
    // loaded SMs sooner (C3 b1 35.5 -> 34.7 us, b2 37.2 -> 36.5) - except for the balanced
    // 4-warp launch (whole units + half-unit clusters, 3.5 units per SM), whose placement
    // only stays even with the release after phase B (2; C2 33.2 vs 35.4 us).
    static const int trig_env = std::getenv("KVQ_TC_TRIGGER") ? std::atoi(std::getenv("KVQ_TC_TRIGGER")) : -1;
    const int late = a.early_trigger || a.tail_lse ? 0 : trig_env >= 0 ? trig_env : (whole > 0 ? 2 : 3);
    TcParams p{a, S, T, groups, whole, T1, split_first, late};
    // TMEM: 512 columns per SM; never let more CTAs share an SM than TMEM can serve (a
    // blocked tcgen05.alloc inside a cluster could deadlock against its partners).
    const size_t max_ctas = W == 4 ? 4 : (OCC == 1 ? 1 : 2);
    size_t smem = tc_smem_bytes<BITS, NT, OCC, W>(S);
    const size_t floor_bytes = 232448 / (max_ctas + 1) + 1;
    if (smem < floor_bytes) smem = floor_bytes;
    auto kern = decode_tc_kernel<BITS, NT, OCC, W, VTOK>;
    static unsigned attr_done = 0;  // per instantiation, bit per device
    e = once_per_device(attr_done, [&] {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return r != cudaSuccess ? r : cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    });
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(whole > 0 ? (unsigned)(whole + 2 * (a.units - whole)) : (unsigned)(a.units * S * groups));
    cfg.blockDim = dim3(W * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;  // (S = 1 grids launch as fast without it,
    attrs[0].val.clusterDim.x = (unsigned)S;            //  measured: c3b1 35.50 vs 35.51 us)
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = 2;
    e = cudaLaunchKernelEx(&cfg, kern, p);
    note_launch();
    return e;
}

}  // namespace

// ---- vx_layout: V codes pre-arranged as the phase-B A operand (V^T registers) ------------
// [unit][32-token block][lane 32][half 2][2*BITS words]: byte j of word (half, x) of lane
// (g, t) holds, in slot s (bits [s BITS, s BITS + BITS)), the code of token
// 2 t + half + 8 j of the block and channel 16 mt + 8 r + g, where rho = x cpb + s = 2 mt + r
// - one LOP3 then yields the A register "4 tokens of channel row g (+8) of tile mt, x 2^(s
// BITS)". Tokens past n are zero codes. Built once per cache (pack_vx_kernel); the
// reference-layout copy stays for read-back.
namespace {
constexpr int kVxWarps = 4;  // 32-token blocks per CTA (one warp each)

// Both layout kernels stage one 32-token block per warp in shared memory (coalesced 16-byte
// global accesses on both sides) and move codes between the two layouts there. (Round 1
// read and wrote single bytes from global memory: C2 82 us, C3 b4 208 us for pack, 1.07 ms
// for unpack.)
template <int BITS>
__global__ void __launch_bounds__(kVxWarps * 32) pack_vx_kernel(const uint8_t* __restrict__ rows, size_t n,
                                                                 size_t nb32, int bx, uint8_t* __restrict__ vx) {
    constexpr int kRowBytes = 16 * BITS;
    constexpr int cpb = 8 / BITS;
    constexpr uint32_t kLevel = (1u << BITS) - 1u;
    __shared__ __align__(16) uint8_t srow[kVxWarps][32 * kRowBytes];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
    const size_t unit = blockIdx.y, blk = (size_t)blockIdx.x * kVxWarps + warp;
    if (blk >= nb32) return;
    uint8_t* sr = srow[warp];
    // the block's rows (tokens past n: zero codes), 16 bytes per lane per pass
    const uint8_t* src = rows + (unit * n + blk * 32) * kRowBytes;
    const size_t valid = min((size_t)32, n - blk * 32) * kRowBytes;
#pragma unroll
    for (int o = lane * 16; o < 32 * kRowBytes; o += 32 * 16) {
        uint4 v = make_uint4(0, 0, 0, 0);
        if ((size_t)o < valid) v = *reinterpret_cast<const uint4*>(src + o);
        *reinterpret_cast<uint4*>(sr + o) = v;
    }
    __syncwarp();
    uint32_t w[2 * 2 * BITS];  // [half][x]
#pragma unroll
    for (int half = 0; half < 2; ++half)
#pragma unroll
        for (int x = 0; x < 2 * BITS; ++x) {
            uint32_t word = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint8_t* rp = sr + (2 * t + half + 8 * j) * kRowBytes;
#pragma unroll
                for (int sl = 0; sl < cpb; ++sl) {
                    const int rho = x * cpb + sl, c = 16 * (rho >> 1) + 8 * (rho & 1) + g;
                    const int i = c % cpb;  // MSB-first code slot in its byte (bitpack.hpp:76-88)
                    const uint32_t code = ((uint32_t)rp[(c / cpb) ^ bx] >> (8 - BITS * (i + 1))) & kLevel;
                    word |= code << (8 * j + BITS * sl);
                }
            }
            w[half * 2 * BITS + x] = word;
        }
    uint4* dst = reinterpret_cast<uint4*>(vx + ((unit * nb32 + blk) * 32 + lane) * (size_t)(16 * BITS));
#pragma unroll
    for (int q = 0; q < BITS; ++q) dst[q] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

}  // namespace

// Inverse of pack_vx_kernel: the reference rows (bitpack.hpp:64-90, M-bit words via the byte
// fold) of every token, for read-back, snapshots and the generic path when V is resident
// only in the operand layout. Warp per 32-token block; lane = token of the block.
namespace {
template <int BITS>
__global__ void __launch_bounds__(kVxWarps * 32) unpack_vx_kernel(const uint8_t* __restrict__ vx, size_t n,
                                                                   size_t nb32, int bx, uint8_t* __restrict__ rows) {
    constexpr int kRowBytes = 16 * BITS;
    constexpr int cpb = 8 / BITS;
    constexpr uint32_t kLevel = (1u << BITS) - 1u;
    __shared__ __align__(16) uint32_t sw[kVxWarps][32 * 4 * BITS];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t unit = blockIdx.y, blk = (size_t)blockIdx.x * kVxWarps + warp;
    if (blk >= nb32) return;
    uint32_t* ws = sw[warp];
    const uint4* src = reinterpret_cast<const uint4*>(vx + (unit * nb32 + blk) * 32 * (size_t)(16 * BITS));
#pragma unroll
    for (int q = 0; q < BITS; ++q) reinterpret_cast<uint4*>(ws)[q * 32 + lane] = src[q * 32 + lane];
    __syncwarp();
    const size_t tok = blk * 32 + lane;
    const int ti = lane;  // token 2 t + half + 8 j of the block
    const int j = ti >> 3, t = (ti & 7) >> 1, half = ti & 1;
    // the row in M = 8 byte order (compile-time register indices), then each 32-bit word's
    // bytes permuted for M = 16 / 32 (byte k of the row is byte k ^ bx of the M = 8 row)
    uint32_t rw[kRowBytes / 4];
#pragma unroll
    for (int k = 0; k < kRowBytes / 4; ++k) rw[k] = 0;
#pragma unroll
    for (int c = 0; c < 128; ++c) {
        const int rho = 2 * (c >> 4) + ((c >> 3) & 1), ln = 4 * (c & 7) + t;
        const int x = rho / cpb, sl = rho % cpb;
        const uint32_t word = ws[ln * 4 * BITS + half * 2 * BITS + x];
        const uint32_t code = (word >> (8 * j + BITS * sl)) & kLevel;
        const int i = c % cpb, q = c / cpb;
        rw[q >> 2] |= code << (8 * (q & 3) + 8 - BITS * (i + 1));
    }
    if (tok >= n) return;
    const uint32_t sel = bx == 0 ? 0x3210u : (bx == 1 ? 0x2301u : 0x0123u);
    uint8_t* dst = rows + (unit * n + tok) * kRowBytes;
#pragma unroll
    for (int k = 0; k < kRowBytes / 4; k += 4)
        *reinterpret_cast<uint4*>(dst + 4 * k) = make_uint4(__byte_perm(rw[k], 0, sel), __byte_perm(rw[k + 1], 0, sel),
                                                            __byte_perm(rw[k + 2], 0, sel), __byte_perm(rw[k + 3], 0, sel));
}
}  // namespace

cudaError_t launch_unpack_vx(const uint8_t* vx, size_t units, size_t n_vis, int bits, int word_bits, uint8_t* rows,
                             cudaStream_t s) {
    if (n_vis == 0 || units == 0) return cudaSuccess;
    const size_t nb32 = (n_vis + 31) / 32;
    dim3 grid((unsigned)((nb32 + kVxWarps - 1) / kVxWarps), (unsigned)units);
    const int bx = word_bits / 8 - 1;
    switch (bits) {
        case 1: unpack_vx_kernel<1><<<grid, kVxWarps * 32, 0, s>>>(vx, n_vis, nb32, bx, rows); break;
        case 2: unpack_vx_kernel<2><<<grid, kVxWarps * 32, 0, s>>>(vx, n_vis, nb32, bx, rows); break;
        case 4: unpack_vx_kernel<4><<<grid, kVxWarps * 32, 0, s>>>(vx, n_vis, nb32, bx, rows); break;
        case 8: unpack_vx_kernel<8><<<grid, kVxWarps * 32, 0, s>>>(vx, n_vis, nb32, bx, rows); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

size_t vx_bytes(size_t units, size_t n_vis, int bits) { return units * ((n_vis + 31) / 32) * 32 * 16 * (size_t)bits; }

cudaError_t launch_pack_vx(const uint8_t* rows, size_t units, size_t n_vis, int bits, int word_bits, uint8_t* vx,
                           cudaStream_t s) {
    if (n_vis == 0 || units == 0) return cudaSuccess;
    const size_t nb32 = (n_vis + 31) / 32;
    dim3 grid((unsigned)((nb32 + kVxWarps - 1) / kVxWarps), (unsigned)units);
    // M = 16 / 32 rows are M = 8 rows with the bytes of each LE word reversed
    // (bitpack.hpp:85: code i of a word at bit M - N(i+1)): read byte k ^ (M/8 - 1).
    const int bx = word_bits / 8 - 1;
    switch (bits) {
        case 1: pack_vx_kernel<1><<<grid, kVxWarps * 32, 0, s>>>(rows, n_vis, nb32, bx, vx); break;
        case 2: pack_vx_kernel<2><<<grid, kVxWarps * 32, 0, s>>>(rows, n_vis, nb32, bx, vx); break;
        case 4: pack_vx_kernel<4><<<grid, kVxWarps * 32, 0, s>>>(rows, n_vis, nb32, bx, vx); break;
        case 8: pack_vx_kernel<8><<<grid, kVxWarps * 32, 0, s>>>(rows, n_vis, nb32, bx, vx); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

size_t decode_tc_scratch_bytes(size_t units) { return units * (2 * 512 * sizeof(uint32_t) + 8 * sizeof(float2)); }

// CTAs per SM the kernel is built for (register bound + ring depth): 2 by default,
// KVQ_TC_OCC=3 selects the 3-CTA variant (fewer registers, shallower ring).
// CTA shape: 8 warps, two CTAs per SM; or 4 warps, four per SM (up to 1024 tokens per warp,
// 128 TMEM columns per CTA). Many short units favour 4-warp CTAs - all of C2's 512 units are
// resident at once instead of in 1.73 waves (56.0 -> 50.4 us; C5 B=512 342 -> 287 us) -
// while fewer or longer units favour 8 warps (C3: a 4-warp CTA would need a 2-CTA cluster,
// 48 -> 52 us; profiles/r01_tc_w4.txt). KVQ_TC_W4=0/1 forces either (tuning).
static bool tc_w4(const DecodeArgs& a) {
    static const char* env = std::getenv("KVQ_TC_W4");
    if (env) return std::atoi(env) != 0;
    size_t pu = a.plan_units ? a.plan_units : a.units;
    if (a.group > 4) pu *= 2;
    // long units (n > 8192) run in several rounds of CTAs either way: the 4-warp shape
    // keeps more, smaller CTAs in flight (C4 137.5 -> 131.3 us; C3's 8192-token units stay
    // 8-warp: 35.8 vs 39.6 us, profiles/r02_configs.md)
    return (pu > 2 * 148 && a.n_vis <= (size_t)cta_tokens(1, 4)) || a.n_vis > (size_t)cta_tokens(1, 8);
}

static int tc_occ() {
    static int occ = [] {
        const char* e = std::getenv("KVQ_TC_OCC");
        return e && e[0] == '3' ? 3 : 2;
    }();
    return occ;
}

// G > 4 (two head groups) needs ~180 registers: one CTA per SM, no spills.
template <int BITS, int NT>
cudaError_t launch_bits(const DecodeArgs& a, cudaStream_t s, int whole = 0) {
    if constexpr (NT == 2) {
        if (a.v_token_wise) return cudaErrorNotSupported;  // (token-wise V: head-split CTAs only)
        return launch_occ<BITS, NT, 1>(a, s);
    } else {
        // G > 4 at NT = 1: two head groups as separate CTAs (two CTAs per SM each)
        const int groups = a.group > 4 ? 2 : 1;
        if (a.v_token_wise)  // (opt-in token-wise V: the default occupancy variants only)
            return tc_w4(a) ? launch_occ<BITS, NT, 4, 4, true>(a, s, groups, whole)
                            : launch_occ<BITS, NT, 2, kWarps, true>(a, s, groups);
        if (tc_w4(a)) return launch_occ<BITS, NT, 4, 4>(a, s, groups, whole);
        return tc_occ() == 3 ? launch_occ<BITS, NT, 3>(a, s, groups) : launch_occ<BITS, NT, 2>(a, s, groups);
    }
}

// G > 4: two CTAs of one head group each (NT = 1, two CTAs per SM, codes streamed twice)
// beat one CTA holding both groups (NT = 2, ~226 registers, one CTA per SM, codes streamed
// once): C4 (G = 6) 246 -> 202 us per step, G = 8 at C2 shape 90 -> 77 us
// (profiles/r01_tc_headsplit.txt). KVQ_TC_HEADSPLIT=0 selects NT = 2 (tuning).
int tc_nt(const DecodeArgs& a) {
    if (a.group <= 4) return 1;
    static const char* env = std::getenv("KVQ_TC_HEADSPLIT");
    const bool split = env ? std::atoi(env) != 0 : true;
    return split ? 1 : 2;
}

template <int BITS, int NT>
static size_t tc_smem_for(const DecodeArgs& a, int S) {
    if constexpr (NT == 2) {
        return tc_smem_bytes<BITS, NT, 1>(S);
    } else if (tc_w4(a)) {
        return tc_smem_bytes<BITS, NT, 4, 4>(S);
    } else {
        return tc_occ() == 3 ? tc_smem_bytes<BITS, NT, 3>(S) : tc_smem_bytes<BITS, NT, 2>(S);
    }
}

bool decode_tc_supported(const DecodeArgs& a) {
    if (a.dim != (size_t)kDim || a.n_vis == 0 || !a.v_codes_x) return false;
    if (a.word_bits != 8 && a.word_bits != 16 && a.word_bits != 32) return false;
    if (a.bits != 1 && a.bits != 2 && a.bits != 4 && a.bits != 8) return false;
    if (a.group < 1 || a.group > 8) return false;
    if (a.units == 0) return false;
    int S, T;
    const int NT = tc_nt(a);
    plan(a, NT, S, T, NT == 1 && tc_w4(a) ? 4 : kWarps);
    if (S > kMaxCluster) return false;
    // the fp32 tail lives in rank 0 (at most kTailMax rows) unless the tail pass owns it
    if (a.tail_cap > (size_t)kTailMax && a.tail_lse == nullptr) return false;
    (void)T;
    size_t smem = 0;
    switch (a.bits * 10 + NT) {
        case 11: smem = tc_smem_for<1, 1>(a, S); break;
        case 12: smem = tc_smem_for<1, 2>(a, S); break;
        case 21: smem = tc_smem_for<2, 1>(a, S); break;
        case 22: smem = tc_smem_for<2, 2>(a, S); break;
        case 41: smem = tc_smem_for<4, 1>(a, S); break;
        case 42: smem = tc_smem_for<4, 2>(a, S); break;
        case 81: smem = tc_smem_for<8, 1>(a, S); break;
        case 82: smem = tc_smem_for<8, 2>(a, S); break;
    }
    return smem <= 220 * 1024;
}

// Units [u0, u1) of `a` (every per-unit array is unit-major; u0 on a request boundary).
static DecodeArgs unit_range(const DecodeArgs& a, size_t u0, size_t u1) {
    DecodeArgs r = a;
    const size_t rb = row_bytes(a.dim, a.bits, a.word_bits), d = a.dim, G = a.group;
    r.k_codes += u0 * a.n_vis * rb;
    if (r.v_codes) r.v_codes += u0 * a.n_vis * rb;
    if (r.v_codes_x) r.v_codes_x += vx_bytes(u0, a.n_vis, a.bits);
    const size_t vs = a.v_token_wise ? a.n_vis : d;  // V stats per unit: per channel or per token
    r.k_alpha += u0 * d, r.k_beta += u0 * d, r.v_alpha += u0 * vs, r.v_beta += u0 * vs;
    if (r.v_tok_so) r.v_tok_so += u0 * a.n_vis;
    r.k_tail += u0 * a.tail_cap * d, r.v_tail += u0 * a.tail_cap * d;
    r.tail_len += u0 / a.kv_heads;
    if (r.k_new) r.k_new += u0 * d, r.v_new += u0 * d, r.append_cnt += u0 / a.kv_heads;
    r.q += u0 * G * d, r.out += u0 * G * d;
    if (r.tail_lse) r.tail_lse += u0 * G;
    r.units = u1 - u0;
    return r;
}

static cudaError_t launch_nt(const DecodeArgs& a, int NT, cudaStream_t s, int whole = 0);

// 4-warp CTAs (four slots per SM) with k whole units per SM plus a remainder r: the SMs
// holding k + 1 whole units set the makespan. The r remainder units are instead cut in
// halves (2-CTA clusters) and launched right behind (programmatic dependent launch) into
// the free slots, when they fit (148 k + 2 r <= 592): every SM carries at most k + 1/2.
// Returns how many of the batch's last units are split (0: no balancing). Decided on the
// whole batch (plan_units), so chunked launches split exactly the same units.
static size_t balance_w4(const DecodeArgs& a) {
    static const char* env = std::getenv("KVQ_TC_BALANCE");
    if (env && std::atoi(env) == 0) return 0;
    const size_t units = a.plan_units ? a.plan_units : a.units;
    if (a.group > 4 || a.split_override || a.n_vis < 2 * 256 || !tc_w4(a)) return 0;
    const size_t k = units / 148;
    size_t r = units - 148 * k;
    r = (r + a.kv_heads - 1) / a.kv_heads * a.kv_heads;  // whole requests
    // measured (profiles/r01_tc_balance.txt): a gain while the remainder is at most half an
    // SM row (r <= 74: 320 units 40.6 -> 38.4 us, 512 units 48.1 -> 45.2 us), a loss beyond
    // (384 and 432 units), where the extra launch and cluster merges outweigh the rebalance
    if (k < 2 || r == 0 || 2 * r > 148 || 148 * k + 2 * r > 4 * 148) return 0;
    return r;
}

// (Tried and dropped: the analogous mixed launch for 8-warp batches of 149-296 units -
// 8-warp whole units plus 4-warp half-unit clusters sharing SMs - was 5-18 % slower,
// profiles/r01_tc_balance.txt.)
cudaError_t launch_decode_tc(const DecodeArgs& a, cudaStream_t s) {
    if (const size_t nsplit = balance_w4(a)) {
        const size_t total = a.plan_units ? a.plan_units : a.units;
        // this launch covers batch units [unit_base, unit_base + units); split from `first`
        const size_t first = total - nsplit;
        const size_t cut = first <= a.unit_base ? 0 : std::min(a.units, first - a.unit_base);
        if (cut > 0 && cut < a.units && cut % 2 == 0 && !std::getenv("KVQ_TC_TWO_LAUNCH")) {
            // one launch: `cut` solo CTAs, then 2-CTA clusters of half units (uniform cluster
            // dimension 2: consecutive solo CTAs pair up as independent cluster mates)
            DecodeArgs M = a;
            M.plan_units = total;
            return launch_nt(M, 1, s, (int)cut);
        }
        DecodeArgs A = unit_range(a, 0, cut), B = unit_range(a, cut, a.units);
        A.plan_units = B.plan_units = total;  // same CTA shape for both
        B.unit_base = a.unit_base + cut;
        B.split_override = 2;
        if (cut > 0) {
            A.early_trigger = 1;  // B overlaps A
            cudaError_t e = launch_nt(A, 1, s);
            if (e != cudaSuccess || cut == a.units) return e;
            B.dep_wait_at_end = 1;  // launched behind A (see the kernel's dependency wait)
            if (B.trace) B.trace += cut * 256;  // debug timelines: A's CTAs first, then B's
        }
        return launch_nt(B, 1, s);
    }
    return launch_nt(a, tc_nt(a), s);
}

static cudaError_t launch_nt(const DecodeArgs& a, int NT, cudaStream_t s, int whole) {
    if (whole > 0 && NT != 1) return cudaErrorInvalidValue;
    switch (a.bits * 10 + NT) {
        case 11: return launch_bits<1, 1>(a, s, whole);
        case 12: return launch_bits<1, 2>(a, s);
        case 21: return launch_bits<2, 1>(a, s, whole);
        case 22: return launch_bits<2, 2>(a, s);
        case 41: return launch_bits<4, 1>(a, s, whole);
        case 42: return launch_bits<4, 2>(a, s);
        case 81: return launch_bits<8, 1>(a, s, whole);
        case 82: return launch_bits<8, 2>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace kvqb
