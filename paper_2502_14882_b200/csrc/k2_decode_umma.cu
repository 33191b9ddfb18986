// k2_decode_umma.cu — K2 throughput path on the 5th-generation tensor cores: fused,
// calibrated, post-scaled quantized decode attention with tcgen05.mma kind::i8
// (UTCIMMA), operands staged in tensor memory, accumulators in tensor memory.
// d = 128, reference M = 8 byte layout for K, b in {1,2,4,8}, G <= 8.
//
// Math (reference: kernels.hpp:14-26, 183-194, 277-283; calibrate.hpp:62-114;
// kvcache.hpp:263-311), per (unit, query head h):
//   score_j = (sum_c qs_c code_jc + q.alpha) / sqrt(d),   qs_c = q_c (beta_c - alpha_c) / L
//   row     = [g(score_vis) | score_tail],   g affine from (gamma, delta) of the vis part
//   out_c   = (s_c sum_j p_j code_jc + alpha_c sum_j p_j + sum_t p_t v_tc) / sum p
// Packed K/V are never dequantized: codes enter the tensor core as raw bytes.
//
// One CTA = 4 warps = 128 threads = the 128 TMEM lanes. A unit (request, KV head) of n
// visual tokens is split over a cluster of S CTAs (contiguous token ranges); blocks of
// 128 tokens stream through a TMA (cp.async.bulk) ring: the unit's K blocks, then its
// V blocks.
//
// Phase A (scores), per 128-token K block: thread m = token m expands its packed row
//   into 32 registers of u8 codes with one LOP3 each (byte = code << s*b, the code's
//   bit slot) and tcgen05.st's them into TMEM (A operand, lane m = row m). One elected
//   thread issues 4 x UTCIMMA M128 N16 K32: D[128 tok][4 heads x 4 digit planes] +=
//   A[tok][ch] * Q[ch][head, plane], Q = the query with the K scales folded in, split in
//   4 signed base-256 digit planes (exact int32 score). The epilogue (tcgen05.ld) turns
//   the digit planes into fp32 scores, kept on chip (shared memory), with per-head
//   min/max.
// Calibration: CTA + cluster (DSMEM) reduction of (min, max, tail max) per head -> the
//   affine g and the softmax offset, identical in every CTA of the unit.
// Phase B (p.V), per 128-token V block, from the token-packed V layout (vt_layout
//   below): thread c = channel c expands its 128 tokens' codes (one LOP3 per 4 tokens)
//   into TMEM; thread m = token m writes p_m = exp2(g(s) - m) as a 32-bit integer (4 u8
//   planes, pre-divided by the code's 2^(s*b) slot scale) into a shared-memory B tile.
//   4 x UTCIMMA M128 N16 K32 accumulate D[128 ch][4 heads x 4 planes] in TMEM across
//   every block of the CTA. Epilogue: out = (s_c D / 2^31 + alpha_c W + tail) / (W + tail).
#include <cooperative_groups.h>

#include "kvq_internal.cuh"
#include "kvq_ptx.cuh"

namespace cg = cooperative_groups;

namespace kvqb {

namespace {

constexpr int kDim = 128;
constexpr int kThreads = 128;
constexpr int kBlk = 128;  // tokens per block
constexpr int kTailMax = 64;
constexpr int kMaxCluster = 16;
constexpr float kLog2e = 1.4426950408889634f;

template <int BITS, int NT>
struct UGeo {
    static constexpr int kRowBytes = 16 * BITS;           // packed K row / V^T channel slice
    static constexpr int kBlockBytes = kBlk * kRowBytes;  // one ring stage
    static constexpr int kCpb = 8 / BITS;                 // codes per byte
    static constexpr uint32_t kMask = 0x01010101u * ((1u << BITS) - 1u);
    static constexpr int kN = 16 * NT;  // MMA N = 4 digit planes x 4 heads per head group
    static constexpr int kHeads = 4 * NT;
    // A deep ring (64 KB): the unit's K/V stream is the only HBM traffic, and ~2 us of
    // bulk-copy latency under load must be covered by bytes in flight.
    static constexpr int kStages = 32 / BITS;
    static constexpr uint32_t kTmemCols = 256;  // two CTAs per SM
    // TMEM columns: NA A-operand buffers (32 columns = 128 K-bytes each), ND phase-A
    // accumulators (kN columns each; the phase-B accumulator reuses the first), then the
    // fp32 scores of the CTA's tokens (kHeads columns per 128-token block, lane = token).
    static constexpr int kNA = NT == 1 ? 3 : 2;
    static constexpr int kND = 2;
    static constexpr uint32_t kColA = 0;
    static constexpr uint32_t kColDA = 32 * kNA;
    static constexpr uint32_t kColDV = kColDA;
    static constexpr uint32_t kColS = 128;
    static constexpr int kMaxTokens = (kTmemCols - kColS) / kHeads * kBlk;  // 4096 (G <= 4) / 2048
    static_assert(kColDA + kND * kN <= kColS, "TMEM budget");
};

struct UParams {
    DecodeArgs a;
    const uint8_t* qb;     // [units][128 rows][16 NT] s8 digit planes (MN-major B tile)
    const float2* qconst;  // [units][8] (isd / S_h, qdota_h * isd)
    int S, T;              // cluster size, tokens per CTA (multiple of 128)
};

// ---- PTX helpers (mbarriers, bulk copies, cluster barriers, PDL: kvq_ptx.cuh) ---------
// Waits here may legitimately be long (the MMA warp waits on whole stages): mbarrier polls
// trap after 2^28 instead of 2^24.
using namespace ptx;
template <typename... A>
__device__ __forceinline__ void mbar_wait_long(A... a) { ptx::mbar_wait<28>(a...); }
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile(
        "{\n .reg .b32 r;\n .reg .pred p;\n elect.sync r|p, 0xffffffff;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(pred));
    return pred != 0;
}

// Debug timeline (KVQ_TRACE_FILE): slot k of this CTA's 256-entry record. Per-block
// stamps (BTRACE) only exist in a -DKVQ_TRACE_BLOCKS build.
#define UTRACE(k)                                                                          \
    do {                                                                                   \
        if (a.trace) a.trace[(size_t)blockIdx.x * 256 + (k)] = gtimer();                   \
    } while (0)
#ifdef KVQ_TRACE_BLOCKS
#define BTRACE(k) UTRACE(k)
#else
#define BTRACE(k) \
    do {          \
    } while (0)
#endif

// tcgen05 -----------------------------------------------------------------------------
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 32 lanes x 32 consecutive columns: thread t of the warp writes lane (warp quarter, t).
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
        "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
        "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
        "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
        : "memory");
}
template <int H>
__device__ __forceinline__ void tmem_st_scores(uint32_t taddr, const uint32_t (&r)[H]) {
    if constexpr (H == 4) {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(taddr), "r"(r[0]), "r"(r[1]),
                     "r"(r[2]), "r"(r[3])
                     : "memory");
    } else {
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                     "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                     : "memory");
    }
}
template <int H>
__device__ __forceinline__ void tmem_ld_scores(uint32_t taddr, uint32_t (&r)[H]) {
    if constexpr (H == 4) {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                     : "r"(taddr));
    } else {
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                     : "r"(taddr));
    }
}
__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

// Shared-memory matrix descriptor: no swizzle, canonical MN-major layout of 8-bit
// elements with rows of 16 bytes (LBO = 128 B between 8-row groups along K, SBO =
// byte stride between 16-column groups along N). Probe: tools/microbench/umma_i8_test.cu.
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr, uint32_t sbo) {
    uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)(128u >> 4) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // sm100 descriptor version
    return d;
}
// kind::i8 instruction descriptor: D s32, A u8 K-major (TMEM), B s8/u8 MN-major, M = 128.
__host__ __device__ constexpr uint32_t idesc_i8(int N, bool b_signed) {
    return (2u << 4) | ((b_signed ? 1u : 0u) << 10) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
                 : "memory");
}

// Channel of K-element k (A column k/4, byte k%4) of a packed K row: register rho =
// u*cpb + s holds bytes 4u..4u+3 of the row masked to code slot s (bits [s*b, s*b+b)).
template <int BITS>
__host__ __device__ __forceinline__ int k_channel(int k, int& shift) {
    constexpr int cpb = 8 / BITS;
    const int rho = k >> 2, i = k & 3;
    const int u = rho / cpb, s = rho % cpb;
    shift = s * BITS;
    return (4 * u + i) * cpb + (cpb - 1 - s);
}

// ---- prep: fold the K scales into the query, emit the phase-A B tile ---------------------
template <int BITS, int NT>
__global__ void __launch_bounds__(kDim) prep_umma_kernel(DecodeArgs a, uint8_t* __restrict__ qb,
                                                         float2* __restrict__ qconst) {
    griddep_launch();  // the decode grid may start streaming codes right away
    __shared__ float s_qs[8][kDim];
    __shared__ float s_red[2][8][4];
    __shared__ float s_scale[8];
    const int unit = blockIdx.x, c = threadIdx.x, G = (int)a.group;
    const int lane = c & 31, wid = c >> 5;
    const float levels = (float)((1u << BITS) - 1u);
    const float isd = __fdiv_rn(1.0f, sqrtf((float)kDim));
    const float ka = a.k_alpha[unit * kDim + c];
    const float range = __fsub_rn(a.k_beta[unit * kDim + c], ka);
    const float step = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
    for (int h = 0; h < 8; ++h) {
        float qs = 0.f, qa = 0.f;
        if (h < G) {
            const float q = a.q[(unit * G + h) * kDim + c];
            qs = range > 0.0f ? __fmul_rn(q, step) : 0.0f;  // detail::scale_query
            qa = __fmul_rn(q, ka);
        }
        s_qs[h][c] = qs;
        float ab = fabsf(qs), sa = qa;
#pragma unroll
        for (int o = 16; o; o >>= 1) {
            ab = fmaxf(ab, __shfl_xor_sync(0xffffffffu, ab, o));
            sa += __shfl_xor_sync(0xffffffffu, sa, o);
        }
        if (lane == 0) {
            s_red[0][h][wid] = ab;
            s_red[1][h][wid] = sa;
        }
    }
    __syncthreads();
    if (c < 8) {
        const int h = c;
        const float max_abs = fmaxf(fmaxf(s_red[0][h][0], s_red[0][h][1]), fmaxf(s_red[0][h][2], s_red[0][h][3]));
        const float qdota = (s_red[1][h][0] + s_red[1][h][1]) + (s_red[1][h][2] + s_red[1][h][3]);
        // |Q_c| <= 2^30: four balanced base-256 digits; per-plane MMA sums stay < 2^22.
        const float S = max_abs > 0.0f ? 1073741824.0f / max_abs : 0.0f;
        s_scale[h] = S;
        if (h < G) qconst[unit * 8 + h] = make_float2(S > 0.0f ? isd / S : 0.0f, qdota * isd);
    }
    __syncthreads();
    // Row k of the B tile (16 bytes per head group): byte 4h' + plane of group hg is the
    // balanced base-256 digit `plane` of Q = round(S_h qs_ch / 2^shift), h = 4 hg + h'.
    const int k = c;
    int sh;
    const int ch = k_channel<BITS>(k, sh);
#pragma unroll
    for (int hg = 0; hg < NT; ++hg) {
        uint32_t w[4];
#pragma unroll
        for (int hh = 0; hh < 4; ++hh) {
            const int h = 4 * hg + hh;
            uint32_t word = 0;
            if (h < G) {
                const int Q = __float2int_rn(__fmul_rn(s_qs[h][ch], s_scale[h]) * __int_as_float((127 - sh) << 23));
                const int d0 = ((Q + 128) & 255) - 128;
                const int q1 = (Q - d0) >> 8;
                const int d1 = ((q1 + 128) & 255) - 128;
                const int q2 = (q1 - d1) >> 8;
                const int d2 = ((q2 + 128) & 255) - 128;
                const int d3 = (q2 - d2) >> 8;
                word = (uint32_t)(d0 & 255) | ((uint32_t)(d1 & 255) << 8) | ((uint32_t)(d2 & 255) << 16) |
                       ((uint32_t)(d3 & 255) << 24);
            }
            w[hh] = word;
        }
        // MN-major tile: head group hg at byte offset hg * 2048, row k at k * 16
        *reinterpret_cast<uint4*>(qb + (size_t)unit * 128 * 16 * NT + hg * 2048 + k * 16) =
            make_uint4(w[0], w[1], w[2], w[3]);
    }
}

// ---- decode ------------------------------------------------------------------------------
struct USmem {
    uint8_t* ring;       // [kStages][kBlockBytes]
    float* recv;         // [S][8 * 128 + 8] rank 0: partial outputs (aliases the drained ring)
    uint8_t* qb;         // [NT][128][16] phase-A B tile
    uint8_t* ptile;      // [NA][NT][128][16] phase-B B tiles (p digit planes)
    float* tail_s;       // [8][kTailMax] fp32 tail scores (rank 0)
    float* red;          // [4 warps][3][8] per-warp (min, max, W) per head
    float* allpart;      // [S][24] per-CTA (min, max, tail max) records
    float* gpar;         // [8][4] softmax parameters per head
    uint64_t* full;      // [kStages] TMA landed            (tx count)
    uint64_t* empty;     // [kStages] consumers read a stage (4 warp arrivals)
    uint64_t* afull;     // [2][4] A operand (+ p tile) in place, per phase and A buffer
    uint64_t* dfull;     // [2][4] MMA retired (tcgen05.commit): phase A per D buffer,
                         //        phase B per A buffer
    uint64_t* dempty;    // [4] phase-A accumulator read back (4 warp arrivals)
    uint32_t* tmem_slot;
};

template <int BITS, int NT>
__host__ __device__ inline size_t umma_smem_bytes(int T, int S, USmem* out = nullptr, uint8_t* base = nullptr) {
    using Gm = UGeo<BITS, NT>;
    size_t off = 0;
    auto take = [&](size_t bytes, size_t align) {
        off = (off + align - 1) / align * align;
        size_t o = off;
        off += bytes;
        return base + o;
    };
    const size_t ring_bytes = (size_t)Gm::kStages * Gm::kBlockBytes;
    const size_t recv_bytes = (size_t)S * (8 * kDim + 8) * 4;
    uint8_t* ring = take(ring_bytes > recv_bytes ? ring_bytes : recv_bytes, 128);
    (void)T;
    uint8_t* qb = take((size_t)NT * 2048, 128);
    uint8_t* ptile = take((size_t)Gm::kNA * NT * 2048, 128);
    uint8_t* tail_s = take((size_t)8 * kTailMax * 4, 16);
    uint8_t* red = take((size_t)4 * 3 * 8 * 4, 16);
    uint8_t* allpart = take((size_t)kMaxCluster * 24 * 4, 16);
    uint8_t* gpar = take(32 * 4, 16);
    uint8_t* full = take((size_t)Gm::kStages * 8, 8);
    uint8_t* empty = take((size_t)Gm::kStages * 8, 8);
    uint8_t* bars = take(20 * 8, 8);
    uint8_t* slot = take(16, 16);
    if (out) {
        out->ring = ring;
        out->recv = reinterpret_cast<float*>(ring);
        out->qb = qb;
        out->ptile = ptile;
        out->tail_s = reinterpret_cast<float*>(tail_s);
        out->red = reinterpret_cast<float*>(red);
        out->allpart = reinterpret_cast<float*>(allpart);
        out->gpar = reinterpret_cast<float*>(gpar);
        out->full = reinterpret_cast<uint64_t*>(full);
        out->empty = reinterpret_cast<uint64_t*>(empty);
        out->afull = reinterpret_cast<uint64_t*>(bars);
        out->dfull = reinterpret_cast<uint64_t*>(bars) + 8;
        out->dempty = reinterpret_cast<uint64_t*>(bars) + 16;
        out->tmem_slot = reinterpret_cast<uint32_t*>(slot);
    }
    return off;
}

// Named barrier over the 4 consumer warps only (the issuer warp never joins it).
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Warp roles: warps 0-3 = consumers (thread = TMEM lane: token row in phase A, channel in
// phase B; operand expansion, epilogues, softmax); warp 4 = MMA issuer (lane 0 issues
// every tcgen05.mma); warp 5 = TMA producer (lane 0 streams the ring). Hand-offs are
// mbarriers only, so no warp waits for another except through a data dependency.
template <int BITS, int NT>
__global__ void __launch_bounds__(kThreads + 64) decode_umma_kernel(const UParams p) {
    using Gm = UGeo<BITS, NT>;
    constexpr int H = Gm::kHeads;
    const DecodeArgs& a = p.a;
    const int G = (int)a.group;
    const int S = p.S;
    const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const int unit = blockIdx.x / S;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    extern __shared__ __align__(1024) uint8_t smem_raw[];
    USmem sm;
    umma_smem_bytes<BITS, NT>(p.T, S, &sm, smem_raw);
    if (tid == 0) UTRACE(0);

    const int n = (int)a.n_vis;
    const int tok0 = rank * p.T;
    const int nv = max(0, min(p.T, n - tok0));  // this CTA's visual tokens
    const int nblk = (nv + kBlk - 1) / kBlk;
    const int nvb = (n + kBlk - 1) / kBlk;       // V^T blocks of the unit
    const int ntl = rank == 0 ? a.tail_len[unit / a.kv_heads] : 0;
    const int total_stages = 2 * nblk;

    if (tid == 0) {
        for (int i = 0; i < Gm::kStages; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 4);
        }
        for (int i = 0; i < 8; ++i) {
            mbar_init(&sm.afull[i], 4);
            mbar_init(&sm.dfull[i], 1);
        }
        for (int i = 0; i < 4; ++i) mbar_init(&sm.dempty[i], 4);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(sm.tmem_slot)),
                     "r"(Gm::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (S > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");  // #0
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tbase = *sm.tmem_slot;

    if (warp == 5) {
        // ======================= TMA producer warp =======================
        // Streams the unit's K blocks then its V^T blocks through the ring, refilling a
        // slot as soon as the 4 consumer warps have read it (decoupled from the MMAs).
        if (S > 1) {
            // This warp publishes nothing at #1; arriving before streaming lets its phase-B
            // refills (which wait on consumers that are past #1) proceed.
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // #0
            cluster_arrive();  // #1
        }
        {
            const uint8_t* kcodes = a.k_codes + ((size_t)unit * n + tok0) * Gm::kRowBytes;
            const uint8_t* vcodes = a.v_codes_t + ((size_t)unit * nvb + tok0 / kBlk) * Gm::kBlockBytes;
            for (int i = 0; i < total_stages; ++i) {
                const int slot = i % Gm::kStages;
                if (i >= Gm::kStages) mbar_wait_long(&sm.empty[slot], ((i / Gm::kStages) - 1) & 1);
                if (lane == 0 && i < 64) BTRACE(192 + i);
                uint32_t bytes;
                const uint8_t* src;
                if (i < nblk) {
                    src = kcodes + (size_t)i * Gm::kBlockBytes;
                    bytes = (uint32_t)(min(kBlk, nv - i * kBlk) * Gm::kRowBytes);
                } else {
                    src = vcodes + (size_t)(i - nblk) * Gm::kBlockBytes;
                    bytes = (uint32_t)Gm::kBlockBytes;
                }
                if (elect_one()) {
                    mbar_expect_tx(&sm.full[slot], bytes);
                    bulk_g2s(sm.ring + slot * Gm::kBlockBytes, src, bytes, &sm.full[slot]);
                }
                __syncwarp();
            }
        }
        if (S > 1) {
            cluster_wait();  // #1
            cluster_arrive();  // #2a
            cluster_wait();
            cluster_arrive();  // #2b
            cluster_wait();
        }
    } else if (warp == 4) {
        // ======================= MMA issuer warp =======================
        {
            constexpr uint32_t kIdA = idesc_i8(Gm::kN, true);
            const uint32_t qb_addr = smem_u32(sm.qb);
            for (int blk = 0; blk < nblk; ++blk) {
                const int x = blk % Gm::kNA, y = blk % Gm::kND;
                mbar_wait_long(&sm.afull[x], (blk / Gm::kNA) & 1);
                if (lane == 0 && blk < 16) BTRACE(128 + 4 * blk);
                if (blk >= Gm::kND) mbar_wait_long(&sm.dempty[y], (blk / Gm::kND - 1) & 1);
                if (lane == 0 && blk < 16) BTRACE(128 + 4 * blk + 1);
                tc_fence_after();
                const uint32_t d = tbase + Gm::kColDA + Gm::kN * y;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_i8(d, tbase + Gm::kColA + 32 * x + 8 * kk, smem_desc_mn(qb_addr + kk * 512, 2048), kIdA,
                                kk > 0);
                    umma_commit(&sm.dfull[y]);
                }
                __syncwarp();
                if (lane == 0 && blk < 16) BTRACE(128 + 4 * blk + 2);
            }
        }
        if (S > 1) {
            asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");  // #0
            cluster_arrive();  // #1
            cluster_wait();
        }
        {
            constexpr uint32_t kIdB = idesc_i8(Gm::kN, false);
            const uint32_t ptile_addr = smem_u32(sm.ptile);
            for (int blk = 0; blk < nblk; ++blk) {
                const int x = blk % Gm::kNA;
                mbar_wait_long(&sm.afull[4 + x], (blk / Gm::kNA) & 1);
                tc_fence_after();
                const uint32_t pt = ptile_addr + x * NT * 2048;
                if (elect_one()) {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk)
                        umma_i8(tbase + Gm::kColDV, tbase + Gm::kColA + 32 * x + 8 * kk,
                                smem_desc_mn(pt + kk * 512, 2048), kIdB, (blk > 0 || kk > 0) ? 1u : 0u);
                    umma_commit(&sm.dfull[4 + x]);
                }
                __syncwarp();
            }
        }
        if (S > 1) {
            cluster_arrive();  // #2a
            cluster_wait();
            cluster_arrive();  // #2b
            cluster_wait();
        }
    } else {
        // ======================= consumer warps =======================
        const uint32_t tlane = tbase + ((uint32_t)(32 * warp) << 16);  // this warp's TMEM lane quarter
        // Warm L2 with the fp32 tail rows (rank 0 reads them after phase A / in the epilogue).
        for (int l = tid; l < 8 * ntl; l += kThreads) {
            const float* base = (l & 4) ? a.v_tail : a.k_tail;
            const float* ptr = base + ((size_t)unit * a.tail_cap + (l >> 3)) * kDim + 32 * (l & 3);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(ptr));
        }
        griddep_wait();  // the prep kernel's B tile and constants are visible from here on
        {
            const uint4* src = reinterpret_cast<const uint4*>(p.qb + (size_t)unit * 2048 * NT);
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) reinterpret_cast<uint4*>(sm.qb)[hg * 128 + tid] = __ldg(src + hg * 128 + tid);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B tile -> tensor core (async proxy)
        float cA[H], cB[H], lo[H], hi[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const float2 qc = h < G ? p.qconst[(size_t)unit * 8 + h] : make_float2(0.f, 0.f);
            cA[h] = qc.x, cB[h] = qc.y;
            lo[h] = INFINITY, hi[h] = -INFINITY;
        }
        consumer_sync();  // B tile complete before the first a-full arrival

        // ---------------- phase A: scores ----------------
        auto epilogue_a = [&](int blk) {
            const int y = blk % Gm::kND;
            mbar_wait_long(&sm.dfull[y], (blk / Gm::kND) & 1);
            if (tid == 0 && blk < 16) BTRACE(64 + 4 * blk + 2);
            tc_fence_after();
            uint32_t r[16 * NT];
#pragma unroll
            for (int hg = 0; hg < NT; ++hg) {
                uint32_t rr[16];
                tmem_ld_x16(tlane + Gm::kColDA + Gm::kN * y + 16 * hg, rr);
#pragma unroll
                for (int j = 0; j < 16; ++j) r[16 * hg + j] = rr[j];
            }
            tc_wait_ld();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.dempty[y]);
            const int tok = blk * kBlk + tid;
            const bool valid = tok < nv;
            float sc[H];
#pragma unroll
            for (int h = 0; h < H; ++h) {
                // digit planes: |D_pl| < 2^22, so planes (0,1) and (2,3) pair up exactly in
                // int32; the 2^16-weighted halves meet in fp32 (the total may exceed 2^31).
                const int lo16 = (int)r[4 * h] + (int)r[4 * h + 1] * 256;
                const int hi16 = (int)r[4 * h + 2] + (int)r[4 * h + 3] * 256;
                sc[h] = __fmaf_rn((float)hi16, cA[h] * 65536.0f, __fmaf_rn((float)lo16, cA[h], cB[h]));
                if (valid) {
                    lo[h] = fminf(lo[h], sc[h]);
                    hi[h] = fmaxf(hi[h], sc[h]);
                }
            }
            uint32_t sv[H];
#pragma unroll
            for (int h = 0; h < H; ++h) sv[h] = __float_as_uint(sc[h]);
            tmem_st_scores<H>(tlane + Gm::kColS + H * blk, sv);
        };
        if (tid == 0) UTRACE(1);
        for (int blk = 0; blk < nblk; ++blk) {
            const int slot = blk % Gm::kStages;
            mbar_wait_long(&sm.full[slot], (blk / Gm::kStages) & 1);
            if (tid == 0 && blk < 16) BTRACE(64 + 4 * blk);
            const uint8_t* row = sm.ring + slot * Gm::kBlockBytes + tid * Gm::kRowBytes;
            uint32_t w[4 * BITS];
#pragma unroll
            for (int u = 0; u < BITS; ++u) {
                const uint4 v = reinterpret_cast<const uint4*>(row)[u];
                w[4 * u] = v.x, w[4 * u + 1] = v.y, w[4 * u + 2] = v.z, w[4 * u + 3] = v.w;
            }
            uint32_t areg[32];
#pragma unroll
            for (int rho = 0; rho < 32; ++rho) areg[rho] = w[rho / Gm::kCpb] & (Gm::kMask << ((rho % Gm::kCpb) * BITS));
            // A[blk % NA] is free: MMA(blk - NA) retired (waited for in epilogue(blk - NA),
            // which ran at iteration blk - NA + L < blk with the lag L = NA - 1).
            tmem_st_x32(tlane + Gm::kColA + 32 * (blk % Gm::kNA), areg);
            tc_wait_st();  // also proves this thread's ring reads landed (the slot may be refilled)
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.empty[slot]);
                mbar_arrive(&sm.afull[blk % Gm::kNA]);
            }
            if (tid == 0 && blk < 16) BTRACE(64 + 4 * blk + 1);
            if (blk >= Gm::kNA - 1) epilogue_a(blk - (Gm::kNA - 1));
        }
        for (int blk = max(0, nblk - (Gm::kNA - 1)); blk < nblk; ++blk) epilogue_a(blk);
        tc_wait_st();  // this thread's score columns are in TMEM before phase B reads them back
        if (tid == 0) UTRACE(2);

        // fp32 tail rows (rank 0): warp w takes rows w, w + NW, ...; lanes split the 128
        // channels; q rows are loaded once.
        const float isd = __fdiv_rn(1.0f, sqrtf((float)kDim));
        float tmax = -INFINITY;  // for head (lane & 7)
        if (warp < 4 && ntl > warp) {
            float4 qv[8];
    #pragma unroll
            for (int h = 0; h < 8; ++h)
                qv[h] = h < G ? *reinterpret_cast<const float4*>(a.q + ((size_t)unit * G + h) * kDim + 4 * lane)
                              : make_float4(0.f, 0.f, 0.f, 0.f);
            for (int j = warp; j < ntl; j += 4) {
                const float4 kv = *reinterpret_cast<const float4*>(a.k_tail + ((size_t)unit * a.tail_cap + j) * kDim + 4 * lane);
    #pragma unroll
                for (int h = 0; h < 8; ++h) {
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
        // Per-warp (min, max) per head -> shared memory -> CTA record.
#pragma unroll
        for (int h = 0; h < H; ++h) {
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                lo[h] = fminf(lo[h], __shfl_xor_sync(0xffffffffu, lo[h], o));
                hi[h] = fmaxf(hi[h], __shfl_xor_sync(0xffffffffu, hi[h], o));
            }
            if (lane == 0) {
                sm.red[(warp * 3 + 0) * 8 + h] = lo[h];
                sm.red[(warp * 3 + 1) * 8 + h] = hi[h];
            }
        }
        {  // tail max per head over the 4 warps (lanes 0..7 hold heads 0..7)
            float tm = tmax;
            if (lane < 8) sm.red[(warp * 3 + 2) * 8 + lane] = tm;
        }
        consumer_sync();
        if (tid < 24) {  // CTA record: (min[8], max[8], tail max[8])
            const int k = tid, kind = k >> 3, h = k & 7;
            float v;
            if (kind == 2) {
                v = fmaxf(fmaxf(sm.red[(0 * 3 + 2) * 8 + h], sm.red[(1 * 3 + 2) * 8 + h]),
                          fmaxf(sm.red[(2 * 3 + 2) * 8 + h], sm.red[(3 * 3 + 2) * 8 + h]));
            } else if (h >= H) {
                v = kind == 0 ? INFINITY : -INFINITY;
            } else {
                v = sm.red[(0 * 3 + kind) * 8 + h];
                for (int w2 = 1; w2 < 4; ++w2)
                    v = kind == 0 ? fminf(v, sm.red[(w2 * 3 + 0) * 8 + h]) : fmaxf(v, sm.red[(w2 * 3 + 1) * 8 + h]);
            }
            if (S > 1) {
                asm volatile("barrier.cluster.wait.acquire;" ::: "memory");  // #0 (non-aligned: part of a warp)
                for (int r = 0; r < S; ++r) st_cluster_f32(sm.allpart + rank * 24 + k, r, v);
            } else {
                sm.allpart[k] = v;
            }
        }
        if (S > 1) {
            if (tid >= 24) asm volatile("barrier.cluster.wait.acquire;" ::: "memory");  // #0, the rest
            cluster_arrive();  // #1: records pushed everywhere
            cluster_wait();
        } else {
            consumer_sync();
        }
        // Global softmax parameters per head (identical in every CTA of the unit).
        if (tid < 8) {
            const int h = tid;
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
        consumer_sync();
        if (tid == 0) UTRACE(3);

        // ---------------- phase B: p . V ----------------
        float pa[H], pb[H], wsum[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            pa[h] = sm.gpar[h * 4 + 0];
            pb[h] = sm.gpar[h * 4 + 1];
            wsum[h] = 0.0f;
        }
        // Token m's A bytes carry its code times 2^(b * ((m / 4) mod cpb)) (vt_layout): its
        // probability row is pre-divided by that slot scale. P = p * 2^31 / 2^shift < 2^32.
        const float pscale = __int_as_float((127 + 31 - BITS * ((tid >> 2) % Gm::kCpb)) << 23);
        for (int blk = 0; blk < nblk; ++blk) {
            const int i = nblk + blk;
            const int slot = i % Gm::kStages;
            const int x = blk % Gm::kNA;
            if (blk >= Gm::kNA) {  // A buffer / p tile of block blk - NA are free once its MMAs retired
                mbar_wait_long(&sm.dfull[4 + x], (blk / Gm::kNA - 1) & 1);
                tc_fence_after();
            }
            // p side first (independent of the TMA): thread m = token m of the block.
            {
                const int tok = blk * kBlk + tid;
                const bool valid = tok < nv;
                uint32_t sraw[H];
                tmem_ld_scores<H>(tlane + Gm::kColS + H * blk, sraw);
                tc_wait_ld();
                uint32_t P[H];
#pragma unroll
                for (int h = 0; h < H; ++h) {
                    const float pr = valid ? ex2(__fmaf_rn(__uint_as_float(sraw[h]), pa[h], pb[h])) : 0.0f;
                    wsum[h] += pr;
                    P[h] = __float2uint_rn(pr * pscale);
                }
                uint8_t* tile = sm.ptile + x * NT * 2048 + tid * 16;
#pragma unroll
                for (int hg = 0; hg < NT; ++hg)
                    *reinterpret_cast<uint4*>(tile + hg * 2048) =
                        make_uint4(P[4 * hg], P[4 * hg + 1], P[4 * hg + 2], P[4 * hg + 3]);
            }
            // V side: thread c = channel c, 4b words = 128 tokens of codes.
            mbar_wait_long(&sm.full[slot], (i / Gm::kStages) & 1);
            {
                const uint8_t* src = sm.ring + slot * Gm::kBlockBytes + tid * Gm::kRowBytes;
                uint32_t w[4 * BITS];
#pragma unroll
                for (int u = 0; u < BITS; ++u) {
                    const uint4 v = reinterpret_cast<const uint4*>(src)[u];
                    w[4 * u] = v.x, w[4 * u + 1] = v.y, w[4 * u + 2] = v.z, w[4 * u + 3] = v.w;
                }
                uint32_t areg[32];
#pragma unroll
                for (int rho = 0; rho < 32; ++rho)
                    areg[rho] = w[rho / Gm::kCpb] & (Gm::kMask << ((rho % Gm::kCpb) * BITS));
                tmem_st_x32(tlane + Gm::kColA + 32 * x, areg);
            }
            tc_wait_st();  // also proves this thread's ring reads landed (the slot may be refilled)
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // p tile -> async proxy
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sm.empty[slot]);
                mbar_arrive(&sm.afull[4 + x]);
            }
        }
        // CTA weight sums (fixed order: warp shuffles, then warps 0..3).
#pragma unroll
        for (int h = 0; h < H; ++h) {
#pragma unroll
            for (int o = 16; o; o >>= 1) wsum[h] += __shfl_xor_sync(0xffffffffu, wsum[h], o);
        }
        if (lane == 0)
            for (int h = 0; h < H; ++h) sm.red[(warp * 3 + 2) * 8 + h] = wsum[h];
        if (nblk > 0) {
            mbar_wait_long(&sm.dfull[4 + (nblk - 1) % Gm::kNA], ((nblk - 1) / Gm::kNA) & 1);
            tc_fence_after();
        }
        consumer_sync();
        if (tid == 0) UTRACE(4);
        // Epilogue, thread c = channel c:
        //   out = (s_c V / 2^31 + alpha_c W_vis + sum_t p_t v_tc) / (W_vis + sum_t p_t)
        uint32_t r[16 * NT];
#pragma unroll
        for (int hg = 0; hg < NT; ++hg) {
            uint32_t rr[16];
            if (nblk > 0) {
                tmem_ld_x16(tlane + Gm::kColDV + 16 * hg, rr);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) rr[j] = 0;
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) r[16 * hg + j] = rr[j];
        }
        tc_wait_ld();
        const int ch = tid;
        constexpr float kInvLevels = 1.0f / (float)((1u << BITS) - 1u);
        const float va = __ldg(a.v_alpha + unit * kDim + ch);
        const float vstep = fmaxf(__fsub_rn(__ldg(a.v_beta + unit * kDim + ch), va) * kInvLevels, 0.0f);
        float num[H], den[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
            const float W = (sm.red[(0 * 3 + 2) * 8 + h] + sm.red[(1 * 3 + 2) * 8 + h]) +
                            (sm.red[(2 * 3 + 2) * 8 + h] + sm.red[(3 * 3 + 2) * 8 + h]);
            const float V = __fmaf_rn((float)r[4 * h + 3], 16777216.0f,
                                      __fmaf_rn((float)r[4 * h + 2], 65536.0f,
                                                __fmaf_rn((float)r[4 * h + 1], 256.0f, (float)r[4 * h])));
            num[h] = __fmaf_rn(vstep, V * 4.656612873077393e-10f /* 2^-31 */, va * W);
            den[h] = W;
            if (h < G) {  // fp32 tail (rank 0), 8 independent loads in flight, j ascending
                const float* vt = a.v_tail + (size_t)unit * a.tail_cap * kDim + ch;
                int j = 0;
                for (; j + 8 <= ntl; j += 8) {
                    float vv[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) vv[u] = __ldg(vt + (size_t)(j + u) * kDim);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const float pt = ex2(__fmaf_rn(sm.tail_s[h * kTailMax + j + u], kLog2e, sm.gpar[h * 4 + 2]));
                        den[h] += pt;
                        num[h] = __fmaf_rn(pt, vv[u], num[h]);
                    }
                }
                for (; j < ntl; ++j) {
                    const float pt = ex2(__fmaf_rn(sm.tail_s[h * kTailMax + j], kLog2e, sm.gpar[h * 4 + 2]));
                    den[h] += pt;
                    num[h] = __fmaf_rn(pt, __ldg(vt + (size_t)j * kDim), num[h]);
                }
            }
        }
        if (S == 1) {
#pragma unroll
            for (int h = 0; h < H; ++h)
                if (h < G) a.out[((size_t)unit * G + h) * kDim + ch] = num[h] / den[h];
        } else {
            // Every CTA is past phase B (its ring is drained) before rank 0's ring becomes
            // the receive buffer of the partial numerators / denominators.
            cluster_arrive();  // #2a
            cluster_wait();
            float* recv = sm.recv;
#pragma unroll
            for (int h = 0; h < H; ++h) {
                if (h >= G) continue;
                st_cluster_f32(recv + rank * (8 * kDim + 8) + h * kDim + ch, 0, num[h]);
                if (ch == 0) st_cluster_f32(recv + rank * (8 * kDim + 8) + 8 * kDim + h, 0, den[h]);
            }
            cluster_arrive();  // #2b: partials are in rank 0
            cluster_wait();
            if (rank == 0) {
                for (int h = 0; h < G; ++h) {
                    float nn = 0.f, dd = 0.f;
                    for (int r2 = 0; r2 < S; ++r2) {
                        nn += recv[r2 * (8 * kDim + 8) + h * kDim + ch];
                        dd += recv[r2 * (8 * kDim + 8) + 8 * kDim + h];
                    }
                    a.out[((size_t)unit * G + h) * kDim + ch] = nn / dd;
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (tid == 0) UTRACE(5);
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "r"(Gm::kTmemCols));
}

// ---- token-packed V layout --------------------------------------------------------------
// vt_layout: [unit][block of 128 tokens][channel][4b u32 words]. Word w of channel c
// holds, in byte i and code slot s (bits [s*b, s*b+b) of the byte), the code of token
// 4 (w cpb + s) + i of the block, so a LOP3 with (2^b - 1) * 0x01010101 << s*b yields
// the codes of tokens 4 rho .. 4 rho + 3 (rho = w cpb + s) as the bytes of one TMEM
// column: the A operand of phase B with K = token order. Tokens past n are zero codes.
template <int BITS>
__global__ void __launch_bounds__(kDim) pack_vt_kernel(const uint8_t* __restrict__ rows, size_t n, size_t nvb,
                                                       uint8_t* __restrict__ vt) {
    constexpr int kRowBytes = 16 * BITS, cpb = 8 / BITS;
    __shared__ __align__(16) uint8_t s_rows[kBlk * kRowBytes];
    const size_t unit = blockIdx.y, blk = blockIdx.x;
    const size_t t0 = blk * kBlk;
    const int valid = (int)min((size_t)kBlk, n - t0);
    const uint8_t* src = rows + (unit * n + t0) * kRowBytes;
    for (int i = threadIdx.x; i < kBlk * kRowBytes / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(s_rows)[i] = i * 4 < valid * kRowBytes ? reinterpret_cast<const uint32_t*>(src)[i] : 0u;
    __syncthreads();
    const int c = threadIdx.x;
    const int byte = c / cpb, bshift = 8 - BITS * (c % cpb + 1);
    const uint32_t mask = (1u << BITS) - 1u;
    uint32_t out[4 * BITS];
#pragma unroll
    for (int w = 0; w < 4 * BITS; ++w) {
        uint32_t word = 0;
#pragma unroll
        for (int s = 0; s < cpb; ++s)
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const int tok = 4 * (w * cpb + s) + i;
                const uint32_t code = (s_rows[tok * kRowBytes + byte] >> bshift) & mask;
                word |= code << (8 * i + BITS * s);
            }
        out[w] = word;
    }
    uint4* dst = reinterpret_cast<uint4*>(vt + ((unit * nvb + blk) * kDim + c) * kRowBytes);
#pragma unroll
    for (int u = 0; u < BITS; ++u) dst[u] = make_uint4(out[4 * u], out[4 * u + 1], out[4 * u + 2], out[4 * u + 3]);
}

void plan(const DecodeArgs& a, int& S, int& T) {
    const int max_tokens = a.group > 4 ? 2048 : 4096;  // UGeo<.., NT>::kMaxTokens
    S = std::max(1, (int)((a.n_vis + max_tokens - 1) / max_tokens));
    const int per = (int)((a.n_vis + S - 1) / S);
    T = (per + kBlk - 1) / kBlk * kBlk;
}

template <int BITS, int NT>
size_t smem_for(const DecodeArgs& a) {
    int S, T;
    plan(a, S, T);
    size_t bytes = umma_smem_bytes<BITS, NT>(T, S);
    // TMEM is kTmemCols per CTA: never let more CTAs share an SM than TMEM can serve
    // (a blocked tcgen05.alloc inside a cluster could deadlock against its partners).
    const size_t max_ctas = 512 / UGeo<BITS, NT>::kTmemCols;
    const size_t floor_bytes = 232448 / (max_ctas + 1) + 1;  // 227 KB per SM usable
    return bytes > floor_bytes ? bytes : floor_bytes;
}

template <int BITS, int NT>
cudaError_t launch_bits(const DecodeArgs& a, cudaStream_t s) {
    int S, T;
    plan(a, S, T);
    prep_umma_kernel<BITS, NT><<<(unsigned)a.units, kDim, 0, s>>>(a, a.umma_qb, a.tc_qconst);
    note_launch();
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    UParams p{a, a.umma_qb, a.tc_qconst, S, T};
    const size_t smem = smem_for<BITS, NT>(a);
    auto kern = decode_umma_kernel<BITS, NT>;
    static unsigned attr_done = 0;  // per instantiation, bit per device
    e = once_per_device(attr_done, [&] {
        cudaError_t r = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        return r != cudaSuccess ? r : cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    });
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(a.units * S));
    cfg.blockDim = dim3(kThreads + 64);  // 4 consumer warps + MMA issuer + TMA producer
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
    e = cudaLaunchKernelEx(&cfg, kern, p);
    note_launch();
    return e;
}

}  // namespace

size_t vt_bytes(size_t units, size_t n_vis, int bits) {
    return units * ((n_vis + kBlk - 1) / kBlk) * (size_t)kBlk * 16 * bits;
}

cudaError_t launch_pack_vt(const uint8_t* rows, size_t units, size_t n_vis, int bits, uint8_t* vt, cudaStream_t s) {
    if (n_vis == 0 || units == 0) return cudaSuccess;
    const size_t nvb = (n_vis + kBlk - 1) / kBlk;
    dim3 grid((unsigned)nvb, (unsigned)units);
    switch (bits) {
        case 1: pack_vt_kernel<1><<<grid, kDim, 0, s>>>(rows, n_vis, nvb, vt); break;
        case 2: pack_vt_kernel<2><<<grid, kDim, 0, s>>>(rows, n_vis, nvb, vt); break;
        case 4: pack_vt_kernel<4><<<grid, kDim, 0, s>>>(rows, n_vis, nvb, vt); break;
        case 8: pack_vt_kernel<8><<<grid, kDim, 0, s>>>(rows, n_vis, nvb, vt); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return cudaGetLastError();
}

size_t decode_umma_scratch_bytes(size_t units) { return units * 2 * 2048; }

bool decode_umma_supported(const DecodeArgs& a) {
    if (a.dim != (size_t)kDim || a.word_bits != 8 || a.n_vis == 0 || !a.v_codes_t) return false;
    if (a.bits != 1 && a.bits != 2 && a.bits != 4 && a.bits != 8) return false;
    if (a.group < 1 || a.group > 8) return false;
    if (a.units == 0) return false;
    int S, T;
    plan(a, S, T);
    if (S > kMaxCluster) return false;
    if (a.tail_cap > (size_t)kTailMax) return false;  // the fp32 tail lives in rank 0
    const int NT = a.group > 4 ? 2 : 1;
    size_t smem = 0;
    switch (a.bits * 10 + NT) {
        case 11: smem = smem_for<1, 1>(a); break;
        case 12: smem = smem_for<1, 2>(a); break;
        case 21: smem = smem_for<2, 1>(a); break;
        case 22: smem = smem_for<2, 2>(a); break;
        case 41: smem = smem_for<4, 1>(a); break;
        case 42: smem = smem_for<4, 2>(a); break;
        case 81: smem = smem_for<8, 1>(a); break;
        case 82: smem = smem_for<8, 2>(a); break;
    }
    return smem <= 220 * 1024;
}

cudaError_t launch_decode_umma(const DecodeArgs& a, cudaStream_t s) {
    if (!a.umma_qb || !a.tc_qconst || !a.v_codes_t) return cudaErrorInvalidValue;
    const int NT = a.group > 4 ? 2 : 1;
    switch (a.bits * 10 + NT) {
        case 11: return launch_bits<1, 1>(a, s);
        case 12: return launch_bits<1, 2>(a, s);
        case 21: return launch_bits<2, 1>(a, s);
        case 22: return launch_bits<2, 2>(a, s);
        case 41: return launch_bits<4, 1>(a, s);
        case 42: return launch_bits<4, 2>(a, s);
        case 81: return launch_bits<8, 1>(a, s);
        case 82: return launch_bits<8, 2>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace kvqb
