// k2_decode_ps.cu — K2 throughput path for many short units: the exact-integer IMMA decode
// of k2_decode_tc.cu as one persistent CTA per SM whose 16 warps pull work from shared
// queues ("ps"), d = 128, b in {1, 2, 4}, G <= 4, n <= 4096 per unit.
//
// Math (reference: kernels.hpp:14-26, 183-194, 277-283; calibrate.hpp:62-114;
// kvcache.hpp:263-311), per (unit, query head h):
//   score_j = (sum_c qs_c code_jc + q.alpha) / sqrt(d),  qs_c = q_c (beta_c - alpha_c) / L
//   row     = [g(score_vis) | score_tail],  g affine from (gamma, delta) of the vis part
//   out_c   = (s_c sum_j p_j code_jc + alpha_c sum_j p_j + sum_t p_t v_tc) / sum p
//
// Why (profiles/r02_tc_trace2_c2.txt): the per-CTA kernel keeps every unit of C2 resident
// at once (four 4-warp CTAs per SM), but the CTAs sharing an SM progress unevenly (the warp
// arbiter favours some), so an SM's last CTA finishes ~8 us after its first, and every CTA
// pays its own prologue and epilogue. Here an SM's units are processed in rounds of up to
// R units (R = 512 tensor-memory columns / (n / 32)):
//   prologue : every unit's query digit planes at once (128 threads per unit);
//   phase A  : chunks of 128/b tokens (unit-major) in four lane-quarter queues, the four
//              warps of a quarter pull them dynamically (shared-memory counter), stream the K
//              rows through private cp.async.bulk rings (chunks grabbed ahead, so the copies
//              are in flight), and park the scores in their quarter's tensor-memory lanes;
//   params   : one CTA barrier, gamma / delta / m per (unit, head) from per-warp partials;
//   phase B  : the same queues over the V operand (vx layout); a warp keeps one unit's 64
//              integer accumulators and flushes them to that unit's shared-memory image
//              (exact red.add) when its next chunk belongs to another unit;
//   epilogue : outputs of every unit of the round from the images.
// Dynamic chunks equalize the warps of an SM; one CTA per SM means one prologue and one
// epilogue per round instead of per unit.
#include <cstdlib>

#include "kvq_internal.cuh"
#include "kvq_ptx.cuh"

namespace kvqb {

namespace {

using namespace ptx;

constexpr int kDim = 128;
constexpr int kW = 16;                   // warps
constexpr int kThreads = 32 * kW;
constexpr int kStages = 3;               // per-warp ring depth (chunks in flight)
constexpr int kChunkBytes = 2048;        // one chunk = 128/b tokens of K rows or V blocks
constexpr int kMaxR = 4;                 // units per round (tensor memory: 4 x 128 columns)
constexpr int kTailMax = 64;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kMagic = 12582912.0f;
constexpr float kPScale = 4190000.0f;
constexpr float kLog2PScale = 21.9985188f;
constexpr int kPRow = 12;

struct PsParams {
    DecodeArgs a;
    int R;  // units per round (tensor memory: R * n / 32 <= 512 columns)
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

template <int BITS>
struct Geo {
    static constexpr int kRowBytes = 16 * BITS;              // reference K row (M = 8)
    static constexpr int kChunkTok = kChunkBytes / kRowBytes;  // 128 / b tokens
    static constexpr int kSteps = kChunkTok / 32;            // 32-token steps per chunk
    static constexpr int kVBlk = 512 * BITS;                 // vx bytes per 32-token block
    static constexpr uint32_t kMask = 0x01010101u * ((1u << BITS) - 1u);
    static constexpr int kCpb = 8 / BITS;
};

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
    uint8_t* ring;      // [kW][kStages][kChunkBytes]
    uint32_t* acc;      // [kMaxR][16 nc][4 r][32 lanes] exact p.V sums per unit of the round
    uint32_t* pw;       // [kW][2][12][kPRow] p digit planes of a warp's block
    uint32_t* frag;     // [kMaxR][512] q digit-plane B fragments per unit
    float* qc;          // [kMaxR][4][2] (score scale, offset) per unit and head
    float* sred;        // [kMaxR][2][4][4] sum|qs|, q.alpha partials (prologue)
    float* part;        // [kW][kMaxR][12] per-warp min[4], max[4], tail max[4]
    float* gpar;        // [kMaxR][4][4] softmax parameters
    float* tail_s;      // [kMaxR][4][kTailMax] fp32 tail scores
    uint32_t* wsum;     // [kW][kMaxR][4] u22 weight sums
    int* qctr;          // [2 phases][4 quarters] chunk counters
    uint64_t* full;     // [kW][kStages]
    uint32_t* tmem_slot;
};

__host__ __device__ inline size_t ps_smem_bytes(Smem* out = nullptr, uint8_t* base = nullptr) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 127) & ~size_t(127);
        return base + o;
    };
    uint8_t* ring = take((size_t)kW * kStages * kChunkBytes);
    uint8_t* acc = take((size_t)kMaxR * 16 * 4 * 32 * 4);
    uint8_t* pw = take((size_t)kW * 2 * 12 * kPRow * 4);
    uint8_t* frag = take((size_t)kMaxR * 512 * 4);
    uint8_t* qc = take((size_t)kMaxR * 8 * 4);
    uint8_t* sred = take((size_t)kMaxR * 32 * 4);
    uint8_t* part = take((size_t)kW * kMaxR * 12 * 4);
    uint8_t* gpar = take((size_t)kMaxR * 16 * 4);
    uint8_t* tail_s = take((size_t)kMaxR * 4 * kTailMax * 4);
    uint8_t* wsum = take((size_t)kW * kMaxR * 4 * 4);
    uint8_t* qctr = take(8 * 4);
    uint8_t* full = take((size_t)kW * kStages * 8);
    uint8_t* slot = take(16);
    if (out) {
        out->ring = ring;
        out->acc = reinterpret_cast<uint32_t*>(acc);
        out->pw = reinterpret_cast<uint32_t*>(pw);
        out->frag = reinterpret_cast<uint32_t*>(frag);
        out->qc = reinterpret_cast<float*>(qc);
        out->sred = reinterpret_cast<float*>(sred);
        out->part = reinterpret_cast<float*>(part);
        out->gpar = reinterpret_cast<float*>(gpar);
        out->tail_s = reinterpret_cast<float*>(tail_s);
        out->wsum = reinterpret_cast<uint32_t*>(wsum);
        out->qctr = reinterpret_cast<int*>(qctr);
        out->full = reinterpret_cast<uint64_t*>(full);
        out->tmem_slot = reinterpret_cast<uint32_t*>(slot);
    }
    return off;
}

#define PSTRACE(k)                                                                         \
    do {                                                                                   \
        if (a.trace) a.trace[(size_t)blockIdx.x * 256 + (k)] = gtimer();                   \
    } while (0)

template <int BITS>
__global__ void __launch_bounds__(kThreads, 1) decode_ps_kernel(const PsParams p) {
    using Gm = Geo<BITS>;
    const DecodeArgs& a = p.a;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int g = lane >> 2, t = lane & 3;
    const int quarter = warp & 3;  // tensor-memory lane quarter (warp % 4)
    const int G = (int)a.group;
    const int n = (int)a.n_vis;
    const int units = (int)a.units;
    const int R = p.R;
    const int nq = (n + 3) / 4;                          // tokens per quarter per unit
    const int nq_pad = (nq + Gm::kChunkTok - 1) / Gm::kChunkTok * Gm::kChunkTok;
    const int chunks_q = nq_pad / Gm::kChunkTok;         // chunks per (unit, quarter)
    const int cols_unit = nq_pad / 32 * 4;               // tensor-memory columns per unit
    const int my_units = ((units - (int)blockIdx.x) + (int)gridDim.x - 1) / (int)gridDim.x;
    auto unit_of = [&](int k) { return (int)blockIdx.x + k * (int)gridDim.x; };
    const size_t nb32 = (size_t)(n + 31) / 32;

    extern __shared__ __align__(128) uint8_t smem_raw[];
    Smem sm;
    ps_smem_bytes(&sm, smem_raw);
    if (threadIdx.x == 0) PSTRACE(0);
    uint8_t* ring = sm.ring + warp * kStages * kChunkBytes;
    uint64_t* full = sm.full + warp * kStages;
    if (lane == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = threadIdx.x; i < kMaxR * 16 * 4 * 32; i += kThreads) sm.acc[i] = 0u;
    if (threadIdx.x < 8) sm.qctr[threadIdx.x] = 0;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(sm.tmem_slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tq = *sm.tmem_slot + ((uint32_t)(32 * quarter) << 16);
    const float levels = (float)((1u << BITS) - 1u);
    const float isd0 = __fdiv_rn(1.0f, sqrtf((float)kDim));
    int ring_i = 0;  // this warp's ring position (stages issued and consumed, monotone)

    // A phase's queue of quarter q lists chunks (unit slot us, chunk c) unit-major: item =
    // us * chunks_q + c, tokens [q nq + c chunk_tok, ...) of unit us. Warps of the quarter
    // grab items ahead (lane 0, shared counter) so their copies are in flight; `slots`
    // holds the grabbed items in ring order.
    auto grab = [&](int phase, int total) {
        int it = 0;
        if (lane == 0) it = atomicAdd(&sm.qctr[phase * 4 + quarter], 1);
        it = __shfl_sync(0xffffffffu, it, 0);
        return it < total ? it : -1;
    };
    // lane 0: the bytes of item `it` of this quarter for phase (0: K rows, 1: V blocks)
    auto issue = [&](int phase, int round0, int it, int slot) {
        const int us = it / chunks_q, c = it - us * chunks_q;
        const int unit = unit_of(round0 + us);
        const int tok0 = quarter * nq + c * Gm::kChunkTok;  // unit-relative
        const int valid = max(0, min(Gm::kChunkTok, min(nq - c * Gm::kChunkTok, n - tok0)));
        const uint8_t* src;
        uint32_t bytes;
        if (phase == 0) {
            src = a.k_codes + ((size_t)unit * n + tok0) * Gm::kRowBytes;
            bytes = (uint32_t)valid * (uint32_t)Gm::kRowBytes;
        } else {
            // vx blocks are 32-token aligned: the quarter's chunk starts at a block boundary
            // (nq multiple of 32 unless n is tiny: see ps_supported)
            src = a.v_codes_x + ((size_t)unit * nb32 + (size_t)(tok0 / 32)) * Gm::kVBlk;
            bytes = (uint32_t)((valid + 31) / 32) * (uint32_t)Gm::kVBlk;
        }
        if (bytes == 0) bytes = 16, src = phase == 0 ? a.k_codes : a.v_codes_x;  // keep the barrier flowing
        mbar_expect_tx(&full[slot], bytes);
        bulk_g2s(ring + slot * kChunkBytes, src, bytes, &full[slot]);
    };

    griddep_wait();  // q and the tail come from the preceding kernels
    griddep_launch();
    if (threadIdx.x == 0) PSTRACE(3);

    for (int round0 = 0; round0 < my_units; round0 += R) {
        const int nr = min(R, my_units - round0);
        const int total = nr * chunks_q;  // items per quarter and phase
        // ---- prologue: every unit's query digit planes (scale_query, kernels.hpp:183-194) ----
        // thread (us = tid / 128, c = tid % 128) of the first 128 nr threads
        {
            const int us = threadIdx.x >> 7, c = threadIdx.x & 127;
            float qsv[4];
            const bool mine = us < nr;
            if (mine) {
                const int unit = unit_of(round0 + us);
                const float ka = __ldg(a.k_alpha + (size_t)unit * kDim + c);
                const float kbeta = __ldg(a.k_beta + (size_t)unit * kDim + c);
                const float range = __fsub_rn(kbeta, ka);
                const float stp = range > 0.0f ? __fdiv_rn(range, levels) : 0.0f;
                float ab[4], sa[4];
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
                    sm.sred[((us * 2 + 0) * 4 + lane) * 4 + (warp & 3)] = x;
                    sm.sred[((us * 2 + 1) * 4 + lane) * 4 + (warp & 3)] = y;
                }
            }
            for (int e = threadIdx.x; e < nr * 512; e += kThreads) sm.frag[e] = 0u;
            __syncthreads();
            auto scale_of = [&](int u2, int h) {
                const float* r = sm.sred + ((u2 * 2 + 0) * 4 + h) * 4;
                const float sum_abs = (r[0] + r[1]) + (r[2] + r[3]);
                return sum_abs > 0.0f ? 1073741824.0f * __frcp_rn(levels * sum_abs) : 0.0f;
            };
            if (mine) {
                int tt, j, sh;
                const int rho = k_rho<BITS>(c, a.word_bits, tt, j, sh);
                const int kb = rho >> 1, r = rho & 1;
                uint8_t* fb = reinterpret_cast<uint8_t*>(sm.frag + us * 512);
#pragma unroll
                for (int h = 0; h < 4; ++h) {
                    if (h >= G) break;
                    const int Q = __float2int_rn(__fmul_rn(qsv[h], scale_of(us, h)) * __int_as_float((127 - sh) << 23));
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
            if (threadIdx.x < nr * 4) {
                const int u2 = threadIdx.x >> 2, h = threadIdx.x & 3;
                float cA = 0.f, cB = 0.f;
                if (h < G) {
                    const float S_h = scale_of(u2, h);
                    const float* r = sm.sred + ((u2 * 2 + 1) * 4 + h) * 4;
                    const float qdota = (r[0] + r[1]) + (r[2] + r[3]);
                    cA = S_h > 0.0f ? isd0 / S_h : 0.0f;
                    cB = qdota * isd0;
                }
                sm.qc[(u2 * 4 + h) * 2 + 0] = cA;
                sm.qc[(u2 * 4 + h) * 2 + 1] = cB;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0 && round0 == 0) PSTRACE(2);

        // ---------------- phase A: chunks of K rows -> scores in tensor memory ----------------
        {
            int slots[kStages];
#pragma unroll
            for (int i = 0; i < kStages; ++i) {
                slots[i] = grab(0, total);
                if (lane == 0 && slots[i] >= 0) issue(0, round0, slots[i], (ring_i + i) % kStages);
            }
            float lo[kMaxR], hi[kMaxR];
#pragma unroll
            for (int u2 = 0; u2 < kMaxR; ++u2) lo[u2] = INFINITY, hi[u2] = -INFINITY;
            int cur_us = -1;
            uint32_t bq[2][4][2];
            float cA = 0.f, cB = 0.f;
            while (slots[0] >= 0) {
                const int it = slots[0];
                const int us = it / chunks_q, c = it - us * chunks_q;
                if (us != cur_us) {  // this chunk's unit: its query fragments
                    cur_us = us;
#pragma unroll
                    for (int pp = 0; pp < 2; ++pp)
#pragma unroll
                        for (int kb = 0; kb < 4; ++kb)
#pragma unroll
                            for (int r = 0; r < 2; ++r) bq[pp][kb][r] = sm.frag[us * 512 + ((pp * 4 + kb) * 2 + r) * 32 + lane];
                    cA = sm.qc[(us * 4 + t) * 2 + 0];
                    cB = sm.qc[(us * 4 + t) * 2 + 1];
                }
                const int slot = ring_i % kStages;
                mbar_wait(&full[slot], (ring_i / kStages) & 1);
                const uint8_t* buf = ring + slot * kChunkBytes + g * Gm::kRowBytes + t * 4 * BITS;
                const int tokq = c * Gm::kChunkTok;                       // quarter-relative
                const int nvq = min(nq, n - quarter * nq);                 // valid tokens of the quarter
                const int nv_chunk = min(Gm::kChunkTok, nvq - tokq);
                const uint32_t tcol = tq + (uint32_t)(us * cols_unit + tokq / 8);
                float l = lo[0], hgh = hi[0];
#pragma unroll
                for (int u2 = 1; u2 < kMaxR; ++u2)
                    if (us == u2) l = lo[u2], hgh = hi[u2];
#pragma unroll
                for (int ks = 0; ks < Gm::kSteps; ++ks) {
                    if (32 * ks >= nv_chunk) break;
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
                    if (32 * ks + 32 <= nv_chunk) {
                        l = fminf(l, fminf(fminf(sc[0], sc[1]), fminf(sc[2], sc[3])));
                        hgh = fmaxf(hgh, fmaxf(fmaxf(sc[0], sc[1]), fmaxf(sc[2], sc[3])));
                    } else {
#pragma unroll
                        for (int i = 0; i < 4; ++i)
                            if (32 * ks + g + 8 * i < nv_chunk) l = fminf(l, sc[i]), hgh = fmaxf(hgh, sc[i]);
                    }
                    tmem_st4(tcol + (uint32_t)(4 * ks), sc[0], sc[1], sc[2], sc[3]);
                }
#pragma unroll
                for (int u2 = 0; u2 < kMaxR; ++u2)
                    if (us == u2) lo[u2] = l, hi[u2] = hgh;
                __syncwarp();
                // the slot is consumed: the next grabbed item takes it
#pragma unroll
                for (int i = 0; i + 1 < kStages; ++i) slots[i] = slots[i + 1];
                slots[kStages - 1] = grab(0, total);
                if (lane == 0 && slots[kStages - 1] >= 0) issue(0, round0, slots[kStages - 1], (ring_i + kStages) % kStages);
                ++ring_i;
            }
            // ring_i counts consumed items; drained slots: -1 entries issued nothing
            // per-warp partials per unit: min / max over the lanes of a head
#pragma unroll
            for (int u2 = 0; u2 < kMaxR; ++u2) {
#pragma unroll
                for (int o : {4, 8, 16}) {
                    lo[u2] = fminf(lo[u2], __shfl_xor_sync(0xffffffffu, lo[u2], o));
                    hi[u2] = fmaxf(hi[u2], __shfl_xor_sync(0xffffffffu, hi[u2], o));
                }
                if (lane < 4 && u2 < nr) {
                    float* pr = sm.part + (warp * kMaxR + u2) * 12;
                    pr[lane] = lo[u2];
                    pr[4 + lane] = hi[u2];
                    pr[8 + lane] = -INFINITY;
                }
            }
        }
        // fp32 tail rows (unless the tail pass owns them): warp w takes rows w, w + 16, ... of
        // every unit of the round; lanes split the channels
        if (a.tail_lse == nullptr) {
            const float isd = __fdiv_rn(1.0f, sqrtf((float)kDim));
            for (int us = 0; us < nr; ++us) {
                const int unit = unit_of(round0 + us);
                const int ntl = __ldcg(a.tail_len + unit / a.kv_heads);
                float tmax = -INFINITY;
                if (ntl > warp) {
                    float4 qv[4];
#pragma unroll
                    for (int h = 0; h < 4; ++h)
                        qv[h] = h < G ? *reinterpret_cast<const float4*>(a.q + ((size_t)unit * G + h) * kDim + 4 * lane)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
                    for (int j = warp; j < ntl; j += kW) {
                        const float4 kv = *reinterpret_cast<const float4*>(a.k_tail + ((size_t)unit * a.tail_cap + j) *
                                                                                           kDim + 4 * lane);
#pragma unroll
                        for (int h = 0; h < 4; ++h) {
                            if (h < G) {
                                float d = kv.x * qv[h].x + kv.y * qv[h].y + kv.z * qv[h].z + kv.w * qv[h].w;
#pragma unroll
                                for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                                d *= isd;
                                if (lane == 0) sm.tail_s[(us * 4 + h) * kTailMax + j] = d;
                                if ((lane & 3) == h) tmax = fmaxf(tmax, d);
                            }
                        }
                    }
                }
                if (lane < 4) sm.part[(warp * kMaxR + us) * 12 + 8 + lane] = tmax;
            }
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        if (threadIdx.x == 0 && round0 == 0) PSTRACE(1);
        // ---- softmax parameters per (unit, head) (calibrate.hpp:62-114) ----
        if (threadIdx.x < nr * 4) {
            const int us = threadIdx.x >> 2, h = threadIdx.x & 3;
            float gamma = INFINITY, delta = -INFINITY, tm = -INFINITY;
            for (int w2 = 0; w2 < kW; ++w2) {
                const float* pr = sm.part + (w2 * kMaxR + us) * 12;
                gamma = fminf(gamma, pr[h]);
                delta = fmaxf(delta, pr[4 + h]);
                tm = fmaxf(tm, pr[8 + h]);
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
            float* gp = sm.gpar + (us * 4 + h) * 4;
            gp[0] = live ? A * kLog2e : 0.0f;
            gp[1] = live ? (B - m) * kLog2e : -INFINITY;
            gp[2] = -m * kLog2e;
        }
        for (int i = threadIdx.x; i < kW * kMaxR * 4; i += kThreads) sm.wsum[i] = 0u;
        __syncthreads();

        // ---------------- phase B: chunks of V blocks, p from tensor memory ----------------
        {
            int slots[kStages];
#pragma unroll
            for (int i = 0; i < kStages; ++i) {
                slots[i] = grab(1, total);
                if (lane == 0 && slots[i] >= 0) issue(1, round0, slots[i], (ring_i + i) % kStages);
            }
            int vacc[16][4];
#pragma unroll
            for (int nc = 0; nc < 16; ++nc) vacc[nc][0] = vacc[nc][1] = vacc[nc][2] = vacc[nc][3] = 0;
            uint32_t wacc = 0;
            int cur_us = -1;
            float pa = 0.f, pb = 0.f;
            uint32_t* pw = sm.pw + warp * 2 * 12 * kPRow;
            const uint32_t* arow = pw + g * kPRow + t;
            auto flush = [&](int us) {  // this warp's sums of unit slot us into its image
                uint32_t* accb = sm.acc + us * 16 * 4 * 32;
#pragma unroll
                for (int nc = 0; nc < 16; ++nc)
#pragma unroll
                    for (int r = 0; r < 4; ++r) {
                        red_add_u32(accb + (nc * 4 + r) * 32 + lane, (uint32_t)vacc[nc][r]);
                        vacc[nc][r] = 0;
                    }
                uint32_t w = wacc;
                w += __shfl_xor_sync(0xffffffffu, w, 4);
                w += __shfl_xor_sync(0xffffffffu, w, 8);
                w += __shfl_xor_sync(0xffffffffu, w, 16);
                if (lane < 4) sm.wsum[(warp * kMaxR + us) * 4 + lane] += w;
                wacc = 0;
            };
            int pb_i = 0;  // p tile double buffer
            while (slots[0] >= 0) {
                const int it = slots[0];
                const int us = it / chunks_q, c = it - us * chunks_q;
                if (us != cur_us) {
                    if (cur_us >= 0) flush(cur_us);
                    cur_us = us;
                    pa = sm.gpar[(us * 4 + t) * 4 + 0];
                    pb = sm.gpar[(us * 4 + t) * 4 + 1];
                }
                const int slot = ring_i % kStages;
                mbar_wait(&full[slot], (ring_i / kStages) & 1);
                const uint8_t* buf = ring + slot * kChunkBytes + lane * (16 * BITS);
                const int tokq = c * Gm::kChunkTok;
                const int nvq = min(nq, n - quarter * nq);
                const int nv_chunk = min(Gm::kChunkTok, nvq - tokq);
                const int nblk = (nv_chunk + 31) / 32;
                const uint32_t tcol = tq + (uint32_t)(us * cols_unit + tokq / 8);
                auto p_write = [&](int blk, uint32_t* tile) {
                    float sc[4];
                    tmem_ld4(tcol + (uint32_t)(4 * blk), sc);
                    uint32_t v[4];
                    if (blk * 32 + 32 <= nv_chunk) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float pr = ex2(__fmaf_rn(sc[j], pa, pb));
                            v[j] = __float_as_uint(__fmaf_rn(pr, kPScale, kMagic));
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const float pr = blk * 32 + g + 8 * j < nv_chunk ? ex2(__fmaf_rn(sc[j], pa, pb)) : 0.0f;
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
                if (nblk > 0) p_write(0, pw + (pb_i & 1) * 12 * kPRow);
                __syncwarp();
#pragma unroll
                for (int blk = 0; blk < Gm::kSteps; ++blk) {
                    if (blk >= nblk) break;
                    const uint32_t* r0 = arow + ((pb_i + blk) & 1) * 12 * kPRow;
                    const uint32_t af0 = r0[0], af2 = r0[4];
                    const uint32_t af1 = g < 4 ? r0[8 * kPRow] : 0u;
                    const uint32_t af3 = g < 4 ? r0[8 * kPRow + 4] : 0u;
                    if (blk + 1 < nblk) p_write(blk + 1, pw + ((pb_i + blk + 1) & 1) * 12 * kPRow);
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
                pb_i += nblk;
#pragma unroll
                for (int i = 0; i + 1 < kStages; ++i) slots[i] = slots[i + 1];
                slots[kStages - 1] = grab(1, total);
                if (lane == 0 && slots[kStages - 1] >= 0) issue(1, round0, slots[kStages - 1], (ring_i + kStages) % kStages);
                ++ring_i;
            }
            if (cur_us >= 0) flush(cur_us);
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        if (threadIdx.x == 0 && round0 == 0) PSTRACE(4);
        // ---------------- epilogue: outputs of the round's units ----------------
        for (int idx = threadIdx.x; idx < nr * G * kDim; idx += kThreads) {
            const int us = idx / (G * kDim), rem = idx % (G * kDim);
            const int h = rem / kDim, ch = rem % kDim;
            const int unit = unit_of(round0 + us);
            constexpr int cpb = Gm::kCpb;
            const int s_slot = cpb - 1 - ch % cpb, rq = ch / cpb;
            const int gcol = rq / (2 * BITS), qq = rq % (2 * BITS);
            const int nc = qq * cpb + s_slot, tt = gcol >> 1, rlo = gcol & 1;
            uint32_t* accb = sm.acc + us * 16 * 4 * 32;
            uint32_t pl[3];
#pragma unroll
            for (int plane = 0; plane < 3; ++plane) {
                const int row = plane * 4 + h;
                const int gg = row & 7, r = ((row >> 3) << 1) | rlo;
                uint32_t* wp = accb + (nc * 4 + r) * 32 + gg * 4 + tt;
                pl[plane] = *wp;
            }
            const float V = __fmaf_rn((float)pl[2], 65536.0f, __fmaf_rn((float)pl[1], 256.0f, (float)pl[0])) *
                            __int_as_float((127 - s_slot * BITS) << 23);
            unsigned long long ws = 0;
            for (int w2 = 0; w2 < kW; ++w2) ws += sm.wsum[(w2 * kMaxR + us) * 4 + h];
            const float wv = (float)ws;
            const float v_a = __ldg(a.v_alpha + (size_t)unit * kDim + ch);
            const float v_b = __ldg(a.v_beta + (size_t)unit * kDim + ch);
            constexpr float kInvLevelsV = 1.0f / (float)((1u << BITS) - 1u);
            const float v_step = fmaxf(__fsub_rn(v_b, v_a) * kInvLevelsV, 0.0f);
            float num = __fmaf_rn(v_step, V, v_a * wv), den = wv;
            const float mh = sm.gpar[(us * 4 + h) * 4 + 2];
            const int ntl = a.tail_lse == nullptr ? __ldcg(a.tail_len + unit / a.kv_heads) : 0;
            const float* vt = a.v_tail + (size_t)unit * a.tail_cap * kDim + ch;
            const float* ts = sm.tail_s + (us * 4 + h) * kTailMax;
            int j = 0;
            for (; j + 8 <= ntl; j += 8) {
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
            for (; j < ntl; ++j) {
                const float pt = ex2(__fmaf_rn(ts[j], kLog2e, mh)) * kPScale;
                den += pt;
                num = __fmaf_rn(pt, __ldg(vt + (size_t)j * kDim), num);
            }
            a.out[((size_t)unit * G + h) * kDim + ch] = num / den;
            if (a.tail_lse && ch == 0) a.tail_lse[(size_t)unit * G + h] = log2f(den) - kLog2PScale - mh;
        }
        __syncthreads();
        // next round: zero the images and the queues
        for (int i = threadIdx.x; i < kMaxR * 16 * 4 * 32; i += kThreads) sm.acc[i] = 0u;
        if (threadIdx.x < 8) sm.qctr[threadIdx.x] = 0;
        __syncthreads();
    }
    if (threadIdx.x == 0) PSTRACE(5);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(*sm.tmem_slot));
    }
}

template <int BITS>
cudaError_t launch_bits(const DecodeArgs& a, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int grid = (int)std::min<size_t>(a.units, (size_t)sms);
    const int nq = (int)((a.n_vis + 3) / 4);
    constexpr int ct = kChunkBytes / (16 * BITS);
    const int cols_unit = (nq + ct - 1) / ct * ct / 32 * 4;
    PsParams p{a, std::min(kMaxR, 512 / cols_unit)};
    const size_t smem = ps_smem_bytes();
    auto kern = decode_ps_kernel<BITS>;
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

}  // namespace

bool decode_ps_supported(const DecodeArgs& a) {
    if (a.dim != (size_t)kDim || a.n_vis == 0 || a.units == 0 || !a.v_codes_x) return false;
    if (a.word_bits != 8 && a.word_bits != 16 && a.word_bits != 32) return false;
    if (a.bits != 1 && a.bits != 2 && a.bits != 4) return false;
    if (a.group < 1 || a.group > 4) return false;
    // a quarter's token range must start on a 32-token vx block: n / 4 a multiple of 32
    if (a.n_vis % 128 != 0 || a.n_vis > 4096) return false;
    if (a.tail_cap > (size_t)kTailMax && a.tail_lse == nullptr) return false;
    return ps_smem_bytes() <= 227 * 1024;
}

cudaError_t launch_decode_ps(const DecodeArgs& a, cudaStream_t s) {
    switch (a.bits) {
        case 1: return launch_bits<1>(a, s);
        case 2: return launch_bits<2>(a, s);
        case 4: return launch_bits<4>(a, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace kvqb
