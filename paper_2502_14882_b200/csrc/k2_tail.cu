// k2_tail.cu — the fp32 tail pass: attention of the G query heads of every
// unit over its dense fp32 tail rows (kvcache.hpp:286-304, naive_qk / naive_wv on the
// generated tokens), merged with the quantized-segment decode by log-sum-exp.
//
// The reference runs ONE softmax over [g(vis) | tail] (calibrate.hpp:100-114). Split in
// two passes this is exact algebra: with the decode's normalised output o_v and base-2
// log-sum-exp l_v of its (calibrated) vis weights, and this pass's reference max M_t, sum
// D_t = sum_j 2^(t_j - M_t) and numerator N_t = sum_j 2^(t_j - M_t) v_j (t_j = score_j log2 e):
//   out = (o_v 2^(l_v - X) + N_t 2^(M_t - X)) / (2^(l_v - X) + D_t 2^(M_t - X)),
//   X = max(l_v, M_t + log2 D_t).
// Without a quantized prefill (build_full_precision) l_v = -inf and this pass is the whole
// decode.
//
// Data movement. A unit's tail is [tail_cap][128] fp32 for K and for V (rows appended by
// K3). The unit's rows are split over a cluster of S CTAs; a CTA's rows are cut in 4-row
// stages (2 KB of K + 2 KB of V, contiguous) dealt round-robin to its 8 warps, and every
// warp streams its stages through its own ring of cp.async.bulk copies (kStages deep,
// mbarrier completion) - the loads never wait on the math, so HBM sees a steady stream.
//
// Math per stage, per warp (lane l owns channels 4l..4l+3):
//   scores  4 rows x GP heads partial dots, then ONE butterfly reduce-scatter across the
//           warp (4 GP values -> one complete score per lane, 16 or 31 shuffles instead of
//           5 per score); lane L holds (row i, head h) = idx / GP, idx % GP, idx = L >> 1
//           (GP = 4) or L (GP = 8);
//   softmax lazy running max per head (warp-uniform): a score is exponentiated against
//           the current reference m as long as it stays below m + kSlack (so weights stay
//           <= 2^kSlack); one vote detects the rare stage that raises it and rescales;
//   values  each lane exponentiates its own score once; the weights are broadcast back
//           (one shuffle per (row, head)) into 4 FMAs per head and row.
// Warps merge in shared memory, ranks through DSMEM into rank 0, which alone waits for the
// decode grid (programmatic dependent launch: the streaming overlaps the decode's tail
// end) and writes the output. HBM-bound: 1024 algorithmic bytes per tail row and unit.
#include "kvq_internal.cuh"
#include "kvq_ptx.cuh"

namespace kvqb {

namespace {

using namespace ptx;

constexpr int kDim = 128;
#ifndef KVQ_TAIL_WARPS  // (tuning builds only: tools/gpu_tail_tune.sh)
#define KVQ_TAIL_WARPS 8
#endif
#ifndef KVQ_TAIL_STAGES
#define KVQ_TAIL_STAGES 3
#endif
constexpr int kWarps = KVQ_TAIL_WARPS;
constexpr int kStageRows = 4;
constexpr int kRowBytes = kDim * 4;
constexpr int kStageBytes = 2 * kStageRows * kRowBytes;  // K rows then V rows
constexpr int kStages = KVQ_TAIL_STAGES;                 // ring depth per warp
constexpr int kMaxCluster = 8;
constexpr float kLog2e = 1.4426950408889634f;
constexpr float kSlack = 8.0f;  // weights stay <= 2^8 against a stale reference max

struct TailParams {
    const float* q;         // [units][G][128]
    const float* k_tail;    // [units][tail_cap][128]
    const float* v_tail;
    const int* tail_len;    // [batch]
    const float* lse;       // [units][G] decode's base-2 log-sum-exp; nullptr: no quantized part
    float* out;             // [units][G][128]: the decode's output in, the merged output out
    float* part;            // nullable: write (M, D, N[128]) per (unit, head) here instead of
                            // merging (the concurrent schedule; tail_merge_kernel merges)
    size_t kv_heads, tail_cap;
    int G, S;
    float scale;            // log2(e) / sqrt(d)
};

template <int GP>
struct TailSmem {
    static constexpr int kRing = kWarps * kStages * kStageBytes;
    // the ring; after the stream drains, the warp partials alias it
    alignas(128) uint8_t ring[kRing];
    uint64_t full[kWarps][kStages];
    float wm[kWarps][GP];
    float wd[kWarps][GP];
    float pm[GP];
    float pd[GP];
    float pn[GP][kDim];
    __device__ float* wn() { return reinterpret_cast<float*>(ring); }  // [kWarps][GP][kDim]
};
static_assert(kWarps * 8 * kDim * 4 <= kWarps * kStages * kStageBytes, "warp partials must fit in the ring");

// Reduce-scatter of N = 4 GP per-lane partial sums: afterwards lane L holds the complete
// warp sum of value idx(L) (idx = L >> 1 for N = 16, L for N = 32).
template <int N>
__device__ __forceinline__ float reduce_scatter(float (&a)[N], int lane) {
    static_assert(N == 16 || N == 32, "4 rows x 4 or 8 heads");
    // N = 32: lane bits 4..0 select halves; N = 16: lane bits 4..1, then bit 0 sums the pair
    constexpr int kSteps = N == 32 ? 5 : 4;
#pragma unroll
    for (int st = 0; st < kSteps; ++st) {
        const int o = 16 >> st, half = N >> (st + 1);
        const bool b = (lane & o) != 0;
#pragma unroll
        for (int k = 0; k < half; ++k) {
            const float keep = b ? a[k + half] : a[k];
            const float send = b ? a[k] : a[k + half];
            a[k] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    float r = a[0];
    if (N == 16) r += __shfl_xor_sync(0xffffffffu, r, 1);
    return r;
}

template <int GP>
__global__ void __launch_bounds__(kWarps * 32) tail_kernel(const TailParams p) {
    constexpr int N = kStageRows * GP;
    extern __shared__ __align__(128) uint8_t smem_raw[];
    TailSmem<GP>& sm = *reinterpret_cast<TailSmem<GP>*>(smem_raw);
    const int S = p.S, G = p.G;
    const int rank = S > 1 ? (int)cluster_rank() : 0;
    const size_t unit = blockIdx.x / S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // tail_len was final before the decode grid passed its own dependency wait, and this
    // grid starts only after every decode CTA did (griddepcontrol.launch_dependents).
    const int len = __ldcg(p.tail_len + unit / p.kv_heads);
    // the request's rows (not its capacity) split evenly over the ranks, in whole stages
    const int rpc = ((len + S - 1) / S + kStageRows - 1) / kStageRows * kStageRows;
    const int r0 = rank * rpc, r1 = min(len, r0 + rpc);
    const int nst = r1 > r0 ? (r1 - r0 + kStageRows - 1) / kStageRows : 0;  // CTA stages
    const int my = nst > warp ? (nst - warp + kWarps - 1) / kWarps : 0;      // this warp's

    uint8_t* ring = sm.ring + warp * kStages * kStageBytes;
    uint64_t* full = sm.full[warp];
    const float* kbase = p.k_tail + unit * p.tail_cap * kDim;
    const float* vbase = p.v_tail + unit * p.tail_cap * kDim;
    auto issue = [&](int k) {  // lane 0: this warp's k-th stage (CTA stage warp + 8k)
        const int row = r0 + (warp + kWarps * k) * kStageRows;
        const uint32_t bytes = (uint32_t)(min(kStageRows, r1 - row) * kRowBytes);
        uint8_t* dst = ring + (k % kStages) * kStageBytes;
        mbar_expect_tx(&full[k % kStages], 2 * bytes);
        bulk_g2s(dst, kbase + (size_t)row * kDim, bytes, &full[k % kStages]);
        bulk_g2s(dst + kStageRows * kRowBytes, vbase + (size_t)row * kDim, bytes, &full[k % kStages]);
    };
    if (lane == 0) {
        for (int i = 0; i < kStages; ++i) mbar_init(&full[i], 1);
        mbar_init_fence();
        for (int k = 0; k < min(kStages, my); ++k) issue(k);
    }
    __syncwarp();

    float4 q[GP];
#pragma unroll
    for (int h = 0; h < GP; ++h)
        q[h] = h < G ? __ldg(reinterpret_cast<const float4*>(p.q + (unit * G + h) * kDim) + lane)
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    const int my_idx = N == 32 ? lane : lane >> 1;  // (row, head) of this lane's score
    const int my_row = my_idx / GP, my_head = my_idx % GP;
    float m[GP];
    float4 acc[GP];
#pragma unroll
    for (int h = 0; h < GP; ++h) m[h] = -INFINITY, acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);
    float mh = -INFINITY;  // m[my_head]
    float dsum = 0.0f;     // sum of this lane's own weights (head my_head)

    for (int k = 0; k < my; ++k) {
        mbar_wait(&full[k % kStages], (uint32_t)((k / kStages) & 1));
        const float* kr = reinterpret_cast<const float*>(ring + (k % kStages) * kStageBytes);
        const float* vr = kr + kStageRows * kDim;
        const int rows = min(kStageRows, r1 - (r0 + (warp + kWarps * k) * kStageRows));
        float part[N];
#pragma unroll
        for (int i = 0; i < kStageRows; ++i) {
            const float4 kv = *reinterpret_cast<const float4*>(kr + i * kDim + 4 * lane);
#pragma unroll
            for (int h = 0; h < GP; ++h) {
                float s = kv.x * q[h].x;
                s = __fmaf_rn(kv.y, q[h].y, s);
                s = __fmaf_rn(kv.z, q[h].z, s);
                part[i * GP + h] = __fmaf_rn(kv.w, q[h].w, s);
            }
        }
        float t = reduce_scatter<N>(part, lane) * p.scale;
        if (my_row >= rows) t = -INFINITY;  // rows past the tail (stale shared memory)
        // lazy max: rescale only when a score passes its head's reference by kSlack
        if (__any_sync(0xffffffffu, my_head < G && t > mh + kSlack)) {
            float nm = fmaxf(mh, t);  // new max of my head over the stage's rows (lane bits 3, 4)
            nm = fmaxf(nm, __shfl_xor_sync(0xffffffffu, nm, 8));
            nm = fmaxf(nm, __shfl_xor_sync(0xffffffffu, nm, 16));
            dsum *= ex2(mh - nm);
#pragma unroll
            for (int h = 0; h < GP; ++h) {
                const float nmh = __shfl_sync(0xffffffffu, nm, N == 32 ? h : 2 * h);
                const float c = ex2(m[h] - nmh);  // 0 on the first stage (m = -inf)
                acc[h].x *= c, acc[h].y *= c, acc[h].z *= c, acc[h].w *= c;
                m[h] = nmh;
            }
            mh = nm;
        }
        const float w = ex2(t - mh);
        dsum += w;
#pragma unroll
        for (int i = 0; i < kStageRows; ++i) {
            if (i >= rows) break;  // warp-uniform: no stale (possibly NaN) rows past the tail
            const float4 vv = *reinterpret_cast<const float4*>(vr + i * kDim + 4 * lane);
#pragma unroll
            for (int h = 0; h < GP; ++h) {
                const float wh = __shfl_sync(0xffffffffu, w, N == 32 ? i * GP + h : 2 * (i * GP + h));
                acc[h].x = __fmaf_rn(wh, vv.x, acc[h].x);
                acc[h].y = __fmaf_rn(wh, vv.y, acc[h].y);
                acc[h].z = __fmaf_rn(wh, vv.z, acc[h].z);
                acc[h].w = __fmaf_rn(wh, vv.w, acc[h].w);
            }
        }
        __syncwarp();  // every lane is done with this slot
        if (lane == 0 && k + kStages < my) issue(k + kStages);
    }
    // warp partials: per-head sum over the lanes that own the head (one copy of each score)
    if (N == 16 && (lane & 1)) dsum = 0.0f;
    dsum += __shfl_xor_sync(0xffffffffu, dsum, 8);
    dsum += __shfl_xor_sync(0xffffffffu, dsum, 16);
    __syncthreads();  // every warp's stream is drained: the ring becomes the partials
    float* wn = sm.wn();
#pragma unroll
    for (int h = 0; h < GP; ++h) {
        if (lane == (N == 32 ? h : 2 * h)) sm.wm[warp][h] = m[h], sm.wd[warp][h] = dsum;
        *reinterpret_cast<float4*>(wn + (warp * GP + h) * kDim + 4 * lane) = acc[h];
    }
    __syncthreads();
    // CTA merge: thread per (head, channel) item.
    constexpr int kItems = (GP * kDim + kWarps * 32 - 1) / (kWarps * 32);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int idx = threadIdx.x + it * kWarps * 32;
        const int h = idx / kDim, ch = idx % kDim;
        if (h >= G) break;
        float M = -INFINITY;
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm.wm[w][h]);
        float D = 0.0f, Nn = 0.0f;
        if (M != -INFINITY)
            for (int w = 0; w < kWarps; ++w) {
                const float c = ex2(sm.wm[w][h] - M);  // 0 for an empty warp (-inf)
                D = __fmaf_rn(sm.wd[w][h], c, D);
                Nn = __fmaf_rn(wn[(w * GP + h) * kDim + ch], c, Nn);
            }
        sm.pn[h][ch] = Nn;
        if (ch == 0) sm.pm[h] = M, sm.pd[h] = D;
    }
    if (S > 1) cluster_sync();  // every rank's partial is readable
    else __syncthreads();
    // Rank 0 folds the ranks in order (registers), then lets them go.
    float RM[kItems], RD[kItems], RN[kItems];
#pragma unroll
    for (int it = 0; it < kItems; ++it) RM[it] = -INFINITY, RD[it] = 0.0f, RN[it] = 0.0f;
    if (rank == 0) {
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const int idx = threadIdx.x + it * kWarps * 32;
            const int h = idx / kDim, ch = idx % kDim;
            if (h >= G) break;
            float mr[kMaxCluster];
            for (int r = 0; r < S; ++r) {
                mr[r] = S > 1 ? ld_cluster_f32(&sm.pm[h], r) : sm.pm[h];
                RM[it] = fmaxf(RM[it], mr[r]);
            }
            if (RM[it] == -INFINITY) continue;
            for (int r = 0; r < S; ++r) {
                const float c = ex2(mr[r] - RM[it]);
                RD[it] = __fmaf_rn(S > 1 ? ld_cluster_f32(&sm.pd[h], r) : sm.pd[h], c, RD[it]);
                RN[it] = __fmaf_rn(S > 1 ? ld_cluster_f32(&sm.pn[h][ch], r) : sm.pn[h][ch], c, RN[it]);
            }
        }
    }
    if (S > 1) cluster_sync();  // remote shared memory stays valid until rank 0 has read it
    if (rank != 0) return;
    if (p.part) {  // concurrent schedule: hand the partials to tail_merge_kernel
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const int idx = threadIdx.x + it * kWarps * 32;
            const int h = idx / kDim, ch = idx % kDim;
            if (h >= G) break;
            float* rec = p.part + (unit * G + h) * (kDim + 2);
            rec[2 + ch] = RN[it];
            if (ch == 0) rec[0] = RM[it], rec[1] = RD[it];
        }
        return;
    }
    griddep_wait();  // the decode's output and log-sum-exp are complete from here on
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int idx = threadIdx.x + it * kWarps * 32;
        const int h = idx / kDim, ch = idx % kDim;
        if (h >= G) continue;
        if (RM[it] == -INFINITY) {  // no tail rows: the decode's output stands; with no decode
            if (!p.lse) p.out[(unit * G + h) * kDim + ch] = 0.0f;  // (empty cache) the row is 0
            continue;                                         // (softmax_inplace no-op, naive_wv zeros)
        }
        const float M = RM[it], D = RD[it], Nn = RN[it];
        float* o = p.out + (unit * G + h) * kDim + ch;
        const float lv = p.lse ? p.lse[unit * G + h] : -INFINITY;
        if (lv == -INFINITY) {
            *o = Nn / D;
        } else {
            const float X = fmaxf(lv, M + __log2f(D));
            const float wv = ex2(lv - X), wt = ex2(M - X);  // tail weight in total: D 2^(M - X)
            *o = __fmaf_rn(*o, wv, Nn * wt) / __fmaf_rn(D, wt, wv);
        }
    }
}

// Concurrent schedule, last step: merge the tail pass's partials into the decode's output
// (one thread per (unit, head, channel); the same log-sum-exp algebra as the in-pass merge).
__global__ void __launch_bounds__(256) tail_merge_kernel(const float* __restrict__ part, const float* __restrict__ lse,
                                                         float* __restrict__ out, size_t rows) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;  // (unit * G + h) * 128 + ch
    if (i >= rows * kDim) return;
    const size_t row = i / kDim, ch = i % kDim;
    const float* rec = part + row * (kDim + 2);
    const float M = rec[0];
    if (M == -INFINITY) {  // no tail rows: the decode's output stands (an empty cache: 0)
        if (!lse) out[i] = 0.0f;
        return;
    }
    const float D = rec[1], Nn = rec[2 + ch];
    const float lv = lse ? lse[row] : -INFINITY;
    if (lv == -INFINITY) {
        out[i] = Nn / D;
    } else {
        const float X = fmaxf(lv, M + __log2f(D));
        const float wv = ex2(lv - X), wt = ex2(M - X);
        out[i] = __fmaf_rn(out[i], wv, Nn * wt) / __fmaf_rn(D, wt, wv);
    }
}

template <int GP>
cudaError_t launch_gp(const TailParams& p, size_t units, cudaStream_t s, bool pdl) {
    auto kern = tail_kernel<GP>;
    const size_t smem = sizeof(TailSmem<GP>);
    static unsigned attr_done = 0;  // per instantiation, bit per device
    const cudaError_t ea = once_per_device(
        attr_done, [&] { return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); });
    if (ea != cudaSuccess) return ea;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(units * p.S));
    cfg.blockDim = dim3(kWarps * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attrs[2];
    attrs[0].id = cudaLaunchAttributeClusterDimension;
    attrs[0].val.clusterDim.x = (unsigned)p.S;
    attrs[0].val.clusterDim.y = 1;
    attrs[0].val.clusterDim.z = 1;
    attrs[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attrs[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attrs;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace

bool decode_tail_supported(const DecodeArgs& a) {
    return a.dim == (size_t)kDim && a.group >= 1 && a.group <= 8 && a.tail_cap > 0 && a.units > 0;
}

#ifndef KVQ_TAIL_CTAS_PER_SM
#define KVQ_TAIL_CTAS_PER_SM 2
#endif
// Cluster size: split a unit only when the units alone leave SMs idle (~2 CTAs per SM;
// splitting further costs more in per-CTA setup and merges than it gains, r01 sweep in
// profiles/r01_tail_tune.txt), at least 64 rows per CTA, at most 8 ranks.
int tail_split(size_t units, size_t tail_cap) {
    const size_t want = (KVQ_TAIL_CTAS_PER_SM * 148 + units - 1) / units;
    size_t s = std::min<size_t>(want, (tail_cap + 63) / 64);
    return (int)std::max<size_t>(1, std::min<size_t>(s, kMaxCluster));
}

cudaError_t launch_decode_tail_partials(const DecodeArgs& a, float* part, cudaStream_t s) {
    TailParams p{};
    p.q = a.q;
    p.k_tail = a.k_tail;
    p.v_tail = a.v_tail;
    p.tail_len = a.tail_len;
    p.out = a.out;
    p.part = part;
    p.kv_heads = a.kv_heads;
    p.tail_cap = a.tail_cap;
    p.G = (int)a.group;
    p.S = tail_split(a.units, a.tail_cap);
    p.scale = kLog2e / sqrtf((float)kDim);
    // every row's M starts at -inf: rows past a request's tail length are skipped by the merge
    const cudaError_t e = a.group <= 4 ? launch_gp<4>(p, a.units, s, false) : launch_gp<8>(p, a.units, s, false);
    note_launch();
    return e;
}

cudaError_t launch_tail_merge(const DecodeArgs& a, const float* part, cudaStream_t s) {
    const size_t rows = a.units * a.group;
    tail_merge_kernel<<<(unsigned)((rows * kDim + 255) / 256), 256, 0, s>>>(part, a.tail_lse, a.out, rows);
    note_launch();
    return cudaGetLastError();
}

cudaError_t launch_decode_tail(const DecodeArgs& a, bool after_decode, cudaStream_t s) {
    TailParams p{};
    p.q = a.q;
    p.k_tail = a.k_tail;
    p.v_tail = a.v_tail;
    p.tail_len = a.tail_len;
    p.lse = after_decode ? a.tail_lse : nullptr;
    p.out = a.out;
    p.kv_heads = a.kv_heads;
    p.tail_cap = a.tail_cap;
    p.G = (int)a.group;
    p.S = tail_split(a.units, a.tail_cap);
    p.scale = kLog2e / sqrtf((float)kDim);
    const cudaError_t e = a.group <= 4 ? launch_gp<4>(p, a.units, s, after_decode)
                                       : launch_gp<8>(p, a.units, s, after_decode);
    note_launch();
    return e;
}

}  // namespace kvqb
