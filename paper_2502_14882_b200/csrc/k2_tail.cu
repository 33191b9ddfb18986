// k2_tail.cu — the fp32 tail pass: attention of the G query heads of every
// unit over its dense fp32 tail rows (kvcache.hpp:286-304, naive_qk / naive_wv on the
// generated tokens), merged with the quantized-segment decode by log-sum-exp.
//
// The reference runs ONE softmax over [g(vis) | tail] (calibrate.hpp:100-114). Split in
// two passes this is exact algebra: with the decode's normalised output o_v and base-2
// log-sum-exp l_v of its (calibrated) vis weights, and this pass's running max M_t, sum
// D_t = sum_j 2^(t_j - M_t) and numerator N_t = sum_j 2^(t_j - M_t) v_j (t_j = score_j log2 e):
//   out = (o_v 2^(l_v - X) + N_t 2^(M_t - X)) / (2^(l_v - X) + D_t 2^(M_t - X)),
//   X = max(l_v, M_t + log2 D_t).
// Without a quantized prefill (build_full_precision) l_v = -inf and this pass is the whole
// decode.
//
// Layout and work split. A unit's tail is [tail_cap][128] fp32 for K and for V (rows
// appended by K3). The rows of a unit are split over a cluster of S CTAs (S sized so the
// grid covers the SMs); inside a CTA warp w takes rows w, w + 8, ...; lane l owns channels
// 4l..4l+3 of every row (one coalesced 512-byte row read per warp and tensor). A warp keeps
// its own online softmax (running max, sum, 4 numerators per head and lane); warps merge in
// shared memory, ranks through DSMEM into rank 0, which alone waits for the decode grid
// (programmatic dependent launch: everything before the merge overlaps the decode's tail
// end) and writes the output. HBM-bound: 1024 algorithmic bytes per tail row and unit.
#include <cooperative_groups.h>

#include "kvq_internal.cuh"

namespace cg = cooperative_groups;

namespace kvqb {

namespace {

constexpr int kDim = 128;
constexpr int kWarps = 8;
constexpr int kRows = 4;  // rows in flight per warp (4 K + 4 V float4 loads per lane)
constexpr int kMaxCluster = 8;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cluster_sync_all() {
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

struct TailParams {
    const float* q;         // [units][G][128]
    const float* k_tail;    // [units][tail_cap][128]
    const float* v_tail;
    const int* tail_len;    // [batch]
    const float* lse;       // [units][G] decode's base-2 log-sum-exp; nullptr: no quantized part
    float* out;             // [units][G][128]: the decode's output in, the merged output out
    size_t kv_heads, tail_cap;
    int S, rows_per_cta;
    float scale;            // log2(e) / sqrt(d)
};

// Per CTA: warp partials, then the CTA's merged (max, sum, 128 numerators) per head, which
// rank 0 reads from every rank through DSMEM.
template <int G>
struct TailSmem {
    float wm[kWarps][G];
    float wd[kWarps][G];
    float wn[kWarps][G][kDim];
    float pm[G];
    float pd[G];
    float pn[G][kDim];
};

__device__ __forceinline__ float ld_cluster(const float* local_ptr, int rank) {
    uint32_t addr;
    float v;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_addr(local_ptr)), "r"(rank));
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
    return v;
}

template <int G>
__global__ void __launch_bounds__(kWarps * 32) tail_kernel(const TailParams p) {
    __shared__ TailSmem<G> sm;
    const int S = p.S;
    const int rank = S > 1 ? (int)cg::this_cluster().block_rank() : 0;
    const size_t unit = blockIdx.x / S;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // tail_len was final before the decode grid passed its own dependency wait, and this
    // grid starts only after every decode CTA did (griddepcontrol.launch_dependents).
    const int len = __ldcg(p.tail_len + unit / p.kv_heads);
    const int r0 = rank * p.rows_per_cta, r1 = min(len, r0 + p.rows_per_cta);

    float4 q[G];
#pragma unroll
    for (int h = 0; h < G; ++h)
        q[h] = __ldg(reinterpret_cast<const float4*>(p.q + (unit * G + h) * kDim) + lane);
    float m[G], d[G];
    float4 acc[G];
#pragma unroll
    for (int h = 0; h < G; ++h) m[h] = -INFINITY, d[h] = 0.0f, acc[h] = make_float4(0.f, 0.f, 0.f, 0.f);

    const float4* kt = reinterpret_cast<const float4*>(p.k_tail + unit * p.tail_cap * kDim) + lane;
    const float4* vt = reinterpret_cast<const float4*>(p.v_tail + unit * p.tail_cap * kDim) + lane;
    for (int j0 = r0 + warp; j0 < r1; j0 += kWarps * kRows) {
        float4 kv[kRows], vv[kRows];
#pragma unroll
        for (int i = 0; i < kRows; ++i) {
            const int j = j0 + i * kWarps;
            kv[i] = j < r1 ? __ldcs(kt + (size_t)j * (kDim / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
            vv[i] = j < r1 ? __ldcs(vt + (size_t)j * (kDim / 4)) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int h = 0; h < G; ++h) {
            float t[kRows];
#pragma unroll
            for (int i = 0; i < kRows; ++i) {
                float s = kv[i].x * q[h].x;
                s = __fmaf_rn(kv[i].y, q[h].y, s);
                s = __fmaf_rn(kv[i].z, q[h].z, s);
                s = __fmaf_rn(kv[i].w, q[h].w, s);
                t[i] = s;
            }
#pragma unroll
            for (int o = 16; o; o >>= 1)
#pragma unroll
                for (int i = 0; i < kRows; ++i) t[i] += __shfl_xor_sync(0xffffffffu, t[i], o);
            float mx = m[h];
#pragma unroll
            for (int i = 0; i < kRows; ++i) {
                t[i] = j0 + i * kWarps < r1 ? t[i] * p.scale : -INFINITY;
                mx = fmaxf(mx, t[i]);
            }
            if (mx > m[h]) {  // warp-uniform: rescale the running sums
                const float c = ex2(m[h] - mx);
                d[h] *= c;
                acc[h].x *= c, acc[h].y *= c, acc[h].z *= c, acc[h].w *= c;
                m[h] = mx;
            }
#pragma unroll
            for (int i = 0; i < kRows; ++i) {
                const float w = ex2(t[i] - mx);
                d[h] += w;
                acc[h].x = __fmaf_rn(w, vv[i].x, acc[h].x);
                acc[h].y = __fmaf_rn(w, vv[i].y, acc[h].y);
                acc[h].z = __fmaf_rn(w, vv[i].z, acc[h].z);
                acc[h].w = __fmaf_rn(w, vv[i].w, acc[h].w);
            }
        }
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        if (lane == 0) sm.wm[warp][h] = m[h], sm.wd[warp][h] = d[h];
        *reinterpret_cast<float4*>(&sm.wn[warp][h][4 * lane]) = acc[h];
    }
    __syncthreads();
    // CTA merge: thread per (head, channel) item.
    constexpr int kItems = (G * kDim + kWarps * 32 - 1) / (kWarps * 32);
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int idx = threadIdx.x + it * kWarps * 32;
        if (idx >= G * kDim) break;
        const int h = idx / kDim, ch = idx % kDim;
        float M = -INFINITY;
        for (int w = 0; w < kWarps; ++w) M = fmaxf(M, sm.wm[w][h]);
        float D = 0.0f, N = 0.0f;
        if (M != -INFINITY)
            for (int w = 0; w < kWarps; ++w) {
                const float c = ex2(sm.wm[w][h] - M);  // 0 for an empty warp (-inf)
                D = __fmaf_rn(sm.wd[w][h], c, D);
                N = __fmaf_rn(sm.wn[w][h][ch], c, N);
            }
        sm.pn[h][ch] = N;
        if (ch == 0) sm.pm[h] = M, sm.pd[h] = D;
    }
    if (S > 1) cluster_sync_all();  // every rank's partial is readable
    else __syncthreads();
    // Rank 0 folds the ranks in order (registers), then lets them go.
    float RM[kItems], RD[kItems], RN[kItems];
    if (rank == 0) {
#pragma unroll
        for (int it = 0; it < kItems; ++it) {
            const int idx = threadIdx.x + it * kWarps * 32;
            RM[it] = -INFINITY, RD[it] = 0.0f, RN[it] = 0.0f;
            if (idx >= G * kDim) continue;
            const int h = idx / kDim, ch = idx % kDim;
            float mr[kMaxCluster];
            for (int r = 0; r < S; ++r) {
                mr[r] = S > 1 ? ld_cluster(&sm.pm[h], r) : sm.pm[h];
                RM[it] = fmaxf(RM[it], mr[r]);
            }
            if (RM[it] == -INFINITY) continue;
            for (int r = 0; r < S; ++r) {
                const float c = ex2(mr[r] - RM[it]);
                RD[it] = __fmaf_rn(S > 1 ? ld_cluster(&sm.pd[h], r) : sm.pd[h], c, RD[it]);
                RN[it] = __fmaf_rn(S > 1 ? ld_cluster(&sm.pn[h][ch], r) : sm.pn[h][ch], c, RN[it]);
            }
        }
    }
    if (S > 1) cluster_sync_all();  // remote shared memory stays valid until rank 0 has read it
    if (rank != 0) return;
    // The decode's output and log-sum-exp are complete from here on.
    asm volatile("griddepcontrol.wait;" ::: "memory");
#pragma unroll
    for (int it = 0; it < kItems; ++it) {
        const int idx = threadIdx.x + it * kWarps * 32;
        if (idx >= G * kDim || RM[it] == -INFINITY) continue;  // no tail rows: the decode's output stands
        const int h = idx / kDim, ch = idx % kDim;
        const float M = RM[it], D = RD[it], N = RN[it];
        float* o = p.out + (unit * G + h) * kDim + ch;
        const float lv = p.lse ? p.lse[unit * G + h] : -INFINITY;
        if (lv == -INFINITY) {
            *o = N / D;
        } else {
            const float X = fmaxf(lv, M + __log2f(D));
            const float wv = ex2(lv - X), wt = ex2(M - X);  // tail weight in total: D 2^(M - X)
            *o = __fmaf_rn(*o, wv, N * wt) / __fmaf_rn(D, wt, wv);
        }
    }
}

template <int G>
cudaError_t launch_g(const TailParams& p, size_t units, cudaStream_t s, bool pdl) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)(units * p.S));
    cfg.blockDim = dim3(kWarps * 32);
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
    return cudaLaunchKernelEx(&cfg, tail_kernel<G>, p);
}

}  // namespace

bool decode_tail_supported(const DecodeArgs& a) {
    return a.dim == (size_t)kDim && a.group >= 1 && a.group <= 8 && a.tail_cap > 0 && a.units > 0;
}

// Cluster size: enough CTAs for ~4 per SM, at least 64 rows per CTA, at most 8 ranks.
int tail_split(size_t units, size_t tail_cap) {
    const size_t want = (4 * 148 + units - 1) / units;
    size_t s = std::min<size_t>(want, (tail_cap + 63) / 64);
    return (int)std::max<size_t>(1, std::min<size_t>(s, kMaxCluster));
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
    p.S = tail_split(a.units, a.tail_cap);
    p.rows_per_cta = (int)((a.tail_cap + p.S - 1) / p.S);
    p.scale = kLog2e / sqrtf((float)kDim);
    cudaError_t e;
    switch (a.group) {
        case 1: e = launch_g<1>(p, a.units, s, after_decode); break;
        case 2: e = launch_g<2>(p, a.units, s, after_decode); break;
        case 3: e = launch_g<3>(p, a.units, s, after_decode); break;
        case 4: e = launch_g<4>(p, a.units, s, after_decode); break;
        case 5: e = launch_g<5>(p, a.units, s, after_decode); break;
        case 6: e = launch_g<6>(p, a.units, s, after_decode); break;
        case 7: e = launch_g<7>(p, a.units, s, after_decode); break;
        case 8: e = launch_g<8>(p, a.units, s, after_decode); break;
        default: return cudaErrorInvalidValue;
    }
    note_launch();
    return e;
}

}  // namespace kvqb
