// Microbenchmark: tcgen05.mma throughput at small N, per CTA and per SM.
// kind::i8 and kind::f16, M = 128, N in {8..256}, A and B from shared memory (K-major,
// no swizzle), back-to-back MMAs into rotating accumulators (4 independent D tiles),
// c CTAs per SM issuing concurrently. Reports cycles per MMA per CTA and SM-wide MAC/clk.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// kind::i8: D s32 (bits 4-5 = 2), A u8, B s8 (bit 10), both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// kind::f16: D f32 (bits 4-5 = 1), A f16 (bits 7-9 = 0), B f16 (bits 10-12 = 0), K-major
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int KIND>  // 0 = i8, 1 = f16
__global__ void rate(long long* out, int N, int nmma, int tmem_cols) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A: 128 rows x 32 B (K-major core matrices) ; B: N x 32 B
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 4096 + 256 * 32; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tb = tmem_base;
    if (tid == 0) {
        const uint32_t id = KIND == 0 ? idesc_i8(128, N) : idesc_f16(128, N);
        // K-major no-swizzle: core matrix = 8 rows x 16 B; LBO = stride between the two
        // K core matrices (K = 32 B), SBO = stride between 8-row groups.
        const uint64_t ad = desc(smem_u32(sm), 128 * 16, 128);
        const uint64_t bd = desc(smem_u32(sm + 4096), N * 16, 128);
        uint32_t phase = 0;
        long long best = 1ll << 60;
        const int ncol = N < 32 ? 32 : N;
        for (int rep = 0; rep < 12; ++rep) {
            long long t0 = clock64();
            for (int k = 0; k < nmma; k += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t d = tb + (uint32_t)(u * ncol);
                    if (KIND == 0)
                        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                     ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(k));
                    else
                        asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                                     ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(k));
                }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
            phase ^= 1;
            long long t = clock64() - t0;
            if (rep > 2 && t < best) best = t;
        }
        out[blockIdx.x] = best;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tb), "r"(tmem_cols));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8 * 148 * 8);
    const int smem = 4096 + 256 * 32 + 1024;
    cudaFuncSetAttribute(rate<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(rate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long h[148 * 8];
    for (int kind : {0, 1})
        for (int N : {16, 32, 64, 128, 256})
            for (int cps : {1, 2, 4}) {
                const int ncol = N < 32 ? 32 : N;
                int cols = 32;
                while (cols < 4 * ncol) cols *= 2;
                if (cols * cps > 512) continue;
                double per[2];
                const int cnt[2] = {16, 256};
                for (int i = 0; i < 2; ++i) {
                    if (kind == 0) rate<0><<<148 * cps, 128, smem>>>(d, N, cnt[i], cols);
                    else rate<1><<<148 * cps, 128, smem>>>(d, N, cnt[i], cols);
                    cudaDeviceSynchronize();
                    cudaMemcpy(h, d, 8 * 148 * cps, cudaMemcpyDeviceToHost);
                    double s = 0;
                    for (int b = 0; b < 148 * cps; ++b) s += (double)h[b];
                    per[i] = s / (148 * cps);
                }
                const double cyc = (per[1] - per[0]) / (cnt[1] - cnt[0]);  // per MMA per CTA
                const int K = kind == 0 ? 32 : 16;
                printf("%s M128 N%3d K%d  ctas/SM %d: %6.1f cycles/MMA/CTA  -> %7.0f MAC/clk/SM  err=%s\n",
                       kind == 0 ? "i8 " : "f16", N, K, cps, cyc, 128.0 * N * K * cps / cyc,
                       cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
