// Microbenchmark: tcgen05.mma kind::i8 M128 cost per instruction vs N and A source
// (TMEM vs shared memory), one CTA per SM issuing back-to-back MMAs (independent and
// chained accumulators); reports cycles per MMA at steady state.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool a_mn) {
    return (2u << 4) | (1u << 10) | ((a_mn ? 1u : 0u) << 15) | (1u << 16) | ((uint32_t)(N >> 3) << 17) |
           ((uint32_t)(M >> 4) << 24);
}

__global__ void rate(long long* out, int N, int a_smem, int nmma) {
    extern __shared__ __align__(1024) uint8_t sm[];  // A: 128 x 32 (K-major interleaved) 4 KB; B: 32 x N MN-major
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 4096 + 32 * 256; i += blockDim.x) sm[i] = (uint8_t)i;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tmem_base)));
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
        const uint32_t id = idesc_i8(128, N, false);
        const uint64_t bd = desc(smem_u32(sm + 4096), 128, 32 * 16);
        const uint64_t ad = desc(smem_u32(sm), 128 * 2 /*LBO: K chunk stride*/, 128 /*SBO: 8-row group*/);
        uint32_t phase = 0;
        long long best = 1ll << 60;
        for (int rep = 0; rep < 20; ++rep) {
            long long t0 = clock64();
            for (int k = 0; k < nmma; ++k) {
                const uint32_t d = tb + 256;  // chained accumulator
                if (a_smem)
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(d), "l"(ad), "l"(bd), "r"(id), "r"(k));
                else
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n"
                                 ::"r"(d), "r"(tb), "l"(bd), "r"(id), "r"(k));
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
        if (blockIdx.x == 0) out[0] = best;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tb));
}

int main() {
    long long* d;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(rate, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int a_smem : {0, 1})
        for (int N : {16, 32, 64, 128, 256}) {
            long long t[2];
            int cnt[2] = {8, 64};
            for (int i = 0; i < 2; ++i) {
                rate<<<148, 128, 64 * 1024>>>(d, N, a_smem, cnt[i]);
                cudaDeviceSynchronize();
                cudaMemcpy(&t[i], d, 8, cudaMemcpyDeviceToHost);
            }
            const double per = (double)(t[1] - t[0]) / (cnt[1] - cnt[0]);
            printf("A %s  M128 N%3d K32 i8: %.1f cycles/MMA (%.0f MAC/clk/SM), 8-MMA latency %lld  err=%s\n",
                   a_smem ? "smem" : "tmem", N, per, 128.0 * N * 32 / per, t[0], cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
