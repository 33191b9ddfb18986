// Microbenchmark: do legacy mma.sync IMMA (m16n8k32 u8.s8) and tcgen05.mma kind::i8 (M128
// N16 K32) share tensor-core throughput on one SM? Per CTA: `iw` warps run IMMA chains,
// one extra warp issues tcgen05 MMAs; modes 1 = IMMA only, 2 = tcgen05 only, 3 = both.
// Reports the kernel time per mode (one CTA per SM, or two).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N) {
    return (2u << 4) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void imma(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t b0,
                                     uint32_t b1) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                 : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__global__ void mix(int* out, int mode, int iw, int n_imma, int n_umma, int N) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 4096 + 256 * 32; i += blockDim.x) sm[i] = (uint8_t)(i * 7);
    if (warp == iw) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tmem_base)));
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
    if (warp < iw) {
        if (mode & 1) {
            int c[8][4] = {};
            uint32_t a = tid * 0x01010101u, b = tid * 3u;
            for (int i = 0; i < n_imma; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) imma(c[j], a, a + j, a ^ j, a, b, b + j);
            }
            int s = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
            out[blockIdx.x * blockDim.x + tid] = s;
        }
    } else if (warp == iw && (mode & 2)) {
        if ((tid & 31) == 0) {
            const uint32_t id = idesc_i8(128, N);
            const uint64_t ad = desc(smem_u32(sm), 128 * 16, 128);
            const uint64_t bd = desc(smem_u32(sm + 4096), N * 16, 128);
            for (int k = 0; k < n_umma; k += 4) {
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
                                 ::"r"(tb + (uint32_t)(u * 32)), "l"(ad), "l"(bd), "r"(id), "r"(k));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
            uint32_t done = 0;
            while (!done)
                asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                             : "=r"(done) : "r"(smem_u32(&bar)) : "memory");
        }
        __syncwarp();
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == iw) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tb));
}

int main() {
    int* d;
    cudaMalloc(&d, 148 * 4 * 1024 * 4);
    const int smem = 4096 + 256 * 32 + 1024;
    cudaFuncSetAttribute(mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int cps : {1, 2})
        for (int iw : {4, 8})
            for (int N : {16, 64}) {
                const int n_imma = 1 << 14;                    // per IMMA warp
                const int n_umma = N == 16 ? 1 << 12 : 1 << 11;  // per CTA
                float t[4] = {};
                for (int mode = 1; mode <= 3; ++mode) {
                    for (int rep = 0; rep < 3; ++rep) {
                        cudaEventRecord(e0);
                        mix<<<148 * cps, 32 * (iw + 1), smem>>>(d, mode, iw, n_imma, n_umma, N);
                        cudaEventRecord(e1);
                        cudaEventSynchronize(e1);
                        cudaEventElapsedTime(&t[mode], e0, e1);
                    }
                }
                const double clk = 1.965e6;  // kHz * ms -> cycles
                const double imma_rate = (double)n_imma * iw * cps / (t[1] * clk);
                const double umma_cyc = t[2] * clk / ((double)n_umma * cps);
                printf("ctas/SM %d imma warps %d N %3d: IMMA only %.3f ms (%.3f IMMA/clk/SM) | tcgen05 only %.3f ms (%.1f cyc/MMA/SM) | both %.3f ms  err=%s\n",
                       cps, iw, N, t[1], imma_rate, t[2], umma_cyc, t[3], cudaGetErrorString(cudaGetLastError()));
            }
    return 0;
}
