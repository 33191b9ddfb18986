// Microbenchmark: HBM streaming throughput of cp.async.bulk (TMA, 1-D bulk copies into
// a shared-memory ring, mbarrier completion) as a function of stage size, ring depth
// and CTAs per SM -- the producer pattern of the K2 decode kernels. No compute: each
// CTA consumes a stage by touching one word and re-arms it.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void stream_kernel(const uint8_t* __restrict__ src, size_t bytes_per_cta, int stage_bytes, int stages,
                              unsigned long long* sink, size_t cta_stride = 0) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * stage_bytes);
    const uint8_t* base = src + (size_t)blockIdx.x * (cta_stride ? cta_stride : bytes_per_cta);
    const int nst = (int)(bytes_per_cta / stage_bytes);
    if (threadIdx.x == 0) {
        for (int i = 0; i < stages; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int i = 0; i < stages && i < nst; ++i) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[i])),
                         "r"(stage_bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(smem + (size_t)i * stage_bytes)),
                         "l"(base + (size_t)i * stage_bytes), "r"(stage_bytes), "r"(smem_u32(&full[i])) : "memory");
        }
    }
    __syncthreads();
    unsigned long long acc = 0;
    for (int i = 0; i < nst; ++i) {
        const int slot = i % stages;
        uint32_t done = 0;
        while (!done)
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&full[slot])), "r"((uint32_t)((i / stages) & 1)) : "memory");
        acc += reinterpret_cast<const uint32_t*>(smem + (size_t)slot * stage_bytes)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && i + stages < nst) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[slot])),
                         "r"(stage_bytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                             smem_u32(smem + (size_t)slot * stage_bytes)),
                         "l"(base + (size_t)(i + stages) * stage_bytes), "r"(stage_bytes), "r"(smem_u32(&full[slot]))
                         : "memory");
        }
    }
    if (acc == 0x123456789ull) sink[0] = acc;
}

int main() {
    const size_t total = (size_t)2 << 30;  // 2 GiB (>> L2)
    uint8_t* buf;
    cudaMalloc(&buf, total);
    cudaMemset(buf, 1, total);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    // Partition-camping probe: 1024 CTAs x 32 KB regions (the c2 decode's K streams) with
    // a power-of-two region stride vs a padded stride.
    for (size_t stride : {(size_t)32768, (size_t)32768 + 256, (size_t)32768 + 2048, (size_t)65536, (size_t)65536 + 256}) {
        const int ctas = 1024;
        stream_kernel<<<ctas, 128, 56 * 1024>>>(buf, 32768, 2048, 5, sink, stride);
        cudaEventRecord(e0);
        stream_kernel<<<ctas, 128, 56 * 1024>>>(buf, 32768, 2048, 5, sink, stride);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("camping: 1024 CTAs x 32 KB, stride %zu: %.1f GB/s (%.1f us)\n", stride, 32768.0 * ctas / (ms * 1e-3) / 1e9, ms * 1e3);
    }
    printf("stage_bytes stages ctas/SM(target) GB/s\n");
    for (int sb : {2048, 4096, 8192, 16384}) {
        for (int st : {2, 4, 6, 8, 12}) {
            for (int per_sm : {1, 2, 4, 8}) {
                const size_t smem = (size_t)sb * st + 16 * 8;
                if (smem * per_sm > 220 * 1024) continue;
                // pad shared memory so that exactly per_sm CTAs fit
                size_t want = 228 * 1024 / per_sm - 1024;
                size_t dyn = smem > want ? smem : want;
                if (dyn > 200 * 1024) dyn = smem;
                const int ctas = 148 * per_sm * 4;
                const size_t per_cta = total / ctas / sb * sb;
                stream_kernel<<<ctas, 128, dyn>>>(buf, per_cta, sb, st, sink);
                cudaEventRecord(e0);
                stream_kernel<<<ctas, 128, dyn>>>(buf, per_cta, sb, st, sink);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("%6d %3d %2d %8.1f  %s\n", sb, st, per_sm, per_cta * ctas / (ms * 1e-3) / 1e9,
                       cudaGetErrorString(cudaGetLastError()));
            }
        }
    }
    return 0;
}
