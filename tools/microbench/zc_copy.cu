// Kernel-driven host<->device copies through mapped pinned memory vs cudaMemcpyAsync:
// can a copy kernel (PDL-chainable, no copy-engine dependency gaps) move a step's 1 MiB of
// queries / outputs as fast as the copy engines?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 zc_copy.cu -o zc_copy && ./zc_copy
#include <cuda_runtime.h>

#include <cstdio>

__global__ void copy_f4(const float4* __restrict__ src, float4* __restrict__ dst, size_t n4) {
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main() {
    const size_t bytes = 1 << 20, n4 = bytes / 16;
    float *h, *d;
    cudaHostAlloc(&h, bytes, cudaHostAllocMapped);
    cudaMalloc(&d, bytes);
    float* hd = nullptr;
    cudaHostGetDevicePointer(&hd, h, 0);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto time = [&](auto&& fn, const char* label) {
        for (int i = 0; i < 20; ++i) fn();
        cudaEventRecord(e0, s);
        for (int i = 0; i < 100; ++i) fn();
        cudaEventRecord(e1, s);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("%-44s %7.1f us  %5.1f GB/s\n", label, ms * 10.0f, bytes / (ms * 1e-2) / 1e6);
    };
    time([&] { cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s); }, "H2D cudaMemcpyAsync 1 MiB");
    time([&] { cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s); }, "D2H cudaMemcpyAsync 1 MiB");
    for (int ctas : {148, 296, 592, 1184}) {
        char l1[64], l2[64];
        snprintf(l1, 64, "H2D kernel reads mapped host, %d CTAs", ctas);
        snprintf(l2, 64, "D2H kernel writes mapped host, %d CTAs", ctas);
        time([&] { copy_f4<<<ctas, 256, 0, s>>>((const float4*)hd, (float4*)d, n4); }, l1);
        time([&] { copy_f4<<<ctas, 256, 0, s>>>((const float4*)d, (float4*)hd, n4); }, l2);
    }
    return 0;
}
