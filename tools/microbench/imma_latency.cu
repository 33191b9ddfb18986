// Microbenchmark: dependent-chain latency of mma.sync m16n8k32 IMMA (u8.s8) and of
// LDS -> LOP3 -> IMMA operand chains on sm_100a; one warp, clock64.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain(long long* out, int iters) {
    int c[4] = {0, 0, 0, 0};
    uint32_t a0 = threadIdx.x * 0x01010101u, a1 = a0 ^ 0x5a5a5a5a, a2 = a0 + 3, a3 = a0 * 7, b0 = 0x01020304, b1 = 0x7f000001;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t1 = clock64();
    // independent: 4 chains interleaved
    int d[4][4] = {};
    long long t2 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 4; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(d[j][0]), "+r"(d[j][1]), "+r"(d[j][2]), "+r"(d[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t3 = clock64();
    // 16 independent chains
    int e[16][4] = {};
    long long t4 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                         : "+r"(e[j][0]), "+r"(e[j][1]), "+r"(e[j][2]), "+r"(e[j][3])
                         : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
    long long t5 = clock64();
    int s = c[0] + c[3];
    for (int j = 0; j < 4; ++j) s += d[j][0] + d[j][3];
    for (int j = 0; j < 16; ++j) s += e[j][1];
    if (threadIdx.x == 0) {
        out[0] = t1 - t0;
        out[1] = t3 - t2;
        out[2] = t5 - t4;
        out[3] = s;
    }
}

int main() {
    long long* d;
    cudaMalloc(&d, 64);
    const int iters = 1000;
    chain<<<1, 32>>>(d, iters);
    cudaDeviceSynchronize();
    chain<<<1, 32>>>(d, iters);
    cudaDeviceSynchronize();
    long long h[4];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("IMMA m16n8k32 u8.s8, one warp: dependent chain %.1f cycles/IMMA; 4 independent chains %.1f cycles/IMMA; "
           "16 chains %.1f cycles/IMMA  (%s)\n",
           (double)h[0] / iters, (double)h[1] / (4.0 * iters), (double)h[2] / (16.0 * iters),
           cudaGetErrorString(cudaGetLastError()));
    return 0;
}
