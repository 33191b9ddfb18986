// Probe: numerics of mma.sync m16n8k32 e4m3 x e4m3 -> f32 on sm_100a.
//  (1) subnormal operands (e4m3 0x01 = 2^-9) survive: D = 2^-9 * 2^-9 * count?
//  (2) accumulation precision: C large, products small -> is every product added?
//  (3) 128-MMA chains of random e4m3 data vs an fp64 reference and vs sequential fp32.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_fp8.h>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_fp8(float (&c)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
    asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
                 : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

// A: [nmma][16][32] e4m3 bytes (row-major), B: [nmma][8][32] (col-major = n-major rows of k),
// C init per element, D out [16][8].
__global__ void run(const uint8_t* A, const uint8_t* B, const float* C0, float* D, int nmma) {
    const int lane = threadIdx.x, g = lane >> 2, t = lane & 3;
    float c[4] = {C0[g * 8 + 2 * t], C0[g * 8 + 2 * t + 1], C0[(g + 8) * 8 + 2 * t], C0[(g + 8) * 8 + 2 * t + 1]};
    for (int m = 0; m < nmma; ++m) {
        const uint8_t* a = A + m * 512;
        const uint8_t* b = B + m * 256;
        uint32_t ar[4], br[2];
        ar[0] = *(const uint32_t*)(a + g * 32 + 4 * t);
        ar[1] = *(const uint32_t*)(a + (g + 8) * 32 + 4 * t);
        ar[2] = *(const uint32_t*)(a + g * 32 + 16 + 4 * t);
        ar[3] = *(const uint32_t*)(a + (g + 8) * 32 + 16 + 4 * t);
        br[0] = *(const uint32_t*)(b + g * 32 + 4 * t);
        br[1] = *(const uint32_t*)(b + g * 32 + 16 + 4 * t);
        mma_fp8(c, ar, br);
    }
    D[g * 8 + 2 * t] = c[0];
    D[g * 8 + 2 * t + 1] = c[1];
    D[(g + 8) * 8 + 2 * t] = c[2];
    D[(g + 8) * 8 + 2 * t + 1] = c[3];
}

static float e4m3_val(uint8_t x) {
    __nv_fp8_e4m3 v;
    v.__x = x;
    return (float)v;
}

int main() {
    const int maxm = 128;
    uint8_t *hA = (uint8_t*)malloc(maxm * 512), *hB = (uint8_t*)malloc(maxm * 256);
    float hC[128], hD[128];
    uint8_t *dA, *dB;
    float *dC, *dD;
    cudaMalloc(&dA, maxm * 512);
    cudaMalloc(&dB, maxm * 256);
    cudaMalloc(&dC, 512);
    cudaMalloc(&dD, 512);
    auto go = [&](int nmma) {
        cudaMemcpy(dA, hA, nmma * 512, cudaMemcpyHostToDevice);
        cudaMemcpy(dB, hB, nmma * 256, cudaMemcpyHostToDevice);
        cudaMemcpy(dC, hC, 512, cudaMemcpyHostToDevice);
        run<<<1, 32>>>(dA, dB, dC, dD, nmma);
        cudaMemcpy(hD, dD, 512, cudaMemcpyDeviceToHost);
    };
    // (1) subnormals: A = 0x01 (2^-9), B = 0x01 -> each product 2^-18, 32 per element
    for (int i = 0; i < 512; ++i) hA[i] = 0x01;
    for (int i = 0; i < 256; ++i) hB[i] = 0x01;
    for (int i = 0; i < 128; ++i) hC[i] = 0.f;
    go(1);
    printf("(1) subnormal x subnormal: D = %.9g (exact %.9g)\n", hD[0], 32.0 * std::ldexp(1.0, -18));
    for (int i = 0; i < 256; ++i) hB[i] = 0x38;  // 1.0
    go(1);
    printf("(1b) subnormal x 1.0: D = %.9g (exact %.9g)\n", hD[0], 32.0 * std::ldexp(1.0, -9));
    // (2) C = 2^12, one product = 2^-9 * 1.0 per k: sum 32 * 2^-9 = 2^-4 -> exact fp32 result 4096.0625
    for (int i = 0; i < 128; ++i) hC[i] = 4096.0f;
    go(1);
    printf("(2) C=4096 + 32 x 2^-9: D = %.9g (exact fp32 %.9g)\n", hD[0], 4096.0 + 0.0625);
    // one product only (k = 0), the others zero: 4096 + 2^-9 -> fp32 ulp(4096) = 2^-11
    for (int i = 0; i < 512; ++i) hA[i] = (i % 32 == 0) ? 0x01 : 0x00;
    go(1);
    printf("(2b) C=4096 + 2^-9: D - C = %.9g (exact %.9g)\n", hD[0] - 4096.0, std::ldexp(1.0, -9));
    for (int i = 0; i < 128; ++i) hC[i] = 1.0f;
    for (int i = 0; i < 512; ++i) hA[i] = (i % 32 == 0) ? 0x38 : ((i % 32 == 1) ? 0x01 : 0x00);  // 1.0, 2^-9
    for (int i = 0; i < 256; ++i) hB[i] = (i % 32 == 1) ? 0x01 : 0x38;
    go(1);
    printf("(2c) C=1 + 1*1 + 2^-9*2^-9: D - 2 = %.9g (exact %.9g)\n", hD[0] - 2.0, std::ldexp(1.0, -18));
    // (3) chains of random data
    srand(7);
    for (int nm : {1, 8, 128}) {
        double worst_ref = 0, worst_seq = 0;
        for (int trial = 0; trial < 20; ++trial) {
            for (int i = 0; i < nm * 512; ++i) {
                uint8_t x = (uint8_t)(rand() & 0x7F);  // positive e4m3, avoid NaN 0x7F
                if (x == 0x7F) x = 0x7E;
                hA[i] = x;
            }
            for (int i = 0; i < nm * 256; ++i) {
                uint8_t x = (uint8_t)(rand() & 0x7F);
                if (x == 0x7F) x = 0x7E;
                hB[i] = (rand() & 1) ? (x | 0x80) : x;
            }
            for (int i = 0; i < 128; ++i) hC[i] = 0.f;
            go(nm);
            for (int r = 0; r < 16; ++r)
                for (int cn = 0; cn < 8; ++cn) {
                    double ref = 0, mag = 0;
                    float seq = 0.f;
                    for (int m = 0; m < nm; ++m)
                        for (int k = 0; k < 32; ++k) {
                            double p = (double)e4m3_val(hA[m * 512 + r * 32 + k]) * e4m3_val(hB[m * 256 + cn * 32 + k]);
                            ref += p;
                            mag += std::fabs(p);
                            seq += (float)p;
                        }
                    const double got = hD[r * 8 + cn];
                    worst_ref = std::fmax(worst_ref, std::fabs(got - ref) / mag);
                    worst_seq = std::fmax(worst_seq, std::fabs((double)seq - ref) / mag);
                }
        }
        printf("(3) %3d MMAs: max |D - exact| / sum|p| = %.3g  (sequential fp32: %.3g)  err=%s\n", nm, worst_ref,
               worst_seq, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
