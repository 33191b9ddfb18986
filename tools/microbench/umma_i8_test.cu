// Probe: tcgen05.mma kind::i8 with A from TMEM (written by tcgen05.st) and B from shared
// memory, s32 accumulators in TMEM read back with tcgen05.ld. Pins down the operand
// layouts the K2 UMMA decode kernel relies on:
//   A (TMEM): lane m = row m, column j holds K elements 4j..4j+3 (byte i = element 4j+i)
//   B (SMEM): no-swizzle canonical layouts, K-major and MN-major, LBO/SBO as below
//   D (TMEM): lane m = row m, column n = D[m][n]
// Prints PASS/FAIL per variant.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

// kind::i8 instruction descriptor: D s32, A u8, B s8|u8, A K-major, B major, M, N.
__host__ __device__ constexpr uint32_t idesc_i8(int M, int N, bool b_signed, bool b_mn_major) {
    return (2u << 4) | (0u << 7) | ((b_signed ? 1u : 0u) << 10) | (0u << 15) | ((b_mn_major ? 1u : 0u) << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int NCOL>
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[NCOL]);

template <>
__device__ __forceinline__ void tmem_st32<8>(uint32_t taddr, const uint32_t (&r)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
                 "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

__global__ void probe(const uint8_t* A, const int8_t* B, int32_t* D, int mode, int M, int N) {
    // mode 0: B K-major; mode 1: B MN-major. Two MMAs (K = 64 total) accumulate.
    __shared__ __align__(1024) int8_t sB[2][32 * 32];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    // B tile for MMA kk: K rows 32kk..32kk+31, N columns
    for (int e = tid; e < 2 * 32 * N; e += blockDim.x) {
        const int kk = e / (32 * N), rem = e % (32 * N);
        const int k = rem / N, n = rem % N;
        const int8_t v = B[(32 * kk + k) * N + n];
        int off;
        if (mode == 0) {  // K-major: (n%8)*16 + (n/8)*SBO + (k/16)*LBO + k%16, SBO=128, LBO=N*16
            off = (n % 8) * 16 + (n / 8) * 128 + (k / 16) * (N * 16) + (k % 16);
        } else {  // MN-major: (k%8)*16 + (k/8)*LBO + (n/16)*SBO + n%16, LBO=128, SBO=512
            off = (k % 8) * 16 + (k / 8) * 128 + (n / 16) * 512 + (n % 16);
        }
        sB[kk][off] = v;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(smem_u32(&tmem_base)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tbase = tmem_base;
    // A rows: thread m (< M) writes row m, K = 64 -> 16 columns (two groups of 8)
    if (tid < 128) {
        const int m = tid;
        for (int kk = 0; kk < 2; ++kk) {
            uint32_t r[8];
            for (int j = 0; j < 8; ++j) {
                uint32_t w = 0;
                for (int i = 0; i < 4; ++i) w |= (uint32_t)(m < M ? A[m * 64 + 32 * kk + 4 * j + i] : 0) << (8 * i);
                r[j] = w;
            }
            const uint32_t taddr = tbase + ((uint32_t)(32 * warp) << 16) + 8 * kk;
            tmem_st32<8>(taddr, r);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t dcol = tbase + 32;
    if (tid == 0) {
        const uint32_t idesc = idesc_i8(M, N, true, mode == 1);
        for (int kk = 0; kk < 2; ++kk) {
            uint64_t bd = mode == 0 ? smem_desc(smem_u32(sB[kk]), N * 16, 128) : smem_desc(smem_u32(sB[kk]), 128, 512);
            const uint32_t acc = kk > 0;
            asm volatile(
                "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(dcol),
                "r"(tbase + 8 * kk), "l"(bd), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar))
                     : "memory");
    }
    // wait for the MMA
    {
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(done)
                : "r"(smem_u32(&bar))
                : "memory");
        }
    }
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid < 128) {
        uint32_t r[16];
        const uint32_t taddr = dcol + ((uint32_t)(32 * warp) << 16);
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
              "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (tid < M)
            for (int n = 0; n < N && n < 16; ++n) D[tid * N + n] = (int32_t)r[n];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tbase));
}

// Latency probe: cycles for (a) STTM.x32 + wait::st, (b) 4 x UTCIMMA M128 N16 K32 issue ->
// commit -> mbarrier completion, (c) LDTM.x16 + wait::ld. One CTA, 128 threads.
__global__ void latency(long long* out, int iters, int nmma, int indep) {
    __shared__ __align__(1024) int8_t sB[32 * 16 * 4];
    __shared__ uint32_t tmem_base;
    __shared__ __align__(8) uint64_t bar;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (int)sizeof(sB); i += blockDim.x) sB[i] = (int8_t)i;
    if (warp == 0) {
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
    const uint32_t tbase = tmem_base;
    const uint32_t tl = tbase + ((uint32_t)(32 * warp) << 16);
    long long t_st = 0, t_mma = 0, t_ld = 0, t_bar = 0;
    uint32_t r[32];
    for (int j = 0; j < 32; ++j) r[j] = tid * 0x01010101u + j;
    uint32_t phase = 0;
    for (int it = 0; it < iters; ++it) {
        long long t0 = clock64();
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tl),
            "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
            "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
            "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
            "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]) : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        long long t1 = clock64();
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
        long long t2 = clock64();
        if (tid == 0) {
            const uint32_t idesc = idesc_i8(128, 16, true, true);
            for (int kk = 0; kk < nmma; ++kk) {
                uint64_t bd = smem_desc(smem_u32(sB + (kk & 3) * 512), 128, 2048);
                const uint32_t dcol = indep ? 64 + 16 * (kk & 3) : 64;
                asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
                             " tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tbase + dcol),
                             "r"(tbase + 8 * (kk & 3)), "l"(bd), "r"(idesc), "r"(indep ? 0 : kk));
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        }
        uint32_t done = 0;
        while (!done) {
            asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(done) : "r"(smem_u32(&bar)), "r"(phase) : "memory");
        }
        phase ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;");
        long long t3 = clock64();
        uint32_t d[16];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
            : "r"(tl + 64));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        long long t4 = clock64();
        for (int j = 0; j < 16; ++j) r[j] += d[j];
        if (it > 0) { t_st += t1 - t0; t_bar += t2 - t1; t_mma += t3 - t2; t_ld += t4 - t3; }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncthreads();
        asm volatile("tcgen05.fence::after_thread_sync;");
    }
    if (tid == 0 && blockIdx.x == 0) { out[0] = t_st; out[1] = t_bar; out[2] = t_mma; out[3] = t_ld; out[4] = r[3]; }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tbase));
}

int main() {
    const int M = 128;
    int fails = 0;
    for (int N : {16, 8}) {
        for (int mode = 0; mode < 2; ++mode) {
            if (N == 8 && mode == 1) continue;  // MN-major needs N >= 16 chunks
            uint8_t hA[128 * 64];
            int8_t hB[64 * 16];
            srand(1234 + mode + N);
            for (auto& x : hA) x = (uint8_t)(rand() & 0xFF);
            for (int i = 0; i < 64 * N; ++i) hB[i] = (int8_t)(rand() & 0xFF);
            uint8_t* dA;
            int8_t* dB;
            int32_t* dD;
            cudaMalloc(&dA, sizeof hA);
            cudaMalloc(&dB, sizeof hB);
            cudaMalloc(&dD, 128 * 16 * 4);
            cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
            cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
            cudaMemset(dD, 0, 128 * 16 * 4);
            probe<<<1, 128>>>(dA, dB, dD, mode, M, N);
            cudaError_t e = cudaDeviceSynchronize();
            int32_t hD[128 * 16];
            cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int m = 0; m < M; ++m)
                for (int n = 0; n < N; ++n) {
                    int32_t want = 0;
                    for (int k = 0; k < 64; ++k) want += (int32_t)hA[m * 64 + k] * (int32_t)hB[k * N + n];
                    if (want != hD[m * N + n]) {
                        if (bad < 4) printf("  m=%d n=%d got %d want %d\n", m, n, hD[m * N + n], want);
                        ++bad;
                    }
                }
            printf("N=%d B %s-major: %s (%d mismatches) err=%s\n", N, mode ? "MN" : "K", bad ? "FAIL" : "PASS", bad,
                   cudaGetErrorString(e));
            fails += bad != 0;
            cudaFree(dA);
            cudaFree(dB);
            cudaFree(dD);
            if (e != cudaSuccess) return 2;
        }
    }
    {
        long long* d;
        cudaMalloc(&d, 64);
        cudaFuncSetAttribute(latency, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        const int iters = 200;
        for (int ctas : {1, 296})
            for (int nmma : {0, 1, 2, 4, 8})
                for (int indep : {0, 1}) {
                    if (nmma == 0 && indep) continue;
                    latency<<<ctas, 128, 100 * 1024>>>(d, iters, nmma, indep);
                    cudaError_t e = cudaDeviceSynchronize();
                    long long h[5];
                    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                    printf("ctas %3d: %d x UTCIMMA M128N16K32 (%s): issue->commit->mbarrier %.0f cycles | STTM.x32+wait "
                           "%.0f | fence+bar %.0f | LDTM.x16+wait %.0f  err=%s\n", ctas, nmma,
                           indep ? "independent D" : "chained D", h[2] / (double)(iters - 1), h[0] / (double)(iters - 1),
                           h[1] / (double)(iters - 1), h[3] / (double)(iters - 1), cudaGetErrorString(e));
                }
    }
    return fails ? 1 : 0;
}
