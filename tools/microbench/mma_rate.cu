// Microbenchmark: legacy mma.sync tensor-core throughput on sm_100a.
// Decides the K2 (decode) inner-loop formulation: HMMA f16 vs IMMA s8/u8 vs FP8.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CHAINS 8
template <int KIND>
__global__ void mma_loop(int iters, float* sink) {
  uint32_t a[4], b[2];
  for (int i = 0; i < 4; ++i) a[i] = 0x3c003c00u ^ (threadIdx.x * 7 + i);
  for (int i = 0; i < 2; ++i) b[i] = 0x3c003c00u ^ (threadIdx.x * 3 + i);
  float c[CHAINS][4];
  int ci[CHAINS][4];
  for (int j = 0; j < CHAINS; ++j) for (int i = 0; i < 4; ++i) { c[j][i] = 0.f; ci[j][i] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CHAINS; ++j) {
      if (KIND == 0) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 1) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(ci[j][0]), "+r"(ci[j][1]), "+r"(ci[j][2]), "+r"(ci[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 2) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.u8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(ci[j][0]), "+r"(ci[j][1]), "+r"(ci[j][2]), "+r"(ci[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 3) {
        asm volatile("mma.sync.aligned.m16n8k32.row.col.f32.e4m3.e4m3.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 4) {
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 5) {
        // f16 accumulate
        uint32_t* cc = reinterpret_cast<uint32_t*>(&c[j][0]);
        asm volatile("mma.sync.aligned.m16n8k16.row.col.f16.f16.f16.f16 {%0,%1}, {%2,%3,%4,%5}, {%6,%7}, {%0,%1};"
                     : "+r"(cc[0]), "+r"(cc[1])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 7) {
        asm volatile("mma.sync.aligned.m16n8k64.row.col.s32.u4.s4.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(ci[j][0]), "+r"(ci[j][1]), "+r"(ci[j][2]), "+r"(ci[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      } else if (KIND == 6) {
        // 1-bit and.popc (emulated?)
        asm volatile("mma.sync.aligned.m16n8k256.row.col.s32.b1.b1.s32.and.popc {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                     : "+r"(ci[j][0]), "+r"(ci[j][1]), "+r"(ci[j][2]), "+r"(ci[j][3])
                     : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
      }
    }
  }
  float s = 0.f;
  for (int j = 0; j < CHAINS; ++j) for (int i = 0; i < 4; ++i) s += c[j][i] + (float)ci[j][i];
  if (s == 1234.5f) sink[threadIdx.x] = s;
}

// ALU throughput probe: LOP3 chains (bit->operand expansion cost model)
__global__ void lop_loop(int iters, uint32_t* sink) {
  uint32_t x[8];
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 0x9e3779b9u + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      asm volatile("lop3.b32 %0, %0, 0x01010101, 0x38383838, 0xea;" : "+r"(x[j]));
    }
  }
  uint32_t s = 0;
  for (int i = 0; i < 8; ++i) s ^= x[i];
  if (s == 12345u) sink[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, clk);
  float* sink; cudaMalloc(&sink, 4096);
  const char* names[] = {"HMMA m16n8k16 f16->f32", "IMMA m16n8k32 s8", "IMMA m16n8k32 u8.s8",
                         "FP8 m16n8k32 e4m3->f32", "HMMA m16n8k16 bf16->f32", "HMMA m16n8k16 f16->f16",
                         "BMMA m16n8k256 and.popc", "IMMA m16n8k64 u4.s4"};
  const double macs[] = {16*8*16, 16*8*32, 16*8*32, 16*8*32, 16*8*16, 16*8*16, 16*8*256, 16*8*64};
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int k = 0; k < 8; ++k) {
      int iters = 2000;
      int blocks = p.multiProcessorCount * 2;
      auto launch = [&]() {
        switch (k) {
          case 0: mma_loop<0><<<blocks, warps * 32>>>(iters, sink); break;
          case 1: mma_loop<1><<<blocks, warps * 32>>>(iters, sink); break;
          case 2: mma_loop<2><<<blocks, warps * 32>>>(iters, sink); break;
          case 3: mma_loop<3><<<blocks, warps * 32>>>(iters, sink); break;
          case 4: mma_loop<4><<<blocks, warps * 32>>>(iters, sink); break;
          case 5: mma_loop<5><<<blocks, warps * 32>>>(iters, sink); break;
          case 6: mma_loop<6><<<blocks, warps * 32>>>(iters, sink); break;
          case 7: mma_loop<7><<<blocks, warps * 32>>>(iters, sink); break;
        }
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double n_mma = (double)blocks * warps * iters * CHAINS;
      double tmacs = n_mma * macs[k] / (ms * 1e-3) / 1e12;
      printf("warps/CTA %2d  %-26s  %.3f ms  %8.1f T-MAC/s  (%.1f TFLOP/s)  %.2f mma/clk/SM@%.0fMHz  err=%s\n", warps, names[k], ms, tmacs, 2*tmacs,
             n_mma / (ms*1e-3) / p.multiProcessorCount / (clk*1e3), clk/1e3, cudaGetErrorString(cudaGetLastError()));
    }
    {
      int iters = 20000, blocks = p.multiProcessorCount * 2;
      lop_loop<<<blocks, warps * 32>>>(iters, (uint32_t*)sink); cudaDeviceSynchronize();
      cudaEventRecord(e0); lop_loop<<<blocks, warps * 32>>>(iters, (uint32_t*)sink); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double n = (double)blocks * warps * iters * 8;
      printf("warps/CTA %2d  LOP3 warp-instr/clk/SM = %.2f\n", warps, n / (ms*1e-3) / p.multiProcessorCount / (clk*1e3));
    }
  }
  return 0;
}
