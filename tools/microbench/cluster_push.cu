// Minimal repro for the decode kernel's cluster protocol: relaxed arrive at start, push
// via st.shared::cluster, arrive/wait, red.shared::cluster into rank 0, arrive/wait.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
template <int VARIANT>
__global__ void k(int* out) {
    __shared__ float allpart[16 * 24];
    __shared__ uint32_t vsum[512];
    const int rank = (int)cg::this_cluster().block_rank();
    const int S = (int)cg::this_cluster().num_blocks();
    const int lane = threadIdx.x;
    if (VARIANT >= 1) { __syncwarp(); asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory"); }
    if (rank == 0) for (int i = lane; i < 512; i += 32) vsum[i] = 0;
    __syncwarp();
    if (VARIANT >= 1) { __syncwarp(); asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
    else { cg::this_cluster().sync(); }
    if (lane < 24)
        for (int r = 0; r < S; ++r) {
            uint32_t addr;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(allpart + rank * 24 + lane)), "r"(r));
            asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"((float)rank) : "memory");
        }
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    __syncwarp();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    for (int i = lane; i < 512; i += 32) {
        uint32_t addr;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(smem_u32(vsum + i)), "r"(0));
        if (VARIANT == 2) asm volatile("red.relaxed.cluster.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(1u) : "memory");
        else asm volatile("red.shared::cluster.add.u32 [%0], %1;" ::"r"(addr), "r"(1u) : "memory");
    }
    __syncwarp();
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    __syncwarp();
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (rank != 0) return;
    if (lane == 0) { float s = 0; for (int r = 0; r < S; ++r) s += allpart[r * 24]; out[blockIdx.x / S] = (int)vsum[7] * 1000 + (int)s; }
}
int main() {
    int* out; cudaMalloc(&out, 4096 * 4);
    for (int variant = 0; variant < 3; ++variant)
        for (int S : {2, 8, 16}) {
            cudaLaunchConfig_t cfg = {}; cfg.gridDim = dim3(64 * S); cfg.blockDim = dim3(32);
            cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = S; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
            cfg.attrs = at; cfg.numAttrs = 1;
            cudaError_t e;
            if (variant == 0) { cudaFuncSetAttribute(k<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); e = cudaLaunchKernelEx(&cfg, k<0>, out); }
            else if (variant == 1) { cudaFuncSetAttribute(k<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); e = cudaLaunchKernelEx(&cfg, k<1>, out); }
            else { cudaFuncSetAttribute(k<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1); e = cudaLaunchKernelEx(&cfg, k<2>, out); }
            cudaError_t e2 = cudaDeviceSynchronize();
            int h = -1; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost);
            printf("variant %d S=%2d launch=%s sync=%s out=%d (want %d)\n", variant, S, cudaGetErrorString(e), cudaGetErrorString(e2), h, S * 1000 + S * (S - 1) / 2);
            fflush(stdout);
        }
    return 0;
}
