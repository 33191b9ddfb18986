// k3_append.cu — K3: HybridKVCache::append (kvcache.hpp:99-109). One fp32 K row and one
// V row per (request, KV head) go to tail slot tail_len[request]; the packed segment is
// never touched and tokens are never re-quantized. tail_len lives on the
// device so append + decode can be captured in one CUDA graph and replayed per step.
#include "kvq_internal.cuh"

namespace kvqb {

namespace {

// One CTA per request: all of its KV heads, then a single increment of its length. A full
// tail (tail_len == tail_cap: e.g. a captured decode + append graph replayed past the rows
// reserve_tail made room for) is never written past: the append is dropped and `overflow`
// set, which the host reports as a domain_error at its next synchronization
// (kvq_cache_sync_tail) instead of corrupting the neighbouring unit's rows.
__global__ void append_kernel(const float* __restrict__ k_new, const float* __restrict__ v_new,
                              size_t kv_heads, size_t dim, size_t tail_cap,
                              float* __restrict__ k_tail, float* __restrict__ v_tail,
                              int* __restrict__ tail_len, int* __restrict__ overflow) {
    const size_t b = blockIdx.x;
    const size_t n = kv_heads * dim;
    const bool vec = (dim % 4) == 0;
    if (vec && n <= 4 * 4 * blockDim.x) {
        // Launched right behind the decode (programmatic dependent launch): the new rows
        // are read while the decode finishes; the tail is written once it has retired.
        float4 kr[4], vr[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const size_t i = threadIdx.x + (size_t)r * blockDim.x;
            if (4 * i < n) {
                kr[r] = *reinterpret_cast<const float4*>(k_new + b * n + 4 * i);
                vr[r] = *reinterpret_cast<const float4*>(v_new + b * n + 4 * i);
            }
        }
        asm volatile("griddepcontrol.wait;" ::: "memory");
        // The next decode (programmatic stream serialization) may start its prologue now; it
        // reads the tail only after its own griddepcontrol.wait (= this grid done). Released
        // only here - once the preceding decode has drained - so the decode's CTAs are placed
        // evenly over free SMs rather than stacked on the first SMs to finish.
        asm volatile("griddepcontrol.launch_dependents;");
        const size_t slot = (size_t)tail_len[b];
        if (slot >= tail_cap) {
            if (threadIdx.x == 0) atomicOr(overflow, 1);
            return;
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            const size_t i = threadIdx.x + (size_t)r * blockDim.x;
            if (4 * i < n) {
                const size_t h = (4 * i) / dim, c = (4 * i) % dim;
                const size_t dst = ((b * kv_heads + h) * tail_cap + slot) * dim + c;
                *reinterpret_cast<float4*>(k_tail + dst) = kr[r];
                *reinterpret_cast<float4*>(v_tail + dst) = vr[r];
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) tail_len[b] = (int)(slot + 1);
        return;
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const size_t slot = (size_t)tail_len[b];
    if (slot >= tail_cap) {
        if (threadIdx.x == 0) atomicOr(overflow, 1);
        return;
    }
    for (size_t i = threadIdx.x; i < (vec ? n / 4 : n); i += blockDim.x) {
        if (vec) {
            size_t h = (i * 4) / dim, c = (i * 4) % dim;
            size_t dst = ((b * kv_heads + h) * tail_cap + slot) * dim + c;
            size_t src = (b * kv_heads + h) * dim + c;
            *reinterpret_cast<float4*>(k_tail + dst) = *reinterpret_cast<const float4*>(k_new + src);
            *reinterpret_cast<float4*>(v_tail + dst) = *reinterpret_cast<const float4*>(v_new + src);
        } else {
            size_t h = i / dim, c = i % dim;
            size_t dst = ((b * kv_heads + h) * tail_cap + slot) * dim + c;
            k_tail[dst] = k_new[(b * kv_heads + h) * dim + c];
            v_tail[dst] = v_new[(b * kv_heads + h) * dim + c];
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) tail_len[b] = (int)(slot + 1);
}

}  // namespace

cudaError_t launch_append(const float* k_new, const float* v_new, size_t batch, size_t kv_heads,
                          size_t dim, size_t tail_cap, float* k_tail, float* v_tail,
                          int* tail_len, int* overflow, cudaStream_t s) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)batch);
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    note_launch();
    return cudaLaunchKernelEx(&cfg, append_kernel, k_new, v_new, kv_heads, dim, tail_cap, k_tail, v_tail, tail_len,
                              overflow);
}

}  // namespace kvqb
