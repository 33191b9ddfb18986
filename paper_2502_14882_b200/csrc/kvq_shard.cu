// kvq_shard.cu — the native host side of the multi-GPU split (shard.py is the
// Python mirror that drives it). The reference has no multi-device code: it runs one cache
// per sequence and splits a request's heads over std::thread (kvcache.hpp:272-274).
//
//   kvq_shard_assign  which (request, KV head) units a rank owns: contiguous request slices
//                     when batch >= world, else units dealt round-robin (u = b * H + h);
//   kvq_shard_place   the gather's last hop on the destination rank: every rank's output
//                     rows, already collected into one device buffer [world][width] (an NCCL
//                     gather), scattered into the global [B][H][G][d] order by one kernel
//                     and copied to the host once.
#include "capi_internal.cuh"

using namespace kvqb::capi;

namespace {

// One CTA per (rank, local row): 16-byte moves when the row allows it.
__global__ void place_rows_kernel(const float* __restrict__ parts, size_t width, const long long* __restrict__ unit_of,
                                  int max_units, size_t row, float* __restrict__ out) {
    const int r = blockIdx.y, i = blockIdx.x;
    const long long u = unit_of[(size_t)r * max_units + i];
    if (u < 0) return;
    const float* src = parts + (size_t)r * width + (size_t)i * row;
    float* dst = out + (size_t)u * row;
    if ((row & 3) == 0 && ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) == 0) {
        for (size_t k = threadIdx.x; k < row / 4; k += blockDim.x)
            reinterpret_cast<float4*>(dst)[k] = reinterpret_cast<const float4*>(src)[k];
    } else {
        for (size_t k = threadIdx.x; k < row; k += blockDim.x) dst[k] = src[k];
    }
}

void assign(size_t batch, size_t kv_heads, int world, int rank, std::vector<long long>& units) {
    units.clear();
    if (batch >= (size_t)world) {  // contiguous slices; the first batch % world ranks take one more
        const size_t base = batch / world, extra = batch % world;
        const size_t start = rank * base + std::min<size_t>(rank, extra);
        const size_t n = base + ((size_t)rank < extra ? 1 : 0);
        for (size_t b = start; b < start + n; ++b)
            for (size_t h = 0; h < kv_heads; ++h) units.push_back((long long)(b * kv_heads + h));
    } else {
        for (size_t u = rank; u < batch * kv_heads; u += world) units.push_back((long long)u);
    }
}

}  // namespace

extern "C" {

int kvq_shard_assign(size_t batch, size_t kv_heads, int world, int rank, long long* units, size_t capacity,
                     size_t* count) {
    return guarded([&] {
        if (world < 1 || rank < 0 || rank >= world) raise(KVQ_ERR_DOMAIN, "shard_assign: rank outside [0, world)");
        std::vector<long long> u;
        assign(batch, kv_heads, world, rank, u);
        if (count) *count = u.size();
        if (units) {
            if (capacity < u.size()) raise(KVQ_ERR_DOMAIN, "shard_assign: units buffer too small");
            std::copy(u.begin(), u.end(), units);
        }
    });
}

int kvq_shard_place(const float* parts, int world, size_t width, size_t batch, size_t kv_heads, size_t row,
                    float* out, int out_on_device, void* stream) {
    return guarded([&] {
        if (world < 1) raise(KVQ_ERR_DOMAIN, "shard_place: world < 1");
        const size_t total = batch * kv_heads;
        if (total == 0 || row == 0) return;
        require_device();
        std::vector<std::vector<long long>> share(world);
        size_t max_units = 0;
        for (int r = 0; r < world; ++r) {
            assign(batch, kv_heads, world, r, share[r]);
            max_units = std::max(max_units, share[r].size());
        }
        if (max_units * row > width) raise(KVQ_ERR_DOMAIN, "shard_place: width smaller than the largest share");
        std::vector<long long> unit_of((size_t)world * max_units, -1);
        for (int r = 0; r < world; ++r) std::copy(share[r].begin(), share[r].end(), unit_of.begin() + (size_t)r * max_units);
        cudaStream_t s = static_cast<cudaStream_t>(stream);
        DevBuf<long long> d_map(unit_of.size());
        d_map.upload(unit_of.data(), unit_of.size(), s);
        DevBuf<float> staging;
        float* dst = out;
        if (!out_on_device) {
            staging.alloc(total * row);
            dst = staging.p;
        }
        place_rows_kernel<<<dim3((unsigned)max_units, (unsigned)world), 128, 0, s>>>(parts, width, d_map.p,
                                                                                    (int)max_units, row, dst);
        ck(cudaGetLastError(), "shard_place launch");
        kvqb::note_launch(1);
        if (!out_on_device) staging.download(out, total * row, s);
        sync(s);
    });
}

}  // extern "C"
