// hub_index.cu — builds the hub search trees (hub_index.cuh) on the device,
// once per graph handle: sizes per vertex, an exclusive scan for the tree
// bases, then one warp per hub fills its levels bottom-up.
#include <cub/cub.cuh>

#include "device.cuh"
#include "hub_index.cuh"

namespace adsb {

namespace {

__global__ void k_hub_sizes(const uint32_t* __restrict__ off, uint32_t n, uint32_t* sizes) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        sizes[v] = hub_tree_words(off[v + 1] - off[v]);
}

// one warp per vertex range; lanes fill a hub's levels together
__global__ void k_hub_build(const uint32_t* __restrict__ off, const uint32_t* __restrict__ nbrs, uint32_t n,
                            const uint32_t* __restrict__ ref, uint32_t* keys) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t warps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t v = warp; v < n; v += warps) {
        const uint32_t o = off[v], d = off[v + 1] - o;
        if (!hub_has_tree(d)) continue;  // warp-uniform
        const uint32_t* A = nbrs + o;
        uint32_t* T = keys + ref[v];
        uint32_t n_prev = (d + kHubLeaf - 1) / kHubLeaf, off_prev = 8, k = 0;
        for (uint32_t j = lane; j < ((n_prev + 7u) & ~7u); j += 32)
            T[off_prev + j] = j < n_prev ? A[min(kHubLeaf * j + kHubLeaf - 1, d - 1)] : 0xFFFFFFFFu;
        if (lane == 0) T[1] = off_prev;
        __syncwarp();
        while (n_prev > kHubFan) {
            const uint32_t n_k = (n_prev + kHubFan - 1) / kHubFan;
            const uint32_t off_k = off_prev + ((n_prev + 7u) & ~7u);
            for (uint32_t j = lane; j < ((n_k + 7u) & ~7u); j += 32)
                T[off_k + j] = j < n_k ? T[off_prev + min(kHubFan * j + kHubFan - 1, n_prev - 1)] : 0xFFFFFFFFu;
            ++k;
            if (lane == 0) T[1 + k] = off_k;
            __syncwarp();
            off_prev = off_k;
            n_prev = n_k;
        }
        if (lane == 0) {
            T[0] = k;
            for (uint32_t i = k + 1; i < 6; ++i) T[1 + i] = 0;
            T[7] = A[d - 1];
        }
    }
}

}  // namespace

void device_hub_index(DeviceContext& ctx) {
    if (ctx.hub_ready) return;
    ctx.hub_ready = true;
    DeviceGraph& g = ctx.graph;
    if (g.n == 0 || g.max_degree < kHubTreeMinDeg) return;  // no hubs: hub_ref stays empty
    cudaStream_t s = ctx.rt->stream;
    g.hub_ref.alloc(g.n);
    const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((g.n + 255ull) / 256, num_sms(ctx.device) * 8ull));
    k_hub_sizes<<<grid, 256, 0, s>>>(g.offsets.ptr, g.n, g.hub_ref.ptr);
    ADSB_CUDA(cudaGetLastError());
    // total words = exclusive sum of the sizes + the last size
    uint32_t last_size = 0, last_base = 0;
    ADSB_CUDA(cudaMemcpyAsync(&last_size, g.hub_ref.ptr + g.n - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    size_t tmp_bytes = 0;
    ADSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, g.hub_ref.ptr, g.hub_ref.ptr, g.n, s));
    void* tmp = ctx.rt->pool.get<uint8_t>(Scratch::kCubTemp, tmp_bytes);
    ADSB_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, g.hub_ref.ptr, g.hub_ref.ptr, g.n, s));
    ADSB_CUDA(cudaMemcpyAsync(&last_base, g.hub_ref.ptr + g.n - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    ADSB_CUDA(cudaStreamSynchronize(s));
    const uint64_t words = static_cast<uint64_t>(last_base) + last_size;
    if (words == 0) {
        g.hub_ref.reset();
        return;
    }
    g.hub_keys.alloc(words);
    k_hub_build<<<num_sms(ctx.device) * 8, 256, 0, s>>>(g.offsets.ptr, g.nbrs.ptr, g.n, g.hub_ref.ptr, g.hub_keys.ptr);
    ADSB_CUDA(cudaGetLastError());
    ADSB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace adsb
