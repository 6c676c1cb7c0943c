// device_graph.cu — device CSR replica and the preprocessing kernels
// (K5 cc_label, K6 bfs_level, argmax degree) that replace, on the GPU,
//   graph.hpp:153-175 connected_components
//   graph.hpp:178-197 eccentricity
//   graph.hpp:202-214 diameter_upper_bound
// (paths relative to /root/reference/proj/include/adsamp/).
//
// Components: lock-free union-find hooking (larger root -> smaller root), so
// every root is its component's smallest vertex; ranking the roots in id
// order then reproduces the reference's DFS numbering exactly. Edges are
// linked Afforest-style: two sampled neighbours per vertex first, then the
// full adjacency only of vertices outside the (sampled) giant component.
// D_ub: one multi-source, level-synchronous BFS from every component's
// max-degree vertex (lowest id on ties); the deepest level is the largest
// eccentricity, D_ub = 2 * that.
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <map>
#include <mutex>

#include "device.cuh"

namespace adsb {

namespace {

constexpr uint32_t kInf = 0xFFFFFFFFu;

// Root with path halving. Parent pointers only ever decrease (hooks link the
// larger root below the smaller; halving skips to a smaller ancestor), and a
// racing halving write always stores an ancestor, so connectivity is safe
// with plain stores while hooking. uf_compress needs kMonotone: there a late
// plain halving write could overwrite parent[v] = root with a non-root
// ancestor and mislabel v, so every write is an atomicMin.
template <bool kMonotone>
__device__ __forceinline__ uint32_t uf_root(uint32_t* parent, uint32_t v) {
    volatile uint32_t* p = parent;
    uint32_t cur = p[v];
    if (cur != v) {
        uint32_t prev = v, next;
        while (cur > (next = p[cur])) {
            if (kMonotone) atomicMin(parent + prev, next);
            else p[prev] = next;
            prev = cur;
            cur = next;
        }
    }
    return cur;
}

__global__ void uf_init(uint32_t* parent, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        parent[v] = v;
}

// Union of the trees holding u and w: hook the larger root below the smaller
// (roots stay the smallest id of their component).
__device__ __forceinline__ void uf_link(uint32_t* parent, uint32_t u, uint32_t w) {
    uint32_t ru = uf_root<false>(parent, u), rw = uf_root<false>(parent, w);
    while (ru != rw) {
        const uint32_t hi = max(ru, rw), lo = min(ru, rw);
        const uint32_t old = atomicCAS(&parent[hi], hi, lo);
        if (old == hi) break;
        ru = uf_root<false>(parent, old);
        rw = uf_root<false>(parent, lo);
    }
}

// Afforest-style sampling: round r links every vertex to its r-th neighbour.
// Two rounds already join nearly all of a giant component.
__global__ void uf_link_round(const uint32_t* __restrict__ off, const uint32_t* __restrict__ nbrs, uint32_t* parent,
                              uint32_t n, uint32_t r) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t b = off[v];
        if (off[v + 1] - b > r) uf_link(parent, v, nbrs[b + r]);
    }
}

// The most frequent root among 256 evenly spaced vertices (one block).
__global__ void uf_sample_mode(uint32_t* parent, uint32_t n, uint32_t* mode) {
    __shared__ uint32_t roots[256];
    __shared__ unsigned long long wbest[8];
    const uint32_t i = threadIdx.x;
    const uint32_t v = static_cast<uint32_t>((static_cast<uint64_t>(i) * n) / 256);
    roots[i] = uf_root<false>(parent, min(v, n - 1));
    __syncthreads();
    uint32_t count = 0;
    for (uint32_t j = 0; j < 256; ++j) count += roots[j] == roots[i] ? 1u : 0u;
    // max of (count, root) by warp shuffles, then over the 8 warps (no 64-bit
    // shared atomics: they are CAS loops on sm_100)
    unsigned long long key = (static_cast<unsigned long long>(count) << 32) | roots[i];
    for (int d = 16; d; d >>= 1) key = max(key, __shfl_xor_sync(0xFFFFFFFFu, key, d));
    if ((i & 31) == 0) wbest[i >> 5] = key;
    __syncthreads();
    if (i == 0) {
        unsigned long long best = 0;
        for (int w = 0; w < 8; ++w) best = max(best, wbest[w]);
        *mode = static_cast<uint32_t>(best);
    }
}

// The rest of the edges, only for vertices outside the sampled giant tree:
// one warp per vertex, lanes over its adjacency beyond the two sampled
// entries (an edge into the giant is seen from the outside endpoint).
__global__ void uf_link_rest(const uint32_t* __restrict__ off, const uint32_t* __restrict__ nbrs, uint32_t* parent,
                             uint32_t n, const uint32_t* mode) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    const uint32_t giant = *mode;
    for (uint32_t u = warp; u < n; u += nwarps) {
        if (uf_root<false>(parent, u) == giant) continue;  // warp-uniform
        const uint32_t b = off[u], e = off[u + 1];
        for (uint32_t i = b + 2 + lane; i < e; i += 32) uf_link(parent, u, nbrs[i]);
    }
}

__global__ void uf_compress(uint32_t* parent, uint32_t* is_root, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t r = uf_root<true>(parent, v);  // hooking is complete: r is final
        atomicMin(parent + v, r);
        is_root[v] = r == v ? 1u : 0u;
    }
}

__global__ void uf_label(const uint32_t* parent, const uint32_t* root_rank, uint32_t* label, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        label[v] = root_rank[parent[v]];
}

// graph.hpp:208: start = max degree, lowest id on ties -> max of (deg, ~v)
__global__ void argmax_degree(const uint32_t* __restrict__ off, const uint32_t* __restrict__ label,
                              unsigned long long* best, uint32_t n) {
    // grid-stride with whole warps (n rounded up) so the warp reduction below
    // always has every lane present; one atomic per warp when the warp's
    // vertices share a component (the common case: one giant component)
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t span = (n + 31u) & ~31u;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < span; v += stride) {
        const bool live = v < n;
        const uint32_t lab = live ? label[v] : 0xFFFFFFFFu;
        unsigned long long key = live ? (static_cast<unsigned long long>(off[v + 1] - off[v]) << 32) |
                                            static_cast<uint32_t>(~v)
                                      : 0ull;
        const uint32_t lab0 = __shfl_sync(0xFFFFFFFFu, lab, 0);
        if (__all_sync(0xFFFFFFFFu, lab == lab0 || !live)) {
#pragma unroll
            for (int d = 16; d >= 1; d >>= 1) {
                const unsigned long long o = __shfl_xor_sync(0xFFFFFFFFu, key, d);
                key = o > key ? o : key;
            }
            if ((threadIdx.x & 31) == 0 && lab0 != 0xFFFFFFFFu) atomicMax(&best[lab0], key);
        } else if (live) {
            atomicMax(&best[lab], key);
        }
    }
}

__global__ void seed_sources(const unsigned long long* best, uint32_t comps, uint32_t* dist,
                             uint32_t* frontier, uint32_t* count0) {
    for (uint32_t c = blockIdx.x * blockDim.x + threadIdx.x; c < comps; c += gridDim.x * blockDim.x) {
        const uint32_t s = ~static_cast<uint32_t>(best[c] & 0xFFFFFFFFull);
        dist[s] = 0;
        frontier[c] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *count0 = comps;
}

__global__ void init_dist(uint32_t* dist, uint32_t n) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
        dist[v] = kInf;
}

// Next free position of a counter for the converged lanes of a warp (one
// atomic per group).
__device__ __forceinline__ uint32_t warp_agg_inc(uint32_t* ctr) {
    namespace cg = cooperative_groups;
    const cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, g.size());
    return g.shfl(base, 0) + g.thread_rank();
}

// K6: one level of a (multi-source) BFS, direction chosen on the device from
// the frontier size (every level of a chunk is launched without a host check):
// * large frontier (> n/24): bottom-up. Every unvisited vertex looks for a
//   neighbour on this level and stops at the first; only its own thread
//   writes dist[v]. This covers the few huge middle levels of small-world graphs.
// * frontier smaller than the grid: one block per frontier vertex (a hub
//   source would otherwise be walked by a single warp);
// * otherwise one warp per frontier vertex.
// The depth and dist values equal any level-synchronous BFS's.
__global__ void bfs_level(const uint32_t* __restrict__ off, const uint32_t* __restrict__ nbrs,
                          uint32_t* dist, const uint32_t* __restrict__ fin, const uint32_t* cnt_in,
                          uint32_t* fout, uint32_t* cnt_out, uint32_t level, uint32_t n) {
    const uint32_t count = *cnt_in;
    if (count == 0) return;
    if (count > n / 24) {
        for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
            if (dist[v] != kInf) continue;
            const uint32_t b = off[v], e = off[v + 1];
            for (uint32_t j = b; j < e; ++j) {
                if (__ldcg(dist + nbrs[j]) == level) {
                    dist[v] = level + 1;
                    fout[warp_agg_inc(cnt_out)] = v;
                    break;
                }
            }
        }
        return;
    }
    if (count <= gridDim.x) {
        for (uint32_t i = blockIdx.x; i < count; i += gridDim.x) {
            const uint32_t u = fin[i];
            const uint32_t b = off[u], e = off[u + 1];
            for (uint32_t j = b + threadIdx.x; j < e; j += blockDim.x) {
                const uint32_t w = nbrs[j];
                if (dist[w] == kInf && atomicCAS(&dist[w], kInf, level + 1) == kInf) fout[warp_agg_inc(cnt_out)] = w;
            }
        }
        return;
    }
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = warp; i < count; i += nwarps) {
        const uint32_t u = fin[i];
        const uint32_t b = off[u], e = off[u + 1];
        for (uint32_t j = b + lane; j < e; j += 32) {
            const uint32_t w = nbrs[j];
            if (dist[w] == kInf && atomicCAS(&dist[w], kInf, level + 1) == kInf) fout[warp_agg_inc(cnt_out)] = w;
        }
    }
}

}  // namespace

int num_sms(int device) {
    int v = 0;
    ADSB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device));
    return v;
}

int resolve_device(int requested) {
    int count = 0;
    const cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        fail(ADSB_ERR_CUDA, std::string("no CUDA device available (") + cudaGetErrorString(e) +
                                "); the adsb engine has no CPU fallback");
    int dev = requested;
    if (dev < 0) ADSB_CUDA(cudaGetDevice(&dev));
    if (dev >= count) invalid("CUDA device ordinal out of range");
    return dev;
}

DeviceRuntime& device_runtime(int device) {
    static std::mutex mu;
    static std::map<int, DeviceRuntime*> runtimes;  // intentionally leaked (see device.cuh)
    std::lock_guard<std::mutex> lock(mu);
    DeviceRuntime*& rt = runtimes[device];
    if (!rt) {
        ADSB_CUDA(cudaSetDevice(device));
        auto* r = new DeviceRuntime;
        r->device = device;
        ADSB_CUDA(cudaStreamCreateWithFlags(&r->stream, cudaStreamNonBlocking));
        ADSB_CUDA(cudaStreamCreateWithFlags(&r->stream2, cudaStreamNonBlocking));
        r->pinned = PinnedBuf<unsigned long long>(128);
        rt = r;
    }
    return *rt;
}

DevBuf<uint32_t> take_buffer(DeviceRuntime& rt, size_t count) {
    count = std::max<size_t>(count, 1);
    {
        std::lock_guard<std::mutex> lock(rt.spare_mu);
        size_t best = rt.spare.size();
        for (size_t i = 0; i < rt.spare.size(); ++i)
            if (rt.spare[i].count >= count && rt.spare[i].count <= 2 * count &&
                (best == rt.spare.size() || rt.spare[i].count < rt.spare[best].count))
                best = i;
        if (best != rt.spare.size()) {
            DevBuf<uint32_t> b = std::move(rt.spare[best]);
            rt.spare.erase(rt.spare.begin() + static_cast<long>(best));
            return b;
        }
    }
    ADSB_CUDA(cudaSetDevice(rt.device));
    return DevBuf<uint32_t>(count);
}

void give_buffer(DeviceRuntime& rt, DevBuf<uint32_t>&& b) {
    if (!b.ptr) return;
    std::lock_guard<std::mutex> lock(rt.spare_mu);
    rt.spare.push_back(std::move(b));
    size_t total = 0;
    for (auto& x : rt.spare) total += x.bytes();
    while (rt.spare.size() > 8 || total > (size_t{16} << 30)) {  // keep at most 8 buffers / 16 GiB
        total -= rt.spare.front().bytes();
        rt.spare.erase(rt.spare.begin());
    }
}

DeviceContext::~DeviceContext() {
    if (!rt) return;
    give_buffer(*rt, std::move(graph.offsets));
    give_buffer(*rt, std::move(graph.nbrs));
    give_buffer(*rt, std::move(labels));
}

std::unique_ptr<DeviceContext> make_device_context(const HostGraph& g, int device) {
    if (g.nnz() >= 0xFFFFFFFFull) invalid("device CSR needs fewer than 2^32 adjacency entries");
    ADSB_CUDA(cudaSetDevice(device));
    auto ctx = std::make_unique<DeviceContext>();
    ctx->device = device;
    ctx->rt = &device_runtime(device);
    std::lock_guard<std::mutex> lock(ctx->rt->mu);
    DeviceGraph& dg = ctx->graph;
    dg.device = device;
    dg.n = g.n;
    dg.nnz = g.nnz();
    // u32 offsets on the device: narrow on the host, then one copy each.
    std::vector<uint32_t, NoInitAlloc<uint32_t>> off32(g.offsets.size());  // page-locked when large
    for (size_t i = 0; i < off32.size(); ++i) off32[i] = static_cast<uint32_t>(g.offsets[i]);
    for (uint32_t u = 0; u < g.n; ++u) dg.max_degree = std::max<uint32_t>(dg.max_degree, off32[u + 1] - off32[u]);
    dg.offsets = take_buffer(*ctx->rt, off32.size());
    dg.nbrs = take_buffer(*ctx->rt, std::max<uint64_t>(1, g.nnz()));
    ctx->labels = take_buffer(*ctx->rt, std::max<uint32_t>(1, g.n));
    ADSB_CUDA(cudaMemcpyAsync(dg.offsets.ptr, off32.data(), off32.size() * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, ctx->rt->stream));
    if (g.nnz())
        ADSB_CUDA(cudaMemcpyAsync(dg.nbrs.ptr, g.nbrs.data(), g.nnz() * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, ctx->rt->stream));
    ADSB_CUDA(cudaStreamSynchronize(ctx->rt->stream));
    return ctx;
}

void StreamingUpload::chunk(uint64_t b, uint64_t e, uint64_t nb, uint64_t ne, const HostGraph& g) {
    uint32_t md = 0;
    for (uint64_t u = b; u < e; ++u) {
        off32[u] = static_cast<uint32_t>(g.offsets[u]);
        if (u + 1 < e) md = std::max<uint32_t>(md, static_cast<uint32_t>(g.offsets[u + 1] - g.offsets[u]));
    }
    // the range's last vertex ends where the range's adjacency ends
    if (e > b) md = std::max<uint32_t>(md, static_cast<uint32_t>(ne - g.offsets[e - 1]));
    uint32_t cur = max_degree.load();
    while (md > cur && !max_degree.compare_exchange_weak(cur, md)) {
    }
    DeviceGraph& dg = ctx->graph;
    ADSB_CUDA(cudaMemcpyAsync(dg.offsets.ptr + b, off32.data() + b, (e - b) * sizeof(uint32_t),
                              cudaMemcpyHostToDevice, ctx->rt->stream));
    if (ne > nb)
        ADSB_CUDA(cudaMemcpyAsync(dg.nbrs.ptr + nb, g.nbrs.data() + nb, (ne - nb) * sizeof(uint32_t),
                                  cudaMemcpyHostToDevice, ctx->rt->stream));
}

std::unique_ptr<StreamingUpload> begin_streaming_upload(uint32_t n, uint64_t nnz, int device) {
    if (nnz >= 0xFFFFFFFFull) invalid("device CSR needs fewer than 2^32 adjacency entries");
    ADSB_CUDA(cudaSetDevice(device));
    auto up = std::make_unique<StreamingUpload>();
    up->ctx = std::make_unique<DeviceContext>();
    DeviceContext& ctx = *up->ctx;
    ctx.device = device;
    ctx.rt = &device_runtime(device);
    up->lock = std::unique_lock<std::mutex>(ctx.rt->mu);
    ctx.graph.device = device;
    ctx.graph.n = n;
    ctx.graph.nnz = nnz;
    up->off32.resize(static_cast<size_t>(n) + 1);
    ctx.graph.offsets = take_buffer(*ctx.rt, static_cast<size_t>(n) + 1);
    ctx.graph.nbrs = take_buffer(*ctx.rt, std::max<uint64_t>(1, nnz));
    ctx.labels = take_buffer(*ctx.rt, std::max<uint32_t>(1, n));
    return up;
}

std::unique_ptr<DeviceContext> finish_streaming_upload(std::unique_ptr<StreamingUpload> up, const HostGraph& g) {
    DeviceContext& ctx = *up->ctx;
    up->off32[g.n] = static_cast<uint32_t>(g.offsets[g.n]);
    ADSB_CUDA(cudaMemcpyAsync(ctx.graph.offsets.ptr + g.n, up->off32.data() + g.n, sizeof(uint32_t),
                              cudaMemcpyHostToDevice, ctx.rt->stream));
    ctx.graph.max_degree = up->max_degree.load();
    // off32 is released below: the copies from it must have landed
    ADSB_CUDA(cudaStreamSynchronize(ctx.rt->stream));
    return std::move(up->ctx);
}

void abort_streaming_upload(std::unique_ptr<StreamingUpload> up) {
    if (up && up->ctx && up->ctx->rt) cudaStreamSynchronize(up->ctx->rt->stream);
}

static unsigned grid_for(uint64_t work, int device, unsigned block = 256) {
    const uint64_t want = (work + block - 1) / block;
    const uint64_t cap = static_cast<uint64_t>(num_sms(device)) * 8;
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min(want, cap)));
}

uint32_t device_components(DeviceContext& ctx) {
    if (ctx.labels_ready) return ctx.num_components;
    const uint32_t n = ctx.graph.n;
    cudaStream_t s = ctx.rt->stream;
    uint32_t* parent = ctx.rt->pool.get<uint32_t>(Scratch::kParent, n);
    uint32_t* is_root = ctx.rt->pool.get<uint32_t>(Scratch::kIsRoot, n + 1);  // zero tail: scanned with n+1 inputs
    uint32_t* rank = ctx.rt->pool.get<uint32_t>(Scratch::kRank, n + 1);
    if (ctx.labels.count < n) ctx.labels = take_buffer(*ctx.rt, n);
    const unsigned g = grid_for(n, ctx.device);
    uint32_t* mode = ctx.rt->pool.get<uint32_t>(Scratch::kMode, 1);
    uf_init<<<g, 256, 0, s>>>(parent, n);
    for (uint32_t r = 0; r < 2; ++r) uf_link_round<<<g, 256, 0, s>>>(ctx.graph.offsets.ptr, ctx.graph.nbrs.ptr, parent, n, r);
    uf_sample_mode<<<1, 256, 0, s>>>(parent, n, mode);
    uf_link_rest<<<grid_for(static_cast<uint64_t>(n) * 32, ctx.device), 256, 0, s>>>(
        ctx.graph.offsets.ptr, ctx.graph.nbrs.ptr, parent, n, mode);
    uf_compress<<<g, 256, 0, s>>>(parent, is_root, n);
    ADSB_CUDA(cudaMemsetAsync(is_root + n, 0, sizeof(uint32_t), s));
    size_t temp_bytes = 0;
    ADSB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, is_root, rank, n + 1, s));
    uint8_t* temp = ctx.rt->pool.get<uint8_t>(Scratch::kCubTemp, temp_bytes);
    ADSB_CUDA(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, is_root, rank, n + 1, s));
    uf_label<<<g, 256, 0, s>>>(parent, rank, ctx.labels.ptr, n);
    uint32_t* comps_h = reinterpret_cast<uint32_t*>(ctx.rt->pinned.ptr);
    ADSB_CUDA(cudaMemcpyAsync(comps_h, rank + n, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
    ADSB_CUDA(cudaStreamSynchronize(s));
    ADSB_CUDA(cudaGetLastError());
    const uint32_t comps = *comps_h;
    ctx.num_components = comps;
    ctx.labels_ready = true;
    return comps;
}

// Level-synchronous BFS from `sources` (already written into frontier A with
// dist 0); returns the deepest non-empty level. Levels are launched in
// chunks so the host synchronises once per chunk, not once per level.
static uint64_t bfs_depth(DeviceContext& ctx, uint32_t* dist, uint32_t* fa, uint32_t* fb, uint32_t* counts) {
    const uint32_t n = ctx.graph.n;
    cudaStream_t s = ctx.rt->stream;
    const unsigned grid = static_cast<unsigned>(num_sms(ctx.device) * 8);
    uint32_t kChunk = 8;  // levels launched per host check: 8 first, then 32
    uint32_t level = 0;
    uint32_t* host = reinterpret_cast<uint32_t*>(ctx.rt->pinned.ptr);  // 64 words of pinned staging
    for (;;) {
        for (uint32_t k = 0; k < kChunk && level + k + 1 <= n; ++k) {
            const uint32_t L = level + k;
            uint32_t* fin = (L & 1) ? fb : fa;
            uint32_t* fout = (L & 1) ? fa : fb;
            bfs_level<<<grid, 256, 0, s>>>(ctx.graph.offsets.ptr, ctx.graph.nbrs.ptr, dist, fin, counts + L, fout,
                                           counts + L + 1, L, n);
        }
        const uint32_t avail = std::min<uint32_t>(kChunk, n - level);
        ADSB_CUDA(cudaMemcpyAsync(host, counts + level + 1, avail * sizeof(uint32_t),
                                  cudaMemcpyDeviceToHost, s));
        ADSB_CUDA(cudaStreamSynchronize(s));
        ADSB_CUDA(cudaGetLastError());
        for (uint32_t k = 0; k < avail; ++k)
            if (host[k] == 0) return level + k;
        level += avail;
        if (level >= n) return level;
        kChunk = 32;
    }
}

uint64_t device_eccentricity(DeviceContext& ctx, uint32_t source) {
    const uint32_t n = ctx.graph.n;
    if (source >= n) invalid("source vertex out of range");
    cudaStream_t s = ctx.rt->stream;
    uint32_t* dist = ctx.rt->pool.get<uint32_t>(Scratch::kDist, n);
    uint32_t* fa = ctx.rt->pool.get<uint32_t>(Scratch::kFrontA, n);
    uint32_t* fb = ctx.rt->pool.get<uint32_t>(Scratch::kFrontB, n);
    uint32_t* counts = ctx.rt->pool.get<uint32_t>(Scratch::kLevelCounts, static_cast<size_t>(n) + 2);
    ADSB_CUDA(cudaMemsetAsync(counts, 0, (static_cast<size_t>(n) + 2) * sizeof(uint32_t), s));
    init_dist<<<grid_for(n, ctx.device), 256, 0, s>>>(dist, n);
    const uint32_t zero = 0, one = 1;
    ADSB_CUDA(cudaMemcpyAsync(dist + source, &zero, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    ADSB_CUDA(cudaMemcpyAsync(fa, &source, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    ADSB_CUDA(cudaMemcpyAsync(counts, &one, sizeof(uint32_t), cudaMemcpyHostToDevice, s));
    ADSB_CUDA(cudaStreamSynchronize(s));  // the host-side sources above are stack values
    return bfs_depth(ctx, dist, fa, fb, counts);
}

uint64_t device_diameter_bound(DeviceContext& ctx) {
    if (ctx.dub_ready) return ctx.diameter_bound;
    const uint32_t n = ctx.graph.n;
    const uint32_t comps = device_components(ctx);
    cudaStream_t s = ctx.rt->stream;
    unsigned long long* best = ctx.rt->pool.get<unsigned long long>(Scratch::kBest, comps);
    uint32_t* dist = ctx.rt->pool.get<uint32_t>(Scratch::kDist, n);
    uint32_t* fa = ctx.rt->pool.get<uint32_t>(Scratch::kFrontA, n);
    uint32_t* fb = ctx.rt->pool.get<uint32_t>(Scratch::kFrontB, n);
    uint32_t* counts = ctx.rt->pool.get<uint32_t>(Scratch::kLevelCounts, static_cast<size_t>(n) + 2);
    ADSB_CUDA(cudaMemsetAsync(best, 0, static_cast<size_t>(comps) * sizeof(unsigned long long), s));
    ADSB_CUDA(cudaMemsetAsync(counts, 0, (static_cast<size_t>(n) + 2) * sizeof(uint32_t), s));
    argmax_degree<<<grid_for(n, ctx.device), 256, 0, s>>>(ctx.graph.offsets.ptr, ctx.labels.ptr, best, n);
    init_dist<<<grid_for(n, ctx.device), 256, 0, s>>>(dist, n);
    seed_sources<<<grid_for(comps, ctx.device), 256, 0, s>>>(best, comps, dist, fa, counts);
    ctx.diameter_bound = 2 * bfs_depth(ctx, dist, fa, fb, counts);
    ctx.dub_ready = true;
    return ctx.diameter_bound;
}

}  // namespace adsb
