// brandes.cu — exact betweenness centrality on the device (validation
// oracle for the sampler).
//
// The reference validates KADABRA against an exact all-pairs oracle
// (tests/test_util.hpp:164-206 ApspOracle, O(n^2) memory) and acceptance.cpp
// compares scores within eps of Brandes-normalised BC. That is infeasible on
// the CPU beyond ~10^4 vertices; here Brandes' algorithm (double sigma, exact
// dependency accumulation) runs one source per thread block:
//
//   * persistent grid, dynamic source tickets; per block a private region
//     (dist i32, sigma f64, delta f64, BFS order u32, bc partial f64);
//   * forward BFS level by level: one warp per frontier vertex claims
//     unvisited neighbours (CAS on dist), then sigma of the new level is
//     PULLED from its predecessors (sigma[v] = sum over N(v) at level L), so
//     no floating-point atomics and no per-source clearing of sigma;
//   * backward pass in successor form: delta[w] = sum over successors v of
//     sigma[w] / sigma[v] * (1 + delta[v]), level by level from the deepest;
//     bc_partial[w] += delta[w] (w != s), owned by the block, no atomics;
//   * only dist is reset afterwards (over the BFS order); sigma/delta are
//     assigned before they are read.
//
// Scores are normalised by n(n-1) (ordered pairs), as KADABRA's estimate
// data[v]/tau and oracle/oracle.c or_brandes. Summation order differs from
// the sequential predecessor-push form, so results agree to rounding.
#include <algorithm>
#include <vector>

#include "device.cuh"

namespace adsb {

namespace {

constexpr int kBT = 256;
constexpr int kWarps = kBT / 32;

struct BrandesParams {
    const uint32_t* off;
    const uint32_t* nbrs;
    uint32_t n;
    uint32_t sources;       // sources [0, sources) (all vertices)
    unsigned long long* ticket;
    int32_t* dist;          // blocks * n
    double* sigma;          // blocks * n
    double* delta;          // blocks * n
    uint32_t* order;        // blocks * n
    double* bc;             // blocks * n partial sums
};

__global__ void init_region(int32_t* dist, double* bc, size_t count) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        dist[i] = -1;
        bc[i] = 0.0;
    }
}

__global__ void __launch_bounds__(kBT) brandes_kernel(BrandesParams p) {
    __shared__ unsigned long long s_src;
    __shared__ uint32_t s_tail;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t base = static_cast<size_t>(blockIdx.x) * p.n;
    int32_t* dist = p.dist + base;
    double* sigma = p.sigma + base;
    double* delta = p.delta + base;
    uint32_t* order = p.order + base;
    double* bc = p.bc + base;
    for (;;) {
        if (threadIdx.x == 0) s_src = atomicAdd(p.ticket, 1ull);
        __syncthreads();
        const unsigned long long src = s_src;
        if (src >= p.sources) break;
        const uint32_t s = static_cast<uint32_t>(src);
        if (threadIdx.x == 0) {
            dist[s] = 0;
            sigma[s] = 1.0;
            order[0] = s;
            s_tail = 1;
        }
        __syncthreads();
        // forward: levels are contiguous ranges of `order` (BFS order); the
        // backward pass finds each level's start by binary search on dist
        uint32_t lo = 0, hi = 1;
        int32_t L = 0;
        while (lo < hi) {
            // claim level L+1 (one warp per frontier vertex)
            for (uint32_t i = lo + warp; i < hi; i += kWarps) {
                const uint32_t u = order[i];
                const uint32_t b = p.off[u], e = p.off[u + 1];
                for (uint32_t j = b + lane; j < e; j += 32) {
                    const uint32_t v = p.nbrs[j];
                    bool won = false;
                    if (__ldcg(dist + v) < 0) won = atomicCAS(dist + v, -1, L + 1) == -1;
                    const unsigned m = __activemask();
                    const unsigned wb = __ballot_sync(m, won);
                    if (wb) {
                        const int leader = __ffs(wb) - 1;
                        uint32_t pos = 0;
                        if (static_cast<int>(lane) == leader) pos = atomicAdd(&s_tail, __popc(wb));
                        pos = __shfl_sync(m, pos, leader);
                        if (won) order[pos + __popc(wb & ((1u << lane) - 1u))] = v;
                    }
                }
            }
            __syncthreads();
            const uint32_t nhi = s_tail;
            // sigma of level L+1, pulled from level L
            for (uint32_t i = hi + warp; i < nhi; i += kWarps) {
                const uint32_t v = order[i];
                const uint32_t b = p.off[v], e = p.off[v + 1];
                double acc = 0.0;
                for (uint32_t j = b + lane; j < e; j += 32) {
                    const uint32_t u = p.nbrs[j];
                    if (__ldcg(dist + u) == L) acc += __ldcg(sigma + u);
                }
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
                if (lane == 0) sigma[v] = acc;
            }
            __syncthreads();
            lo = hi;
            hi = nhi;
            ++L;
        }
        // backward, deepest level first: levels are contiguous ranges of order
        const uint32_t tail = hi;
        uint32_t end = tail;
        while (end > 0) {
            const int32_t lev = __ldcg(dist + order[end - 1]);
            // start of this level: binary search over order positions [0, end)
            // (dist is non-decreasing along order)
            uint32_t l = 0, r = end - 1;
            while (l < r) {
                const uint32_t mid = (l + r) >> 1;
                if (__ldcg(dist + order[mid]) < lev) l = mid + 1;
                else r = mid;
            }
            const uint32_t beg = l;
            for (uint32_t i = beg + warp; i < end; i += kWarps) {
                const uint32_t w = order[i];
                const uint32_t b = p.off[w], e = p.off[w + 1];
                const double sw = __ldcg(sigma + w);
                double acc = 0.0;
                for (uint32_t j = b + lane; j < e; j += 32) {
                    const uint32_t v = p.nbrs[j];
                    if (__ldcg(dist + v) == lev + 1) acc += sw / __ldcg(sigma + v) * (1.0 + __ldcg(delta + v));
                }
#pragma unroll
                for (int d = 16; d >= 1; d >>= 1) acc += __shfl_xor_sync(0xFFFFFFFFu, acc, d);
                if (lane == 0) {
                    delta[w] = acc;
                    if (w != s) bc[w] += acc;
                }
            }
            __syncthreads();
            end = beg;
        }
        for (uint32_t i = threadIdx.x; i < tail; i += kBT) dist[order[i]] = -1;
        __syncthreads();
    }
}

__global__ void reduce_bc(const double* part, uint32_t blocks, uint32_t n, double scale, double* out) {
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        double acc = 0.0;
        for (uint32_t b = 0; b < blocks; ++b) acc += part[static_cast<size_t>(b) * n + v];
        out[v] = acc * scale;
    }
}

}  // namespace

// Exact normalised BC of every vertex into host_bc (n doubles). Returns the
// device time in milliseconds.
double device_exact_bc(DeviceContext& ctx, double* host_bc) {
    const uint32_t n = ctx.graph.n;
    if (n == 0) return 0.0;
    DeviceRuntime& rt = *ctx.rt;
    cudaStream_t st = rt.stream;
    int per_sm = 0;
    ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, brandes_kernel, kBT, 0));
    size_t free_b = 0, total_b = 0;
    ADSB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t per_block = static_cast<size_t>(n) * (4 + 8 + 8 + 4 + 8);
    size_t blocks = static_cast<size_t>(num_sms(ctx.device)) * std::max(per_sm, 1);
    blocks = std::min<size_t>(blocks, static_cast<size_t>(free_b * 0.5) / per_block);
    blocks = std::min<size_t>(blocks, n);
    if (blocks == 0) fail(ADSB_ERR_CUDA, "not enough device memory for exact BC scratch");
    DevBuf<int32_t> dist(blocks * n);
    DevBuf<double> sigma(blocks * n), delta(blocks * n), bc(blocks * n), out(n);
    DevBuf<uint32_t> order(blocks * n);
    DevBuf<unsigned long long> ticket(1);
    ADSB_CUDA(cudaMemsetAsync(ticket.ptr, 0, sizeof(unsigned long long), st));
    init_region<<<static_cast<unsigned>(num_sms(ctx.device) * 8), 256, 0, st>>>(dist.ptr, bc.ptr, blocks * n);
    BrandesParams p{};
    p.off = ctx.graph.offsets.ptr;
    p.nbrs = ctx.graph.nbrs.ptr;
    p.n = n;
    p.sources = n;
    p.ticket = ticket.ptr;
    p.dist = dist.ptr;
    p.sigma = sigma.ptr;
    p.delta = delta.ptr;
    p.order = order.ptr;
    p.bc = bc.ptr;
    cudaEvent_t ev0, ev1;
    ADSB_CUDA(cudaEventCreate(&ev0));
    ADSB_CUDA(cudaEventCreate(&ev1));
    ADSB_CUDA(cudaEventRecord(ev0, st));
    brandes_kernel<<<static_cast<unsigned>(blocks), kBT, 0, st>>>(p);
    ADSB_CUDA(cudaGetLastError());
    ADSB_CUDA(cudaEventRecord(ev1, st));
    const double pairs = static_cast<double>(n) * static_cast<double>(n - 1);
    reduce_bc<<<static_cast<unsigned>(num_sms(ctx.device) * 8), 256, 0, st>>>(bc.ptr, static_cast<uint32_t>(blocks), n,
                                                      n > 1 ? 1.0 / pairs : 0.0, out.ptr);
    ADSB_CUDA(cudaGetLastError());
    ADSB_CUDA(cudaMemcpyAsync(host_bc, out.ptr, static_cast<size_t>(n) * sizeof(double), cudaMemcpyDeviceToHost, st));
    ADSB_CUDA(cudaStreamSynchronize(st));
    float ms = 0.f;
    ADSB_CUDA(cudaEventElapsedTime(&ms, ev0, ev1));
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    return ms;
}

}  // namespace adsb
