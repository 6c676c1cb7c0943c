// sampler_cta.cu — block-per-sample K1/K2 sampler with shared-memory state.
//
// Same contract as sampler.cu (bit-exact kadabra.hpp:190-258 under the
// engine.hpp:595-610 keying; paths relative to /root/reference/proj/include/
// adsamp/), restructured for B200's memory hierarchy:
//
//   * one thread block (128 or 256 threads; both are instantiated from
//     sampler_cta_body.cuh) owns one sample at a time (persistent grid,
//     dynamic tickets);
//   * the per-sample visited set (vertex -> side/dist/dag, sigma) lives in a
//     shared-memory open-addressing hash table, cleared per sample; the CSR is
//     the only global data a sample reads (L2-resident for C1-C3);
//   * every BFS level first PROBES its frontier's adjacency for the other
//     side's ball and only CLAIMS new vertices when the frontiers did not meet,
//     so the large meeting level (typically >90% of the scanned adjacency)
//     performs no insertions at all and only the two pre-meeting balls occupy
//     the table (C2: mean 121 vertices, C3: 673);
//   * frontier adjacency is flattened across the whole block: a block scan over
//     the frontier degrees, then each thread takes edges e = tid, tid+256, ...
//     and finds its owner vertex by binary search in the scan (hubs and
//     low-degree frontiers are balanced alike);
//   * a sample whose balls outgrow the table is redone with the per-block
//     dense global state (stamped 16-byte words, as sampler.cu), which is also
//     the only path for graphs whose balls are routinely large (grid, C5).
//
// The sigma-weighted backtrack (kadabra.hpp:227-242) is block-wide: a 65-bit
// block prefix sum over the ascending-neighbour candidates per round.

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>

#include "device.cuh"
#include "hub_index.cuh"
#include "rng.hpp"
#include "sampler.cuh"

#ifndef ADSB_LOAD_BATCH
#define ADSB_LOAD_BATCH 1  // adjacency loads in flight per thread in for_edges (A/B: 1 beats 2 and 4)
#endif
#ifndef ADSB_SMEM_FILTER
#define ADSB_SMEM_FILTER 0
#endif
#ifndef ADSB_GLOBAL_MINB
#define ADSB_GLOBAL_MINB 4  // min blocks/SM of the global-store-only kernel (256 threads; register budget)
#endif
#ifndef ADSB_MINB_PER_256
#define ADSB_MINB_PER_256 4  // __launch_bounds__ min blocks for 256-thread blocks (register budget)
#endif

// ADSB_PHASE_TIMING (diagnostic builds only): thread 0 of every block adds
// clock64 deltas per sampler phase into adsb_phase[]; sampler_phase_report()
// prints and resets them.
#ifdef ADSB_PHASE_TIMING
__device__ unsigned long long adsb_phase[16];
#define ADSB_PHASE_MARK(x) const long long x = clock64()
#define ADSB_PHASE_ADD(i, v) \
    do {                     \
        if (threadIdx.x == 0) atomicAdd(&adsb_phase[i], static_cast<unsigned long long>(v)); \
    } while (0)
#else
#define ADSB_PHASE_MARK(x) \
    do {                   \
    } while (0)
#define ADSB_PHASE_ADD(i, v) \
    do {                     \
    } while (0)
#endif

#ifdef ADSB_DEBUG_CHECKS
#include <cstdio>
#define ADSB_DCHECK(cond, ...)                                                              \
    do {                                                                                    \
        if (!(cond)) {                                                                      \
            printf("ADSB_DCHECK failed %s:%d block %d thread %d: %s\n", __FILE__, __LINE__,  \
                   blockIdx.x, threadIdx.x, #cond);                                         \
            __trap();                                                                       \
        }                                                                                   \
    } while (0)
#else
#define ADSB_DCHECK(cond, ...) \
    do {                       \
    } while (0)
#endif

namespace adsb {

constexpr int kModeDet = 0, kModeEpoch = 1, kModeFused = 2;

namespace bt128 {
constexpr int kBT = 128;
#include "sampler_cta_body.cuh"
}  // namespace bt128

namespace bt256 {
constexpr int kBT = 256;
#include "sampler_cta_body.cuh"
}  // namespace bt256

// 512-thread teams for the global-store-only kernel (low-degree graphs:
// half the samples in flight for the same threads, so more of each
// sample's frontier state stays in L2)
namespace bt512 {
constexpr int kBT = 512;
#include "sampler_cta_body.cuh"
}  // namespace bt512

namespace bt1024 {
constexpr int kBT = 1024;
#include "sampler_cta_body.cuh"
}  // namespace bt1024

size_t sampler_cta_smem_bytes(uint32_t hash_cap, bool vec4) {
    // sigma, key|meta, queue (+ the membership filter) (+ the vector kernels' row ranges)
    size_t bytes = static_cast<size_t>(hash_cap) * 12 + static_cast<size_t>(hash_cap / 2) * 4;
#if ADSB_SMEM_FILTER
    bytes += bt256::SmemStore::kFbWords * 4;
#endif
    if (vec4) bytes += 2 * 256 * sizeof(uint32_t);
    return bytes;
}

namespace {
template <class K>
void allow_big_smem(K kernel) {
    // dynamic shared memory up to 200 KB, within the per-block opt-in limit
    // left by the kernel's static Shared block
    int dev = 0, optin = 0;
    ADSB_CUDA(cudaGetDevice(&dev));
    ADSB_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    ADSB_CUDA(cudaFuncGetAttributes(&fa, kernel));
    const int room = optin - static_cast<int>(fa.sharedSizeBytes);
    ADSB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, std::min(200 * 1024, room)));
}
void configure_once() {
    static bool done = false;
    if (done) return;
    allow_big_smem(bt128::sampler_cta_kernel<kModeDet, false>);
    allow_big_smem(bt128::sampler_cta_kernel<kModeEpoch, false>);
    allow_big_smem(bt128::sampler_cta_kernel<kModeFused, false>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeDet, false>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeEpoch, false>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeFused, false>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeDet, false, true>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeEpoch, false, true>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeFused, false, true>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeDet, true>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeEpoch, true>);
    allow_big_smem(bt256::sampler_cta_kernel<kModeFused, true>);
    allow_big_smem(bt512::sampler_cta_kernel<kModeDet, true>);
    allow_big_smem(bt512::sampler_cta_kernel<kModeEpoch, true>);
    allow_big_smem(bt512::sampler_cta_kernel<kModeFused, true>);
    allow_big_smem(bt1024::sampler_cta_kernel<kModeDet, true>);
    allow_big_smem(bt1024::sampler_cta_kernel<kModeEpoch, true>);
    allow_big_smem(bt1024::sampler_cta_kernel<kModeFused, true>);
    done = true;
}
}  // namespace

int sampler_cta_blocks_per_sm(uint32_t hash_cap, uint32_t block_threads, bool vec4) {
    configure_once();
    const bool v = vec4 && block_threads == 256;
    const size_t dyn = sampler_cta_smem_bytes(hash_cap, v);
    int blocks = 0;
    if (block_threads == 128)
        ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, bt128::sampler_cta_kernel<kModeDet, false>, 128, dyn));
    else if (v)
        ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, bt256::sampler_cta_kernel<kModeDet, false, true>, 256, dyn));
    else
        ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, bt256::sampler_cta_kernel<kModeDet, false>, 256, dyn));
    return blocks;
}

// Global-store-only variant (no shared-memory table): used when the table is
// switched off for a graph. 128 registers, 2 blocks/SM, 4 loads in flight.
int sampler_global_blocks_per_sm() {
    configure_once();
    int blocks = 0;
    ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, bt256::sampler_cta_kernel<kModeDet, true>, 256, 0));
    return blocks;
}

void launch_sampler_cta(bool deterministic, const SamplerParams& p, cudaStream_t stream) {
    configure_once();
    const size_t dyn = sampler_cta_smem_bytes(p.hash_cap, p.vec4 && p.block_threads == 256);
    if (!p.use_smem) {
        const unsigned grid = std::min<unsigned>(p.slots, p.global_grid);
        if (p.global_threads == 1024) {
            if (deterministic) bt1024::sampler_cta_kernel<kModeDet, true><<<grid, 1024, 0, stream>>>(p);
            else bt1024::sampler_cta_kernel<kModeEpoch, true><<<grid, 1024, 0, stream>>>(p);
        } else if (p.global_threads == 512) {
            if (deterministic) bt512::sampler_cta_kernel<kModeDet, true><<<grid, 512, 0, stream>>>(p);
            else bt512::sampler_cta_kernel<kModeEpoch, true><<<grid, 512, 0, stream>>>(p);
        } else if (deterministic) bt256::sampler_cta_kernel<kModeDet, true><<<grid, 256, 0, stream>>>(p);
        else bt256::sampler_cta_kernel<kModeEpoch, true><<<grid, 256, 0, stream>>>(p);
        ADSB_CUDA(cudaGetLastError());
        return;
    }
    if (p.block_threads == 128) {
        if (deterministic) bt128::sampler_cta_kernel<kModeDet, false><<<p.blocks, 128, dyn, stream>>>(p);
        else bt128::sampler_cta_kernel<kModeEpoch, false><<<p.blocks, 128, dyn, stream>>>(p);
    } else if (p.vec4) {
        if (deterministic) bt256::sampler_cta_kernel<kModeDet, false, true><<<p.blocks, 256, dyn, stream>>>(p);
        else bt256::sampler_cta_kernel<kModeEpoch, false, true><<<p.blocks, 256, dyn, stream>>>(p);
    } else {
        if (deterministic) bt256::sampler_cta_kernel<kModeDet, false><<<p.blocks, 256, dyn, stream>>>(p);
        else bt256::sampler_cta_kernel<kModeEpoch, false><<<p.blocks, 256, dyn, stream>>>(p);
    }
    ADSB_CUDA(cudaGetLastError());
}

void launch_sampler_fused(const SamplerParams& p, cudaStream_t stream) {
    configure_once();
    const size_t dyn = sampler_cta_smem_bytes(p.hash_cap, p.vec4 && p.block_threads == 256);
    if (!p.use_smem) {
        if (p.global_threads == 1024)
            bt1024::sampler_cta_kernel<kModeFused, true><<<std::min<unsigned>(p.slots, p.global_grid), 1024, 0, stream>>>(p);
        else if (p.global_threads == 512)
            bt512::sampler_cta_kernel<kModeFused, true><<<std::min<unsigned>(p.slots, p.global_grid), 512, 0, stream>>>(p);
        else
            bt256::sampler_cta_kernel<kModeFused, true><<<std::min<unsigned>(p.slots, p.global_grid), 256, 0, stream>>>(p);
        ADSB_CUDA(cudaGetLastError());
        return;
    }
    if (p.block_threads == 128) bt128::sampler_cta_kernel<kModeFused, false><<<p.blocks, 128, dyn, stream>>>(p);
    else if (p.vec4) bt256::sampler_cta_kernel<kModeFused, false, true><<<p.blocks, 256, dyn, stream>>>(p);
    else bt256::sampler_cta_kernel<kModeFused, false><<<p.blocks, 256, dyn, stream>>>(p);
    ADSB_CUDA(cudaGetLastError());
}

void sampler_phase_report() {
#ifdef ADSB_PHASE_TIMING
    unsigned long long h[16];
    cudaMemcpyFromSymbol(h, adsb_phase, sizeof(h));
    const double samples = h[7] ? static_cast<double>(h[7]) : 1.0;
    std::fprintf(stderr,
                 "[adsb] phase cycles per sample (thread 0): bfs %.0f rebuild %.0f backtrack %.0f clear %.0f | "
                 "kernel per block %.3g, samples %llu, levels/sample %.2f, edge passes/sample %.2f\n",
                 h[0] / samples, h[1] / samples, h[2] / samples, h[3] / samples, static_cast<double>(h[4]),
                 h[7], h[5] / samples, h[6] / samples);
    std::fprintf(stderr, "[adsb]   sample cycles (thread 0): fallback samples %.3g total, others %.3g total\n",
                 static_cast<double>(h[14]), static_cast<double>(h[15]));
    std::fprintf(stderr,
                 "[adsb]   for_edges per chunk: prep %.0f, edge loop (thread 0) %.0f, end barrier wait %.0f | "
                 "edges/chunk %.1f, chunks/sample %.2f, level degree passes %.0f per sample\n",
                 h[13] ? h[8] / static_cast<double>(h[13]) : 0.0, h[13] ? h[9] / static_cast<double>(h[13]) : 0.0,
                 h[13] ? h[11] / static_cast<double>(h[13]) : 0.0, h[13] ? h[12] / static_cast<double>(h[13]) : 0.0,
                 h[13] / samples, h[10] / samples);
    unsigned long long z[16] = {};
    cudaMemcpyToSymbol(adsb_phase, z, sizeof(z));
#endif
}

}  // namespace adsb
