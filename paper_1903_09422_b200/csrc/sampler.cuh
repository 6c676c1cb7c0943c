// sampler.cuh — launch interface of the K1/K2 sampler kernels (sampler.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "rule.cuh"

namespace adsb {

// Per-vertex state word layout (one u64 "meta" + one u64 sigma per vertex and slot):
//   bits 63..32  tag   (per-slot sample generation; stale tags mean "unvisited")
//   bit  31      side  (0: reached from s, 1: reached from t)
//   bit  30      dag   (t-side vertex on a shortest s-t path)
//   bits 29..0   distance from the side's root
constexpr unsigned long long kSideT = 1ull << 31;
constexpr unsigned long long kDag = 1ull << 30;
constexpr unsigned long long kDistMask = (1ull << 30) - 1;

enum SamplerStat {
    kStatEdges = 0,
    kStatVertices = 1,
    kStatSamples = 2,
    kStatErrors = 3,
    kStatRebuildEdges = 4,
    kStatBacktrackEdges = 5,
    kStatFallbacks = 6,
    kStatDegenerate = 7,
    kStatCount = 8
};

// Control words of the fused epoch pipeline (SamplerParams::ctl).
enum FusedCtl {
    kCtlTicket = 0,   // next sample index
    kCtlFolded = 1,   // epochs folded into `total` so far
    kCtlStop = 2,     // epoch at which the run stopped (~0 while running)
    kCtlLock = 3,     // fold lock
    kCtlMax = 4,      // running max of `total`
    kCtlCapped = 5,   // 1 when stopped by max_cycles rather than by the rule
    kCtlDone = 8,     // kCtlDone + k: samples finished in ring slot k
    kCtlWords = 8 + 64
};

struct SamplerParams {
    // graph (device CSR, u32 offsets) and component labels
    const uint32_t* off;
    const uint32_t* nbrs;
    const uint32_t* label;
    uint32_t n;
    uint32_t slot_stride;  // per-slot vertex capacity of the (shared) arena, >= n
    uint32_t slots;
    uint32_t level_cap;
    uint32_t rank;         // this GPU's rank: items map to positions first + item*world + rank
    uint32_t world;
    uint32_t hash_cap;     // block sampler: shared-memory hash capacity (power of two)
    uint32_t use_smem;     // block sampler: try the shared-memory store first
    uint32_t block_threads; // block sampler: 128 or 256
    uint32_t global_grid;   // block sampler: resident blocks of the global-store-only variant
    uint32_t global_threads; // block sampler: threads per block of the global-store-only variant (256 or 512)
    uint32_t max_degree;    // graph max degree (low-degree graphs use thread-per-vertex expansion)
    uint32_t clear_layout;  // block teams: global state in the cleared layout (else tagged)
    float csr_hint;         // block teams: fraction of CSR reads marked L2 evict_last (1 when the CSR fits L2/2)
    uint32_t vec4;          // block teams, shared-memory store: 16-byte adjacency vectors (CSR larger than L2)
    uint32_t hub_factor;    // probe passes: search a frontier row of degree > (hub_factor/4) |L| log2(deg) (0 = never)
    // work: items [0, num_items) map to stream positions first + item*world + rank
    uint64_t seed;
    uint64_t spf;          // samples per item (deterministic frames); 1 in epoch mode
    uint64_t first;
    uint64_t num_items;
    unsigned long long* ticket;
    // slot scratch
    unsigned long long* state;  // slots * n * 2
    uint32_t* queue;            // slots * n
    uint2* qrange;              // slots * n
    uint32_t* tlev;             // slots * level_cap
    uint32_t* dagq;             // block teams: slots * n t-side DAG lists (low-degree push rebuild)
    uint32_t* slot_tag;         // slots
    uint32_t* slot_busy;        // block teams: region bitmap (fallback samples borrow a region)
    uint32_t blocks;            // block teams: shared-memory kernel grid
    // hub search trees (hub_index.cuh), used by the vector kernels; nullptr: plain binary searches
    const uint32_t* hub_ref;
    const uint32_t* hub_keys;
    // deterministic output: (v << 32) | frame-in-batch
    unsigned long long* events;
    unsigned long long* ev_cursor;
    uint64_t ev_cap;
    // epoch output: per-vertex counts of this epoch
    uint32_t* counts;
    unsigned long long* stats;  // kStatCount
    // fused epoch mode (one GPU): the kernel folds finished epochs in order and
    // evaluates the stopping rule itself
    unsigned long long* ctl;    // kCtlWords
    uint32_t* ring_cnt;         // ring_k * n per-epoch counts
    uint32_t* ring_list;        // ring_k * n distinct vertices touched per epoch
    uint32_t* ring_len;         // ring_k
    uint32_t* total;            // n running counts
    uint64_t epoch_b;
    uint64_t max_epochs;
    uint32_t ring_k;
    uint32_t* audit;  // fused diagnostics (ADSB_FUSED_AUDIT): [epoch] recorded, [max_epochs + epoch] folded
    RuleParams rule;
};

// Warp-team sampler (sampler.cu): slots = resident warps.
int sampler_warps_per_sm(bool deterministic);
void launch_sampler_warp(bool deterministic, const SamplerParams& p, cudaStream_t stream);
// Block-team sampler with shared-memory state (sampler_cta.cu): slots = blocks.
size_t sampler_cta_smem_bytes(uint32_t hash_cap, bool vec4);
int sampler_cta_blocks_per_sm(uint32_t hash_cap, uint32_t block_threads, bool vec4);
void launch_sampler_cta(bool deterministic, const SamplerParams& p, cudaStream_t stream);
int sampler_global_blocks_per_sm();
// single-launch epoch pipeline with device-side folding and stopping (block teams)
void launch_sampler_fused(const SamplerParams& p, cudaStream_t stream);
// diagnostic builds (-DADSB_PHASE_TIMING): print and reset per-phase cycle sums
void sampler_phase_report();

enum class SamplerKind { kWarp, kBlock };
SamplerKind sampler_kind();  // ADSB_SAMPLER=warp|block (default block)
void launch_sampler(SamplerKind kind, bool deterministic, const SamplerParams& p, cudaStream_t stream);

}  // namespace adsb
