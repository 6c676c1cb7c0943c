// engine.cu — estimate_bc on the device (kadabra.hpp:308-348) with two
// pipelines (paths relative to /root/reference/proj/include/adsamp/):
//
// Deterministic (indexed-frame, engine.hpp:490-643). Frame p holds spf
// samples from stream_rng(seed, p). A batch of frames is sampled at once
// (K1); every interior vertex becomes an event (v << 32 | frame). K4, the
// ordered cutoff, sorts the events by (v, frame), turns each into "count of v
// after this frame", takes per-frame maxima and a running max over frames,
// and evaluates the stopping rule after EVERY frame in position order; the
// first passing frame P stops the run and only frames <= P are folded. With
// uniform deltas kadabra_converged (kadabra.hpp:133-144) holds iff f and g
// pass at the maximum count, because both are monotone in b under IEEE
// round-to-nearest; the device evaluates them with explicit _rn intrinsics in
// the reference's expression order (no FMA contraction). Result: tau, data,
// check_cycles bit-identical to run_indexed at any thread/GPU count.
//
// Epoch (non-det variants, cumulative semantics as run_barrier,
// engine.hpp:267-341). Sample i draws from stream_rng(seed, i); epoch e holds
// samples [eB, (e+1)B). The sampler (K2) for epoch e+1 runs on stream 1 into
// count[(e+1)&1] while K3 folds count[e&1] into the running total, zeroes it
// and checks the rule on stream 2 (after an NCCL all-reduce when several GPUs
// share the epoch). The run stops at the first epoch whose cumulative state
// passes (the reference's run_epoch checks one epoch only, a defect we do not
// reproduce).
#include <cub/cub.cuh>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "comm.hpp"
#include "engine.hpp"
#include "rule.cuh"
#include "sampler.cuh"

namespace adsb {

// ---------------------------------------------------------------------------
// Scalar rules (host)
// ---------------------------------------------------------------------------
uint64_t compute_omega(uint64_t diameter_bound, double eps, double delta, double c) {
    if (!(eps > 0.0 && eps < 1.0)) invalid("epsilon must lie in (0,1)");
    if (!(delta > 0.0 && delta < 1.0)) invalid("delta must lie in (0,1)");
    const uint64_t vd = diameter_bound + 1;
    const uint64_t arg = vd > 4 ? vd - 2 : 2;
    const double log2_floor = static_cast<double>(63 - __builtin_clzll(arg));
    const double value = (c / (eps * eps)) * (log2_floor + 1.0 + std::log(1.0 / delta));
    return static_cast<uint64_t>(std::ceil(value));
}

double f_kernel(double b, double log_inv, double omega, double tau) {
    const double t = 1.0 / 3.0 - omega / tau;
    return (log_inv / tau) * (t + std::sqrt(t * t + 2.0 * b * omega / log_inv));
}

double g_kernel(double b, double log_inv, double omega, double tau) {
    const double t = 1.0 / 3.0 + omega / tau;
    return (log_inv / tau) * (t + std::sqrt(t * t + 2.0 * b * omega / log_inv));
}

bool converged_at_max(uint64_t max_count, uint64_t tau, uint64_t omega, double eps, double log_inv) {
    const double b = static_cast<double>(max_count) / static_cast<double>(tau);
    if (f_kernel(b, log_inv, static_cast<double>(omega), static_cast<double>(tau)) > eps) return false;
    if (g_kernel(b, log_inv, static_cast<double>(omega), static_cast<double>(tau)) > eps) return false;
    return true;
}

namespace {

constexpr uint32_t kNoStop = 0xFFFFFFFFu;
// the shared-memory table stores vertex + 1 in 24 bits (sampler_cta_body.cuh SmemStore)
constexpr uint32_t kSmemMaxN = (1u << 24) - 1;
// word offsets into DeviceContext::pinned (words 0..15 belong to the BFS level counts)
constexpr int kPinUsed = 48, kPinStop = 49, kPinEmax = 50, kPinMax = 51, kPinFlags = 52, kPinStat0 = 56, kPinStats = 64,
              kPinAdapt = 72, kPinCtl = 80, kPinCursor = 96;  // kPinCtl: 9 words; kPinCursor: 2 words
static_assert(kStatCount <= 8, "pinned staging layout");

// K4a: value of each sorted event = count of v after its frame; per-frame max
__global__ void k_event_values(const unsigned long long* __restrict__ sorted, uint64_t count,
                               const uint32_t* __restrict__ total, uint32_t* frame_max) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long key = sorted[i];
        if (key == ~0ull) continue;
        const unsigned long long target = key & 0xFFFFFFFF00000000ull;
        uint64_t lo = 0, hi = i;  // first index of this vertex's run
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (sorted[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        const uint32_t v = static_cast<uint32_t>(key >> 32);
        const uint32_t value = total[v] + static_cast<uint32_t>(i - lo) + 1u;
        atomicMax(frame_max + static_cast<uint32_t>(key), value);
    }
}

// K4b: first frame of the batch at which the rule holds (or the cap frame)
// (frames_before is a multiple of C; the rule is evaluated after every C-th frame)
__global__ void k_find_stop(const uint32_t* __restrict__ run_max, uint32_t frames,
                            const uint32_t* base_max, uint64_t frames_before, uint64_t spf, uint64_t C,
                            RuleParams r, uint32_t* stop) {
    const uint32_t bm = *base_max;
    for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < frames; f += gridDim.x * blockDim.x) {
        if ((f + 1) % C != 0) continue;
        const uint64_t tau = (frames_before + f + 1) * spf;
        if (rule_passes(max(run_max[f], bm), tau, r)) atomicMin(stop, f);
    }
}

// K4c: fold the events of frames <= limit into the running counts
__global__ void k_apply(const unsigned long long* __restrict__ events, uint64_t count, uint32_t limit,
                        uint32_t* total) {
    for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
        const unsigned long long key = events[i];
        if (key == ~0ull) continue;
        if (static_cast<uint32_t>(key) <= limit) atomicAdd(total + (key >> 32), 1u);
    }
}

__global__ void k_update_base(const uint32_t* run_max, uint32_t limit, uint32_t* base_max) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *base_max = max(*base_max, run_max[limit]);
}

struct MaxOp {
    __device__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

// K3: total += epoch; epoch = 0; max over vertices
__global__ void k_fold_epoch(uint32_t* __restrict__ total, uint32_t* __restrict__ epoch, uint32_t n,
                             uint32_t* max_out) {
    uint32_t local = 0;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
        const uint32_t t = total[v] + epoch[v];
        total[v] = t;
        epoch[v] = 0;
        local = max(local, t);
    }
    using BlockReduce = cub::BlockReduce<uint32_t, 256>;
    __shared__ typename BlockReduce::TempStorage tmp;
    const uint32_t bmax = BlockReduce(tmp).Reduce(local, MaxOp());
    if (threadIdx.x == 0) atomicMax(max_out, bmax);
}

__global__ void k_epoch_rule(uint32_t* max_in, uint64_t tau, RuleParams r, uint32_t* flag) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        *flag = rule_passes(*max_in, tau, r) ? 1u : 0u;
        *max_in = 0;
    }
}

unsigned grid_for(uint64_t work, int device) {
    const uint64_t want = (work + 255) / 256;
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>(want, num_sms(device) * 8ull)));
}

struct Timer {
    std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
    double seconds() const {
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
};

SamplerArena& arena(DeviceContext& ctx) { return *ctx.rt->arena[ctx.rt->active]; }

// Pick the team kind for this graph and make sure the device's arena of that
// kind covers it (vertex capacity and t-level capacity). Arenas are shared by
// all graphs on the device; per-slot generation tags live with the arena, so
// state left by an earlier graph always reads as "unvisited".
void ensure_arena(DeviceContext& ctx, uint32_t level_cap) {
    const uint32_t n = ctx.graph.n;
    // Warp teams win when samples are tiny (C1: ~600 adjacency entries per
    // sample); block teams with shared-memory state win on the larger
    // small-world graphs (C2/C3). ADSB_SAMPLER overrides.
    SamplerKind kind = n <= (1u << 16) ? SamplerKind::kWarp : SamplerKind::kBlock;
    if (std::getenv("ADSB_SAMPLER")) kind = sampler_kind();
    // 2 944 entries of 14 B (1 472 insertions): the shared memory of the former
    // 2 304 x 18 B table, 4 blocks per SM (profiles/r01_hash_cap_sweep.txt)
    uint32_t hash_cap = 2944;
    if (const char* e = std::getenv("ADSB_HASH_CAP")) hash_cap = static_cast<uint32_t>(std::strtoul(e, nullptr, 10));
    uint32_t block_threads = 256;
    if (const char* e = std::getenv("ADSB_BLOCK")) block_threads = std::strtoul(e, nullptr, 10) == 128 ? 128 : 256;
    if (hash_cap < 64 || hash_cap % 64) invalid("ADSB_HASH_CAP must be a multiple of 64");
    const int k = kind == SamplerKind::kWarp ? 0 : 1;
    // vectorised adjacency reads where the CSR misses L2 (C5: -2.4%); on an
    // L2-resident CSR the scalar loop is faster (C2 -7%, C3 -10%). The vector
    // kernels use 2 KB more dynamic shared memory (blocks per SM below).
    bool vec4 = false;
    {
        int l2 = 0;
        ADSB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx.device));
        vec4 = k == 1 && 4ull * (ctx.graph.n + 1) + 4ull * ctx.graph.nnz > static_cast<uint64_t>(l2);
        if (const char* e = std::getenv("ADSB_VEC4")) vec4 = k == 1 && std::strtoul(e, nullptr, 10) != 0;
    }
    DeviceRuntime& rt = *ctx.rt;
    rt.active = k;
    std::unique_ptr<SamplerArena>& slot = rt.arena[k];
    // Global-state layout (sampler_cta_body.cuh GlobalStoreT): cleared words
    // for low-degree graphs, generation tags otherwise. Regions hold the other
    // layout's leftovers after a switch, so the state is zeroed then.
    const int layout = k == 1 && ctx.graph.max_degree <= 32 && !std::getenv("ADSB_TAGGED") ? 1 : 0;
    if (slot && slot->n >= n && slot->level_cap >= level_cap && slot->hash_cap == hash_cap &&
        slot->block_threads == block_threads && slot->vec4 == vec4) {
        if (slot->layout != layout) {
            ADSB_CUDA(cudaMemsetAsync(slot->state.ptr, 0, slot->state.bytes(), rt.stream));
            ADSB_CUDA(cudaMemsetAsync(slot->slot_tag.ptr, 0, slot->slot_tag.bytes(), rt.stream));
            ADSB_CUDA(cudaStreamSynchronize(rt.stream));
            slot->layout = layout;
        }
        return;
    }
    const uint32_t cap_n = slot ? std::max(slot->n, n) : n;
    const uint32_t cap_levels = slot ? std::max(slot->level_cap, level_cap) : level_cap;
    slot.reset();
    ADSB_CUDA(cudaSetDevice(ctx.device));
    const int sms = num_sms(ctx.device);
    const int per_sm = kind == SamplerKind::kWarp ? std::max(sampler_warps_per_sm(true), 8)
                                                  : std::max(sampler_cta_blocks_per_sm(hash_cap, block_threads, vec4), 1);
    size_t free_b = 0, total_b = 0;
    ADSB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    // per region: state (16 B/vertex), queue (4), warp teams also ranges (8)
    // (block teams: + 4 for the t-side DAG lists of the low-degree push rebuild)
    const uint64_t per_vertex = kind == SamplerKind::kWarp ? 16 + 4 + 8 : 16 + 4 + 4;
    const uint64_t per_slot = static_cast<uint64_t>(cap_n) * per_vertex + static_cast<uint64_t>(cap_levels) * 4;
    const uint64_t budget = static_cast<uint64_t>(static_cast<double>(free_b) * 0.55);
    const uint64_t resident = static_cast<uint64_t>(sms) * per_sm;
    // regions: enough for every resident block of the global-store-only kernel too
    const uint64_t resident_regions =
        kind == SamplerKind::kWarp ? resident
                                   : std::max<uint64_t>(resident, static_cast<uint64_t>(sms) *
                                                                      std::max(sampler_global_blocks_per_sm(), 1));
    uint64_t slots = std::min<uint64_t>(resident_regions, budget / std::max<uint64_t>(per_slot, 1));
    if (kind == SamplerKind::kWarp) slots = slots / 8 * 8;
    if (slots < (kind == SamplerKind::kWarp ? 8u : 1u))
        fail(ADSB_ERR_CUDA, "not enough device memory for the sampler scratch (" +
                                std::to_string(per_slot >> 20) + " MiB per team)");
    auto a = std::make_unique<SamplerArena>();
    a->kind = k;
    a->hash_cap = hash_cap;
    a->block_threads = block_threads;
    a->vec4 = vec4;
    a->layout = layout;
    a->slots = static_cast<uint32_t>(slots);
    // Block teams launch every resident block for the shared-memory kernels
    // even when fewer global regions fit (huge graphs): a sample that
    // overflows the table borrows a free region for its redo.
    a->blocks = kind == SamplerKind::kWarp ? a->slots : static_cast<uint32_t>(resident);
    a->n = cap_n;
    a->level_cap = cap_levels;
    a->state.alloc(slots * cap_n * 2);
    a->queue.alloc(slots * cap_n);
    if (kind == SamplerKind::kWarp) a->qrange.alloc(slots * cap_n);
    else a->dagq.alloc(slots * cap_n);
    a->tlev.alloc(2 * slots * cap_levels);  // t-level then s-level boundaries per region
    a->slot_tag.alloc(slots);
    a->slot_busy.alloc((slots + 31) / 32);
    ADSB_CUDA(cudaMemsetAsync(a->slot_busy.ptr, 0, a->slot_busy.bytes(), rt.stream));
    ADSB_CUDA(cudaMemsetAsync(a->state.ptr, 0, a->state.bytes(), rt.stream));
    ADSB_CUDA(cudaMemsetAsync(a->slot_tag.ptr, 0, a->slot_tag.bytes(), rt.stream));
    ADSB_CUDA(cudaStreamSynchronize(rt.stream));
    slot = std::move(a);
}

SamplerParams base_params(DeviceContext& ctx, uint64_t seed, uint64_t spf) {
    SamplerArena& a = arena(ctx);
    SamplerParams p{};
    p.off = ctx.graph.offsets.ptr;
    p.nbrs = ctx.graph.nbrs.ptr;
    p.label = ctx.labels.ptr;
    p.n = ctx.graph.n;
    p.slot_stride = a.n;
    p.max_degree = std::getenv("ADSB_NO_LOWDEG") ? 0xFFFFFFFFu : ctx.graph.max_degree;
    p.slots = a.slots;
    p.level_cap = a.level_cap;
    p.rank = 0;
    p.world = 1;
    p.seed = seed;
    p.spf = spf;
    p.state = a.state.ptr;
    p.queue = a.queue.ptr;
    p.qrange = a.qrange.ptr;
    p.tlev = a.tlev.ptr;
    p.clear_layout = static_cast<uint32_t>(a.layout);
    {
        int l2 = 0;
        ADSB_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, ctx.device));
        const uint64_t csr = 4ull * (ctx.graph.n + 1) + 4ull * ctx.graph.nnz;
        p.csr_hint = csr * 2 <= static_cast<uint64_t>(l2) ? 1.0f : 0.0f;
        if (const char* e = std::getenv("ADSB_CSR_HINT")) p.csr_hint = std::strtof(e, nullptr);
        p.vec4 = a.vec4 ? 1u : 0u;  // chosen with the arena (ensure_arena)
        // hub probes when deg > (hub_factor / 4) |L| cost(deg), cost = dependent loads of one
        // search: 1.0 beat 0.5-4 with plain binary searches (C5 -1%, C2 -5% vs 4.0); with
        // search trees (cost ~ log2(deg) / 3 + 1) 3.0 beat 1-2 and equals 4 (profiles/r02_ab_hub_trees.txt)
        p.hub_factor = a.vec4 && !std::getenv("ADSB_NO_HUB_TREES") ? 12 : 4;
        if (const char* e = std::getenv("ADSB_HUB_FACTOR")) p.hub_factor = std::strtoul(e, nullptr, 10);
    }
    p.dagq = a.dagq.ptr;
    p.slot_tag = a.slot_tag.ptr;
    p.slot_busy = a.slot_busy.ptr;
    p.blocks = a.blocks;
    p.hash_cap = a.hash_cap;
    // Hub search trees where the CSR misses L2 (the vector kernels, chosen by
    // the same test): a search's dependent loads are HBM round trips there. On
    // an L2-resident CSR the plain binary search is as fast (C2 +4% with trees).
    if (a.kind == 1 && a.vec4 && !std::getenv("ADSB_NO_HUB_TREES")) {
        device_hub_index(ctx);  // once per handle
        if (ctx.graph.hub_keys.ptr) {
            p.hub_ref = ctx.graph.hub_ref.ptr;
            p.hub_keys = ctx.graph.hub_keys.ptr;
        }
    }
    p.use_smem = ctx.use_smem == 1 ? 1u : 0u;
    p.global_grid = static_cast<uint32_t>(num_sms(ctx.device) * std::max(sampler_global_blocks_per_sm(), 1));
    // Low-degree graphs (cleared layout): fewer, wider teams. Half the samples
    // in flight for the same threads keeps more of each sample's frontier
    // state in L2: 2 blocks of 512 per SM beat 3 of 256 (C4 -19%), which beat
    // 4 of 256 (-4%); profiles/r01_ab_round3.txt.
    p.global_threads = 256;
    if (a.layout == 1) {
        p.global_threads = 512;
        p.global_grid = static_cast<uint32_t>(num_sms(ctx.device) * 2);
    }
    if (const char* e = std::getenv("ADSB_GLOBAL_BT")) {
        const unsigned long bt = std::strtoul(e, nullptr, 10);
        p.global_threads = bt == 1024 ? 1024 : bt == 512 ? 512 : 256;
    }
    if (const char* e = std::getenv("ADSB_GLOBAL_GRID")) p.global_grid = static_cast<uint32_t>(std::strtoul(e, nullptr, 10));
    p.block_threads = a.block_threads;
    return p;
}

struct Launches {
    uint64_t count = 0;
};

// Stop trying the shared-memory table for this graph when most samples
// overflow it (their balls are too large); results do not depend on the store.
void adapt_store(DeviceContext& ctx, const unsigned long long* stats, cudaStream_t s) {
    SamplerArena& a = arena(ctx);
    if (a.kind == 0 || ctx.use_smem != 1) return;
    unsigned long long* h = ctx.rt->pinned.ptr + kPinAdapt;
    ADSB_CUDA(cudaMemcpyAsync(h, stats, kStatCount * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s));
    ADSB_CUDA(cudaStreamSynchronize(s));
    if (h[kStatSamples] >= 256 && h[kStatFallbacks] * 2 > h[kStatSamples]) ctx.use_smem = 0;
}

// One deterministic batch through the sampler; grows the event buffer until it fits.
uint64_t run_det_batch(DeviceContext& ctx, SamplerParams p, unsigned long long*& events, unsigned long long* scal,
                       Launches& L, cudaEvent_t e0, cudaEvent_t e1, double& sampler_ms) {
    unsigned long long* used_h = ctx.rt->pinned.ptr + kPinUsed;
    for (;;) {
        ADSB_CUDA(cudaMemsetAsync(scal, 0, 2 * sizeof(unsigned long long), ctx.rt->stream));
        p.ticket = scal;
        p.ev_cursor = scal + 1;
        p.events = events;
        p.ev_cap = ctx.rt->pool.capacity<unsigned long long>(Scratch::kEvents);
        ADSB_CUDA(cudaEventRecord(e0, ctx.rt->stream));
        launch_sampler(static_cast<SamplerKind>(arena(ctx).kind == 0 ? 0 : 1), true, p, ctx.rt->stream);
        ADSB_CUDA(cudaEventRecord(e1, ctx.rt->stream));
        L.count++;
        ADSB_CUDA(cudaMemcpyAsync(used_h, scal + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, ctx.rt->stream));
        ADSB_CUDA(cudaStreamSynchronize(ctx.rt->stream));
        float ms = 0;
        ADSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        sampler_ms += ms;
        const unsigned long long used = *used_h;
        if (used <= p.ev_cap) return used;
        events = ctx.rt->pool.get<unsigned long long>(Scratch::kEvents, used + used / 4 + 1024);  // rerun the batch
    }
}

// Frames still needed before the rule can pass, predicting that the largest
// count keeps growing in proportion to tau (b = max_count / tau stays fixed):
// the smallest tau with f(b) <= eps and g(b) <= eps (both decrease in tau at
// fixed b), found by bisection with the host formulas. Used only to size
// batches; the stop itself is decided exactly by the ordered cutoff.
uint64_t predict_stop_tau(uint64_t max_count, uint64_t tau, uint64_t omega, double eps, double log_inv) {
    if (tau == 0) return omega;
    const double b = static_cast<double>(max_count) / static_cast<double>(tau);
    auto pass = [&](uint64_t t) {
        if (t >= omega) return true;
        const double td = static_cast<double>(t);
        return f_kernel(b, log_inv, static_cast<double>(omega), td) <= eps &&
               g_kernel(b, log_inv, static_cast<double>(omega), td) <= eps;
    };
    uint64_t lo = tau, hi = omega;
    if (pass(lo)) return lo;
    while (lo + 1 < hi) {
        const uint64_t mid = lo + (hi - lo) / 2;
        if (pass(mid)) hi = mid;
        else lo = mid;
    }
    return hi;
}

bool trace_enabled() {
    static const bool on = std::getenv("ADSB_TRACE") != nullptr;
    return on;
}

bool rule_passes_host(uint64_t max_count, uint64_t tau, const RuleParams& r) {
    return tau >= r.omega || converged_at_max(max_count, tau, r.omega, r.eps, r.log_inv);
}

// ADSB_AUDIT=<file>: a validate_consistency-style log (audit.hpp:101-161
// analogue, diagnostics only) of the host-orchestrated pipelines, replayed by
// tests/test_gpu_parity.py: per frame batch its first frame, size, the
// running max after every frame (the check record) and every increment
// event; per barrier round the all-reduced round counts and the check.
// u64 records:  [1, first, F, events, limit, stopped, base_max] run_max[F] events[events]
//               [2, epoch, B, pass, max] counts[n]
//               [3, tau, check_cycles]
struct AuditLog {
    FILE* f = nullptr;
    AuditLog() {
        if (const char* path = std::getenv("ADSB_AUDIT")) f = std::fopen(path, "wb");
    }
    ~AuditLog() {
        if (f) std::fclose(f);
    }
    explicit operator bool() const { return f != nullptr; }
    void words(std::initializer_list<uint64_t> w) {
        for (uint64_t x : w) std::fwrite(&x, 8, 1, f);
    }
    template <class T>
    void device_array(const T* dev, uint64_t count, cudaStream_t s) {
        std::vector<T> h(count);
        if (count) ADSB_CUDA(cudaMemcpyAsync(h.data(), dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
        ADSB_CUDA(cudaStreamSynchronize(s));
        for (T x : h) {
            const uint64_t w = static_cast<uint64_t>(x);
            std::fwrite(&w, 8, 1, f);
        }
    }
};

}  // namespace

EngineOutput estimate_bc(DeviceContext& ctx, double eps, double delta, const EngineOptions& opt) {
    EngineOutput out;
    const uint32_t n = ctx.graph.n;
    if (n == 0) invalid("graph has no vertices");
    if (!(delta > 0.0 && delta < 1.0)) invalid("delta must lie in (0,1)");
    if (!(eps > 0.0 && eps < 1.0)) invalid("epsilon must lie in (0,1)");
    ADSB_CUDA(cudaSetDevice(ctx.device));
    if (n == 1) {  // kadabra.hpp:314-317
        return out;  // counts == nullptr: the single vertex scores 0
    }
    const int world = opt.comm ? opt.comm->nranks : 1;
    const int rank = opt.comm ? opt.comm->rank : 0;
    out.world = static_cast<uint32_t>(world);

    // ---- preprocessing (kadabra.hpp:319-325): components, D_ub, omega, deltas
    Timer pre;
    // components and D_ub depend only on the (immutable) graph: computed on the
    // first call for this handle and reused (the reference recomputes them per
    // call inside preprocess_seconds, kadabra.hpp:319-325)
    out.num_components = device_components(ctx);
    const double t_cc = pre.seconds();
    out.diameter_bound = device_diameter_bound(ctx);
    const double t_dub = pre.seconds();
    out.omega = compute_omega(out.diameter_bound, eps, delta, opt.c);
    // Device counts are u32 (every count is <= tau <= omega): refuse runs whose
    // omega does not fit rather than wrap (the reference's data[] is u64,
    // frame.hpp:118; omega >= 2^32 needs eps below ~5e-5)
    if (out.omega > 0xFFFFFFFFull)
        invalid("omega = " + std::to_string(out.omega) + " exceeds 2^32-1 (u32 device counts); raise epsilon");
    const double delta_v = delta / (2.0 * static_cast<double>(n));  // kadabra.hpp:34
    const double log_inv = std::log(1.0 / delta_v);                 // kadabra.hpp:123
    const uint32_t level_cap = static_cast<uint32_t>(std::min<uint64_t>(out.diameter_bound + 3, n + 2));
    ensure_arena(ctx, level_cap);
    if (ctx.use_smem < 0) {
        // Deep graphs (grid: D_ub 8182) need far more t-levels than the table
        // tracks and far larger balls than it holds: go global-only at once.
        ctx.use_smem = std::getenv("ADSB_NO_SMEM") || out.diameter_bound > 128 || n >= kSmemMaxN ? 0 : 1;
    }
    out.preprocess_seconds = pre.seconds();
    if (trace_enabled())
        std::fprintf(stderr, "[adsb] preprocess: components %.3f ms, D_ub %.3f ms, arena %.3f ms (kind %d, slots %u)\n",
                     1e3 * t_cc, 1e3 * (t_dub - t_cc), 1e3 * (out.preprocess_seconds - t_dub), arena(ctx).kind,
                     arena(ctx).kind == 0 ? arena(ctx).slots : arena(ctx).blocks);

    Timer ads;
    const RuleParams rule{out.omega, static_cast<double>(out.omega), log_inv, eps};
    cudaStream_t s1 = ctx.rt->stream, s2 = ctx.rt->stream2;
    uint32_t* total = ctx.rt->pool.get<uint32_t>(Scratch::kTotal, n);
    unsigned long long* stats = ctx.rt->pool.get<unsigned long long>(Scratch::kStats, kStatCount);
    unsigned long long* scal = ctx.rt->pool.get<unsigned long long>(Scratch::kScal, 4);
    ADSB_CUDA(cudaMemsetAsync(total, 0, static_cast<size_t>(n) * sizeof(uint32_t), s1));
    ADSB_CUDA(cudaMemsetAsync(stats, 0, kStatCount * sizeof(unsigned long long), s1));
    if (!ctx.rt->ev_a) {
        ADSB_CUDA(cudaEventCreate(&ctx.rt->ev_a));
        ADSB_CUDA(cudaEventCreate(&ctx.rt->ev_b));
    }
    cudaEvent_t e0 = ctx.rt->ev_a, e1 = ctx.rt->ev_b;
    Launches L;
    const uint32_t* max_dev32 = nullptr;  // device copy of max_v counts[v] when a branch keeps one
    bool max_known = false;
    uint64_t max_host = 0;
    // work units that keep every team busy: warps are many and light, blocks few
    // and heavy. Batch and epoch sizes derive from it, and every rank must make
    // the same sizing decisions (they set the collectives' sizes and order), so
    // ranks agree on the smallest.
    uint64_t team_slots = arena(ctx).kind == 0 ? arena(ctx).slots : 8ull * arena(ctx).blocks;
    if (world > 1) comm_allreduce_host(opt.comm, &team_slots, 1, RedOp::kMin, s1);

    // Pipelines. Deterministic variants: frames of spf samples, the rule after
    // every frame (run_indexed). Non-deterministic variants: cumulative epochs of
    // B samples (sample i from stream_rng(seed, i)), the rule after every epoch:
    //  * one GPU, block teams: one persistent kernel folds epochs in order (fused);
    //  * barrier on several GPUs: run_barrier's rounds, each split across the
    //    ranks and combined by an all-reduce of the n-length count vector;
    //  * otherwise (several GPUs, or warp teams): the frame pipeline with spf = 1
    //    and the rule evaluated at epoch ends only — the ranks' per-sample
    //    increments are all-gathered and folded in index order, so tau and the
    //    counts do not depend on the GPU count.
    // All non-det paths give identical results for the same B.
    const uint64_t epoch_B = opt.epoch_samples ? opt.epoch_samples : (opt.barrier ? opt.check_interval : 1024);
    const bool fused_mode = !opt.deterministic && world == 1 && arena(ctx).kind == 1 && !std::getenv("ADSB_NO_FUSED");
    const bool dense_mode = !opt.deterministic && !fused_mode && (opt.barrier || std::getenv("ADSB_DENSE_EPOCHS")) &&
                            (world > 1 || std::getenv("ADSB_DENSE_EPOCHS"));
    const bool frames_mode = opt.deterministic || (!fused_mode && !dense_mode);
    // queue statistics (engine.hpp:156-161): frames sampled ahead of the in-order
    // consumption point, per sampler team
    const uint64_t teams = std::max<uint64_t>(arena(ctx).kind == 0 ? team_slots : team_slots / 8, 1) * world;
    const double teams_total = static_cast<double>(teams);
    uint64_t depth_obs = 0;
    double depth_sum = 0;
    auto observe_depth = [&](uint64_t frames_ahead) {
        const uint64_t d = static_cast<uint64_t>(std::ceil(static_cast<double>(frames_ahead) / teams_total));
        out.queue_max_depth = std::max(out.queue_max_depth, d);
        depth_sum += static_cast<double>(d);
        ++depth_obs;
        out.queue_allocated = std::max(out.queue_allocated, frames_ahead);
    };

    if (frames_mode) {
        // C = frames per check: 1 (run_indexed), or B single-sample frames (epochs)
        const uint64_t spf = opt.deterministic ? opt.spf : 1;
        const uint64_t C = opt.deterministic ? 1 : epoch_B;
        uint64_t frame_limit = (out.omega + spf - 1) / spf;  // the rule holds by tau >= omega
        frame_limit = (frame_limit + C - 1) / C * C;           // epochs end on a multiple of B
        if (opt.max_cycles) frame_limit = std::min(frame_limit, opt.max_cycles * C);
        frame_limit = std::max<uint64_t>(frame_limit, C);
        // bounded memory (engine.hpp:92, :137-144): at most a+1 frames ahead per team
        const uint64_t bounded_cap =
            opt.bounded_memory ? std::max<uint64_t>(teams * (opt.reservation_block + 1ull), C) : ~0ull;
        uint32_t* base_max = ctx.rt->pool.get<uint32_t>(Scratch::kBaseMax, 1);
        uint32_t* stop_idx = ctx.rt->pool.get<uint32_t>(Scratch::kStopIdx, 1);
        uint32_t* stop_h = reinterpret_cast<uint32_t*>(ctx.rt->pinned.ptr + kPinStop);
        unsigned long long* emax_h = ctx.rt->pinned.ptr + kPinEmax;
        ADSB_CUDA(cudaMemsetAsync(base_max, 0, sizeof(uint32_t), s1));
        unsigned long long* events = ctx.rt->pool.get<unsigned long long>(Scratch::kEvents, 1 << 20);
        AuditLog audit;
        uint64_t done = 0;  // frames folded so far
        uint64_t sampled_frames = 0;
        bool stopped = false;
        uint32_t stop_local = kNoStop;
        uint64_t cur_max = 0;  // largest count after the frames folded so far
        uint64_t growth = 3;   // batch cap: growth x the frames done (ADSB_DET_GROWTH; 3 beat 2 and 4 on C1/C3/C4)
        if (const char* g = std::getenv("ADSB_DET_GROWTH")) growth = std::max<uint64_t>(2, std::strtoull(g, nullptr, 10));
        while (!stopped) {
            // Batch size: the predicted remaining frames (+5%), at least a few
            // frames per team; the first batch has no prediction yet.
            uint64_t F = 2 * team_slots * world;
            if (done > 0) {
                const uint64_t tau_star = predict_stop_tau(cur_max, done * spf, out.omega, eps, log_inv);
                const uint64_t need = (tau_star > done * spf ? (tau_star - done * spf + spf - 1) / spf : 1);
                // at most `growth` x the frames done so far: early max counts are
                // biased high, so the prediction overshoots then
                F = std::min<uint64_t>(std::max<uint64_t>(need + need / 20 + 1, team_slots * world / 2),
                                       std::max<uint64_t>((growth - 1) * done, F));
            }
            F = std::min<uint64_t>(F, bounded_cap);
            F = (F + C - 1) / C * C;  // whole epochs
            F = std::min<uint64_t>(F, frame_limit - done);
            F = std::min<uint64_t>(F, (1ull << 30) / C * C);
            observe_depth(F);
            SamplerParams p = base_params(ctx, opt.seed, spf);
            p.first = done;
            p.rank = static_cast<uint32_t>(rank);
            p.world = static_cast<uint32_t>(world);
            p.num_items = (F > static_cast<uint64_t>(rank)) ? (F - rank + world - 1) / world : 0;
            p.stats = stats;
            const uint64_t E = run_det_batch(ctx, p, events, scal, L, e0, e1, out.sampler_ms);
            sampled_frames += F;
            adapt_store(ctx, stats, s1);
            unsigned long long* ev = events;
            uint64_t count = E;
            if (world > 1) {
                // gather every rank's events so each rank runs the identical cutoff
                uint64_t emax = E;
                comm_allreduce_host(opt.comm, &emax, 1, RedOp::kMax, s1);
                if (ctx.rt->pool.capacity<unsigned long long>(Scratch::kEvents) < emax) {
                    unsigned long long* tmp = ctx.rt->pool.get<unsigned long long>(Scratch::kSorted, E);
                    ADSB_CUDA(cudaMemcpyAsync(tmp, events, E * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s1));
                    events = ctx.rt->pool.get<unsigned long long>(Scratch::kEvents, emax);
                    ADSB_CUDA(cudaMemcpyAsync(events, tmp, E * sizeof(unsigned long long), cudaMemcpyDeviceToDevice, s1));
                }
                if (emax > E)  // padding: all-ones keys sort last and are skipped
                    ADSB_CUDA(cudaMemsetAsync(events + E, 0xFF, (emax - E) * sizeof(unsigned long long), s1));
                unsigned long long* gathered = ctx.rt->pool.get<unsigned long long>(Scratch::kGathered, emax * world);
                comm_allgather_u64(opt.comm, events, gathered, emax, s1);
                ev = gathered;
                count = emax * world;
            }
            // K4: ordered cutoff over the batch
            unsigned long long* sorted = ctx.rt->pool.get<unsigned long long>(Scratch::kSorted, count);
            uint32_t* frame_max = ctx.rt->pool.get<uint32_t>(Scratch::kFrameMax, F);
            uint32_t* run_max = ctx.rt->pool.get<uint32_t>(Scratch::kRunMax, F);
            int end_bit = 64;
            if (world == 1) {
                int vbits = 1;
                while (vbits < 32 && (1ull << vbits) < n) ++vbits;
                end_bit = 32 + vbits;
            }
            size_t tb = 0, tb2 = 0;
            ADSB_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, ev, sorted, count, 0, end_bit, s1));
            ADSB_CUDA(cub::DeviceScan::InclusiveScan(nullptr, tb2, frame_max, run_max, MaxOp(),
                                                     static_cast<int64_t>(F), s1));
            tb = std::max(tb, tb2);
            uint8_t* temp = ctx.rt->pool.get<uint8_t>(Scratch::kSortTemp, tb);
            ADSB_CUDA(cub::DeviceRadixSort::SortKeys(temp, tb, ev, sorted, count, 0, end_bit, s1));
            ADSB_CUDA(cudaMemsetAsync(frame_max, 0, F * sizeof(uint32_t), s1));
            k_event_values<<<grid_for(count, ctx.device), 256, 0, s1>>>(sorted, count, total, frame_max);
            ADSB_CUDA(cub::DeviceScan::InclusiveScan(temp, tb, frame_max, run_max, MaxOp(), static_cast<int64_t>(F), s1));
            ADSB_CUDA(cudaMemsetAsync(stop_idx, 0xFF, sizeof(uint32_t), s1));
            k_find_stop<<<grid_for(F, ctx.device), 256, 0, s1>>>(run_max, static_cast<uint32_t>(F), base_max, done, spf,
                                                                 C, rule, stop_idx);
            ADSB_CUDA(cudaMemcpyAsync(stop_h, stop_idx, sizeof(uint32_t), cudaMemcpyDeviceToHost, s1));
            ADSB_CUDA(cudaMemcpyAsync(stop_h + 1, run_max + (F - 1), sizeof(uint32_t), cudaMemcpyDeviceToHost, s1));
            ADSB_CUDA(cudaStreamSynchronize(s1));
            L.count += 3;
            const uint32_t stop_host = *stop_h;
            cur_max = std::max<uint64_t>(cur_max, stop_h[1]);
            uint32_t limit = static_cast<uint32_t>(F - 1);
            if (stop_host != kNoStop) {
                limit = stop_host;
                stopped = true;
                stop_local = stop_host;
            } else if (done + F >= frame_limit) {
                stopped = true;  // max_cycles cap
                stop_local = limit;
                out.reason = ADSB_REASON_CAPPED;
            }
            if (audit) {
                uint32_t bm = 0;
                ADSB_CUDA(cudaMemcpyAsync(&bm, base_max, sizeof bm, cudaMemcpyDeviceToHost, s1));
                ADSB_CUDA(cudaStreamSynchronize(s1));
                audit.words({1, done, F, count, limit, stopped ? 1u : 0u, bm});
                audit.device_array(run_max, F, s1);
                audit.device_array(ev, count, s1);
            }
            k_apply<<<grid_for(count, ctx.device), 256, 0, s1>>>(ev, count, limit, total);
            k_update_base<<<1, 32, 0, s1>>>(run_max, limit, base_max);
            L.count += 2;
            if (trace_enabled())
                std::fprintf(stderr, "[adsb] det batch: frames %llu..%llu events %llu stop %d t=%.3f ms\n",
                             static_cast<unsigned long long>(done), static_cast<unsigned long long>(done + F),
                             static_cast<unsigned long long>(count), stop_host == kNoStop ? -1 : static_cast<int>(stop_host),
                             1e3 * ads.seconds());
            if (!stopped) done += F;
            else done += static_cast<uint64_t>(stop_local) + 1;
        }
        max_dev32 = base_max;  // k_update_base folded the running max up to the stop frame
        out.total_samples = sampled_frames * spf;
        out.tau = done * spf;
        if (audit) audit.words({3, done * spf, opt.deterministic ? done : done / C});
        if (opt.deterministic) {
            out.check_cycles = done;
            out.stop_epoch = (done - 1) / std::max<uint32_t>(opt.nominal_threads, 1) + 1;  // engine.hpp:562
        } else {
            out.check_cycles = done / C;
            out.stop_epoch = out.check_cycles;
        }
    } else if (fused_mode) {
        // ---- cumulative epochs, fused: one persistent launch folds finished
        // epochs in order and evaluates the rule on the device (no host round
        // trip per epoch), so epochs can be as small as the reference's check
        // interval and the run stops within ~K epochs + one sample per block.
        const uint64_t B = epoch_B;
        uint64_t max_epochs = (out.omega + B - 1) / B;
        if (opt.max_cycles) max_epochs = std::min(max_epochs, opt.max_cycles);
        max_epochs = std::max<uint64_t>(max_epochs, 1);
        // Ring of K epoch slots: a block may start epoch e only after e - K was
        // folded, and one slow sample holds its epoch's fold. K = 32 keeps
        // the blocks busy through C5's long-tailed samples (K = 8: 23% of
        // warp stall samples waited for a slot; C5 1.30 s -> 0.92 s to stop;
        // profiles/r01_ab_round3.txt). Memory 8 B x K x n.
        uint32_t K = 32;
        if (const char* e = std::getenv("ADSB_RING_K")) K = std::min<uint32_t>(std::max<uint32_t>(std::strtoul(e, nullptr, 10), 2), 64);
        observe_depth(static_cast<uint64_t>(K) * B);
        unsigned long long* ctl = ctx.rt->pool.get<unsigned long long>(Scratch::kCtl, kCtlWords);
        uint32_t* ring_cnt = ctx.rt->pool.get<uint32_t>(Scratch::kRingCnt, static_cast<size_t>(K) * n);
        uint32_t* ring_list = ctx.rt->pool.get<uint32_t>(Scratch::kRingList, static_cast<size_t>(K) * n);
        uint32_t* ring_len = ctx.rt->pool.get<uint32_t>(Scratch::kRingLen, K);
        ADSB_CUDA(cudaMemsetAsync(ctl, 0, kCtlWords * sizeof(unsigned long long), s1));
        ADSB_CUDA(cudaMemsetAsync(ctl + kCtlStop, 0xFF, sizeof(unsigned long long), s1));
        ADSB_CUDA(cudaMemsetAsync(ring_cnt, 0, static_cast<size_t>(K) * n * sizeof(uint32_t), s1));
        ADSB_CUDA(cudaMemsetAsync(ring_len, 0, K * sizeof(uint32_t), s1));
        SamplerParams p = base_params(ctx, opt.seed, 1);
        p.stats = stats;
        p.ctl = ctl;
        p.ring_cnt = ring_cnt;
        p.ring_list = ring_list;
        p.ring_len = ring_len;
        p.total = total;
        p.epoch_b = B;
        p.max_epochs = max_epochs;
        p.ring_k = K;
        p.rule = rule;
        // ADSB_FUSED_AUDIT=<file>: per sample (ticket) the increments it recorded
        // | its distance << 16, then per epoch the increments folds consumed:
        // u32[max_epochs * B + max_epochs] (diagnostics only)
        const char* audit_path = std::getenv("ADSB_FUSED_AUDIT");
        if (audit_path) {
            p.audit = ctx.rt->pool.get<uint32_t>(Scratch::kAudit, (B + 1) * max_epochs);
            ADSB_CUDA(cudaMemsetAsync(p.audit, 0, (B + 1) * max_epochs * sizeof(uint32_t), s1));
        }
        const double t_launch = ads.seconds();
        ADSB_CUDA(cudaEventRecord(e0, s1));
        launch_sampler_fused(p, s1);
        ADSB_CUDA(cudaEventRecord(e1, s1));
        L.count++;
        unsigned long long* ctl_h = ctx.rt->pinned.ptr + kPinCtl;
        ADSB_CUDA(cudaMemcpyAsync(ctl_h, ctl, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s1));
        ADSB_CUDA(cudaStreamSynchronize(s1));
        float ms = 0;
        ADSB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        out.sampler_ms = ms;
        const uint64_t stop = ctl_h[kCtlStop];
        if (stop == ~0ull) fail(ADSB_ERR_LOGIC, "fused epoch pipeline exited without a stop decision");
        if (ctl_h[kCtlCapped]) out.reason = ADSB_REASON_CAPPED;
        out.tau = (stop + 1) * B;
        out.check_cycles = stop + 1;
        out.stop_epoch = stop + 1;
        max_host = ctl_h[kCtlMax];  // running max of the folded epochs (fold_chain)
        max_known = true;
        ADSB_CUDA(cudaMemcpyAsync(ctl_h + 8, stats + kStatSamples, sizeof(unsigned long long), cudaMemcpyDeviceToHost, s1));
        ADSB_CUDA(cudaStreamSynchronize(s1));
        out.total_samples = ctl_h[8];
        if (audit_path) {
            std::vector<uint32_t> a((B + 1) * max_epochs);
            ADSB_CUDA(cudaMemcpy(a.data(), p.audit, a.size() * sizeof(uint32_t), cudaMemcpyDeviceToHost));
            if (FILE* f = std::fopen(audit_path, "wb")) {
                std::fwrite(a.data(), sizeof(uint32_t), a.size(), f);
                std::fclose(f);
            }
        }
        if (trace_enabled())
            std::fprintf(stderr, "[adsb] fused epochs: B %llu stop epoch %llu drawn %llu launch at %.3f ms, t=%.3f ms\n",
                         static_cast<unsigned long long>(B), static_cast<unsigned long long>(stop),
                         static_cast<unsigned long long>(out.total_samples), 1e3 * t_launch, 1e3 * ads.seconds());
    } else {
        // ---- cumulative epochs as run_barrier rounds (engine.hpp:267-341): each
        // round of B samples is split across the ranks; stream 2 all-reduces the
        // round's n-length count vector, folds it and checks the rule while stream
        // 1 samples the next round into the other buffer.
        const uint64_t B = epoch_B;
        observe_depth(2 * B);
        AuditLog audit;
        uint64_t max_epochs = (out.omega + B - 1) / B;
        if (opt.max_cycles) max_epochs = std::min(max_epochs, opt.max_cycles);
        max_epochs = std::max<uint64_t>(max_epochs, 1);
        uint32_t* cnt = ctx.rt->pool.get<uint32_t>(Scratch::kEpochCnt, 2ull * n);
        uint32_t* dmax = ctx.rt->pool.get<uint32_t>(Scratch::kDmax, 2);
        uint32_t* flag_dev = ctx.rt->pool.get<uint32_t>(Scratch::kFlagDev, 2);
        unsigned long long* tickets = ctx.rt->pool.get<unsigned long long>(Scratch::kTickets, 2);
        uint32_t* flag_host = reinterpret_cast<uint32_t*>(ctx.rt->pinned.ptr + kPinFlags);
        unsigned long long* stat0 = ctx.rt->pinned.ptr + kPinStat0;  // kStatCount words
        ADSB_CUDA(cudaMemsetAsync(cnt, 0, 2ull * n * sizeof(uint32_t), s1));
        ADSB_CUDA(cudaMemsetAsync(dmax, 0, 2 * sizeof(uint32_t), s1));
        ADSB_CUDA(cudaStreamSynchronize(s1));
        if (!ctx.rt->ev_samp[0]) {
            for (int i = 0; i < 2; ++i) {
                ADSB_CUDA(cudaEventCreateWithFlags(&ctx.rt->ev_samp[i], cudaEventDisableTiming));
                ADSB_CUDA(cudaEventCreateWithFlags(&ctx.rt->ev_chk[i], cudaEventDisableTiming));
            }
            ADSB_CUDA(cudaEventCreateWithFlags(&ctx.rt->ev_stat, cudaEventDisableTiming));
        }
        cudaEvent_t* samp = ctx.rt->ev_samp;
        cudaEvent_t* chk = ctx.rt->ev_chk;
        const uint64_t share = (B > static_cast<uint64_t>(rank)) ? (B - rank + world - 1) / world : 0;
        uint64_t launched = 0;
        while (ctx.rt->ev_launch.size() < 2 * max_epochs + 2) {
            cudaEvent_t ev;
            ADSB_CUDA(cudaEventCreate(&ev));
            ctx.rt->ev_launch.push_back(ev);
        }
        auto enqueue_sampler = [&](uint64_t e) {
            const int k = static_cast<int>(e & 1);
            if (e >= 2) ADSB_CUDA(cudaStreamWaitEvent(s1, chk[k], 0));
            SamplerParams p = base_params(ctx, opt.seed, 1);
            p.first = e * B;
            p.rank = static_cast<uint32_t>(rank);
            p.world = static_cast<uint32_t>(world);
            p.num_items = share;
            p.ticket = tickets + k;
            p.counts = cnt + static_cast<size_t>(k) * n;
            p.stats = stats;
            ADSB_CUDA(cudaMemsetAsync(tickets + k, 0, sizeof(unsigned long long), s1));
            ADSB_CUDA(cudaEventRecord(ctx.rt->ev_launch[2 * launched], s1));
            launch_sampler(static_cast<SamplerKind>(arena(ctx).kind == 0 ? 0 : 1), false, p, s1);
            ADSB_CUDA(cudaEventRecord(ctx.rt->ev_launch[2 * launched + 1], s1));
            ADSB_CUDA(cudaEventRecord(samp[k], s1));
            L.count++;
            launched++;
        };
        auto enqueue_check = [&](uint64_t e) {
            const int k = static_cast<int>(e & 1);
            ADSB_CUDA(cudaStreamWaitEvent(s2, samp[k], 0));
            uint32_t* ec = cnt + static_cast<size_t>(k) * n;
            comm_allreduce_u32_sum(opt.comm, ec, n, s2);
            std::vector<uint32_t> round_counts;
            if (audit) {
                round_counts.resize(n);
                ADSB_CUDA(cudaMemcpyAsync(round_counts.data(), ec, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s2));
            }
            k_fold_epoch<<<grid_for(n, ctx.device), 256, 0, s2>>>(total, ec, n, dmax + k);
            if (audit) {
                uint32_t mx = 0;
                ADSB_CUDA(cudaMemcpyAsync(&mx, dmax + k, sizeof mx, cudaMemcpyDeviceToHost, s2));
                ADSB_CUDA(cudaStreamSynchronize(s2));
                const bool pass = rule_passes_host(mx, (e + 1) * B, rule);
                audit.words({2, e, B, pass ? 1u : 0u, mx});
                for (uint32_t x : round_counts) audit.words({x});
            }
            k_epoch_rule<<<1, 32, 0, s2>>>(dmax + k, (e + 1) * B, rule, flag_dev + k);
            ADSB_CUDA(cudaMemcpyAsync(flag_host + k, flag_dev + k, sizeof(uint32_t), cudaMemcpyDeviceToHost, s2));
            ADSB_CUDA(cudaEventRecord(chk[k], s2));
            L.count += 2;
        };
        enqueue_sampler(0);
        ADSB_CUDA(cudaMemcpyAsync(stat0, stats, kStatCount * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s1));
        ADSB_CUDA(cudaEventRecord(ctx.rt->ev_stat, s1));
        enqueue_check(0);
        if (max_epochs > 1) enqueue_sampler(1);
        uint64_t e = 0;
        for (;; ++e) {
            const int k = static_cast<int>(e & 1);
            ADSB_CUDA(cudaEventSynchronize(chk[k]));
            const bool pass = flag_host[k] != 0;
            if (e == 0) {
                ADSB_CUDA(cudaEventSynchronize(ctx.rt->ev_stat));
                if (arena(ctx).kind == 1 && ctx.use_smem == 1 && stat0[kStatSamples] >= 256 &&
                    stat0[kStatFallbacks] * 2 > stat0[kStatSamples])
                    ctx.use_smem = 0;
            }
            if (trace_enabled())
                std::fprintf(stderr, "[adsb] epoch %llu checked: pass %d t=%.3f ms\n", static_cast<unsigned long long>(e),
                             pass ? 1 : 0, 1e3 * ads.seconds());
            if (pass || e + 1 >= max_epochs) {
                if (!pass) out.reason = ADSB_REASON_CAPPED;
                break;
            }
            enqueue_check(e + 1);
            if (e + 2 < max_epochs) enqueue_sampler(e + 2);
        }
        ADSB_CUDA(cudaStreamSynchronize(s1));
        ADSB_CUDA(cudaStreamSynchronize(s2));
        for (uint64_t i = 0; i < launched; ++i) {
            float ms = 0;
            ADSB_CUDA(cudaEventElapsedTime(&ms, ctx.rt->ev_launch[2 * i], ctx.rt->ev_launch[2 * i + 1]));
            out.sampler_ms += ms;  // device time of the sampler launches only
        }
        out.tau = (e + 1) * B;
        out.check_cycles = e + 1;
        out.stop_epoch = e + 1;
        out.total_samples = launched * B;
        if (audit) audit.words({3, out.tau, out.check_cycles});
    }

    // ---- results
    if (ctx.rt->host_counts.count < n) ctx.rt->host_counts = PinnedBuf<uint32_t>(n);
    uint32_t* host32 = ctx.rt->host_counts.ptr;
    ADSB_CUDA(cudaMemcpyAsync(host32, total, n * sizeof(uint32_t), cudaMemcpyDeviceToHost, s1));
    unsigned long long* st_host = ctx.rt->pinned.ptr + kPinStats;
    ADSB_CUDA(cudaMemcpyAsync(st_host, stats, kStatCount * sizeof(unsigned long long), cudaMemcpyDeviceToHost, s1));
    uint32_t* max_h32 = reinterpret_cast<uint32_t*>(ctx.rt->pinned.ptr + kPinMax);
    if (max_dev32) ADSB_CUDA(cudaMemcpyAsync(max_h32, max_dev32, sizeof(uint32_t), cudaMemcpyDeviceToHost, s1));
    ADSB_CUDA(cudaStreamSynchronize(s1));
    ADSB_CUDA(cudaGetLastError());
    if (st_host[kStatErrors] != 0)
        fail(ADSB_ERR_LOGIC, "sampler reported " + std::to_string(st_host[kStatErrors]) +
                                 " inconsistent traversals (all predecessor counts wrapped to 0?)");
    out.counts = host32;
    out.edges_scanned = st_host[kStatEdges];
    out.vertices_expanded = st_host[kStatVertices];
    out.rebuild_edges = st_host[kStatRebuildEdges];
    out.backtrack_edges = st_host[kStatBacktrackEdges];
    out.store_fallbacks = st_host[kStatFallbacks];
    out.degenerate_steps = st_host[kStatDegenerate];
    out.kernel_launches = L.count;
    out.queue_mean_depth = depth_obs ? depth_sum / static_cast<double>(depth_obs) : 0.0;
    out.queue_high_water_exceeded = out.queue_max_depth > opt.queue_high_water;
    // kadabra.hpp:339-343
    if (out.reason != ADSB_REASON_CAPPED) {
        out.reason = ADSB_REASON_OMEGA_REACHED;
        uint64_t mx = 0;
        if (max_dev32) mx = *max_h32;
        else if (max_known) mx = max_host;
        else
            for (uint32_t v = 0; v < n; ++v) mx = std::max<uint64_t>(mx, host32[v]);
        if (out.tau >= 1 && converged_at_max(mx, out.tau, out.omega, eps, log_inv))
            out.reason = ADSB_REASON_EPS_CONVERGED;
    }
    out.ads_seconds = ads.seconds();
    if (trace_enabled()) {
        std::fprintf(stderr, "[adsb] results at %.3f ms (pre %.3f ms)\n", 1e3 * out.ads_seconds,
                     1e3 * out.preprocess_seconds);
        sampler_phase_report();
    }
    return out;
}

void sample_frames(DeviceContext& ctx, uint64_t seed, uint64_t spf, uint64_t first, uint64_t count,
                   uint64_t* frame_offsets, uint32_t* incs, uint64_t cap) {
    if (spf < 1) invalid("samples per frame must be >= 1");
    if (count == 0) {
        frame_offsets[0] = 0;
        return;
    }
    if (count >= (1ull << 32)) invalid("too many frames");
    ADSB_CUDA(cudaSetDevice(ctx.device));
    device_components(ctx);
    const uint64_t dub = device_diameter_bound(ctx);
    ensure_arena(ctx, static_cast<uint32_t>(std::min<uint64_t>(dub + 3, ctx.graph.n + 2)));
    if (ctx.use_smem < 0) ctx.use_smem = std::getenv("ADSB_NO_SMEM") || dub > 128 || ctx.graph.n >= kSmemMaxN ? 0 : 1;
    unsigned long long* events = ctx.rt->pool.get<unsigned long long>(Scratch::kEvents, 1 << 16);
    unsigned long long* scal = ctx.rt->pool.get<unsigned long long>(Scratch::kScal, 4);
    unsigned long long* stats = ctx.rt->pool.get<unsigned long long>(Scratch::kStats, kStatCount);
    ADSB_CUDA(cudaMemsetAsync(stats, 0, kStatCount * sizeof(unsigned long long), ctx.rt->stream));
    SamplerParams p = base_params(ctx, seed, spf);
    p.first = first;
    p.num_items = count;
    p.stats = stats;
    if (!ctx.rt->ev_a) {
        ADSB_CUDA(cudaEventCreate(&ctx.rt->ev_a));
        ADSB_CUDA(cudaEventCreate(&ctx.rt->ev_b));
    }
    Launches L;
    double ms = 0;
    const uint64_t E = run_det_batch(ctx, p, events, scal, L, ctx.rt->ev_a, ctx.rt->ev_b, ms);
    std::vector<unsigned long long> host(E);
    unsigned long long st_host[kStatCount];
    ADSB_CUDA(cudaMemcpy(host.data(), events, E * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    ADSB_CUDA(cudaMemcpy(st_host, stats, sizeof(st_host), cudaMemcpyDeviceToHost));
    if (st_host[kStatErrors] != 0) fail(ADSB_ERR_LOGIC, "sampler reported inconsistent traversals");
    // Events of one frame were reserved in sample order, each sample's in t->s
    // order, so a stable partition by frame restores the reference's layout.
    std::vector<uint64_t> per(count + 1, 0);
    for (auto k : host) per[static_cast<uint32_t>(k) + 1]++;
    for (uint64_t f = 0; f < count; ++f) per[f + 1] += per[f];
    std::memcpy(frame_offsets, per.data(), (count + 1) * sizeof(uint64_t));
    std::vector<uint64_t> cur(per.begin(), per.end() - 1);
    for (uint64_t i = 0; i < E; ++i) {
        const uint64_t slot = cur[static_cast<uint32_t>(host[i])]++;
        if (slot < cap) incs[slot] = static_cast<uint32_t>(host[i] >> 32);
    }
}

}  // namespace adsb
