// engine.hpp — host orchestration of the device sampling pipelines.
#pragma once

#include <cstdint>
#include <vector>

#include "device.cuh"

struct adsb_comm;

namespace adsb {

struct EngineOptions {
    bool deterministic = true;     // indexed frames vs cumulative epochs
    bool barrier = false;          // cumulative epochs as run_barrier rounds (dense count all-reduce on N GPUs)
    uint64_t spf = 1000;           // samples per frame (deterministic)
    uint64_t epoch_samples = 0;    // samples per epoch over all ranks (0 = 1024; barrier: check_interval)
    uint64_t check_interval = 1000;
    bool bounded_memory = false;   // engine.hpp:92: cap frames ahead of the cutoff
    uint32_t reservation_block = 4;
    uint64_t queue_high_water = 64;
    uint64_t seed = 1;
    uint64_t max_cycles = 0;       // 0 = until the stopping rule
    uint32_t nominal_threads = 1;  // T for stop_epoch (engine.hpp:562)
    double c = 0.5;                // omega constant (kadabra.hpp:321)
    adsb_comm* comm = nullptr;
};

struct EngineOutput {
    // RunResult::data: the pinned download buffer of the device runtime, valid
    // while the caller holds the runtime lock (capi copies it out); nullptr = all 0
    const uint32_t* counts = nullptr;
    uint64_t tau = 0, check_cycles = 0, stop_epoch = 0, total_samples = 0;
    uint64_t omega = 0, diameter_bound = 0;
    int32_t reason = ADSB_REASON_EPS_CONVERGED;
    uint32_t num_components = 0;
    double preprocess_seconds = 0, ads_seconds = 0;
    uint64_t edges_scanned = 0, vertices_expanded = 0, kernel_launches = 0;
    uint64_t rebuild_edges = 0, backtrack_edges = 0, store_fallbacks = 0, degenerate_steps = 0;
    double sampler_ms = 0;
    // engine.hpp:156-161 QueueStats (per sampler team)
    uint64_t queue_max_depth = 0, queue_allocated = 0;
    double queue_mean_depth = 0;
    bool queue_high_water_exceeded = false;
    uint32_t world = 1;
};

// kadabra.hpp:41-53
uint64_t compute_omega(uint64_t diameter_bound, double eps, double delta, double c);
// kadabra.hpp:59-67 (host evaluation; the device uses the same operation order)
double f_kernel(double b, double log_inv, double omega, double tau);
double g_kernel(double b, double log_inv, double omega, double tau);
// kadabra_converged with uniform deltas reduces to the test at the max count
bool converged_at_max(uint64_t max_count, uint64_t tau, uint64_t omega, double eps, double log_inv);

EngineOutput estimate_bc(DeviceContext& ctx, double eps, double delta, const EngineOptions& opt);

// Parity hook: per-frame increments of frames [first, first+count).
void sample_frames(DeviceContext& ctx, uint64_t seed, uint64_t spf, uint64_t first, uint64_t count,
                   uint64_t* frame_offsets, uint32_t* incs, uint64_t cap);

}  // namespace adsb
