// adsamp_b200.hpp — header-only C++ drop-in for the reference's adsamp API,
// implemented over the C ABI of libadsb.so (include/adsb.h).
//
// A reference user switches by replacing
//     #include "adsamp/graph.hpp"       (graph.hpp:29-131)
//     #include "adsamp/kadabra.hpp"     (kadabra.hpp:295-348)
// with
//     #include "adsamp_b200.hpp"
// and linking -ladsb. Types, names, argument meaning and exception classes
// mirror the reference; every traversal runs on the GPU.
#pragma once

#include <cstdint>
#include <istream>
#include <iterator>
#include <memory>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "adsb.h"

namespace adsamp_b200 {

struct ParseError : std::runtime_error {  // graph.hpp:85-87
    explicit ParseError(const std::string& w) : std::runtime_error(w) {}
};

namespace detail {
[[noreturn]] inline void raise(adsb_status s) {
    const std::string msg = adsb_last_error();
    switch (s) {
        case ADSB_ERR_INVALID_ARGUMENT: throw std::invalid_argument(msg);
        case ADSB_ERR_DOMAIN: throw std::domain_error(msg);
        case ADSB_ERR_PARSE: throw ParseError(msg);
        case ADSB_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}
inline void check(adsb_status s) {
    if (s != ADSB_OK) raise(s);
}
}  // namespace detail

using VertexId = std::uint32_t;

// graph.hpp:29-76
class Graph {
public:
    Graph() = default;
    explicit Graph(adsb_graph* h) : h_(h, &adsb_graph_destroy) { refresh(); }

    static Graph from_edges(VertexId num_vertices, std::span<const std::pair<VertexId, VertexId>> edges) {
        std::vector<std::uint32_t> flat;
        flat.reserve(edges.size() * 2);
        for (auto [u, v] : edges) {
            flat.push_back(u);
            flat.push_back(v);
        }
        adsb_graph* h = nullptr;
        detail::check(adsb_graph_from_edges(num_vertices, flat.data(), edges.size(), &h));
        return Graph(h);
    }

    VertexId num_vertices() const noexcept { return n_; }
    std::uint64_t num_edges() const noexcept { return nnz_ / 2; }
    const std::vector<std::uint64_t>& offsets() const { load(); return offsets_; }
    const std::vector<VertexId>& neighbor_list() const { load(); return neighbors_; }
    std::span<const VertexId> neighbors(VertexId u) const {
        load();
        return {neighbors_.data() + offsets_[u], neighbors_.data() + offsets_[u + 1]};
    }
    std::uint64_t degree(VertexId u) const { load(); return offsets_[u + 1] - offsets_[u]; }
    const adsb_graph* handle() const noexcept { return h_.get(); }

private:
    void refresh() { detail::check(adsb_graph_info(h_.get(), &n_, &nnz_)); }
    void load() const {
        if (loaded_) return;
        offsets_.resize(static_cast<size_t>(n_) + 1);
        neighbors_.resize(nnz_);
        detail::check(adsb_graph_copy_csr(h_.get(), offsets_.data(), neighbors_.data()));
        loaded_ = true;
    }
    std::shared_ptr<adsb_graph> h_;
    std::uint32_t n_ = 0;
    std::uint64_t nnz_ = 0;
    mutable bool loaded_ = false;
    mutable std::vector<std::uint64_t> offsets_;
    mutable std::vector<VertexId> neighbors_;
};

struct ParsedGraph {  // graph.hpp:80-83
    Graph graph;
    std::vector<std::uint64_t> original_ids;
};

inline ParsedGraph parsed_from(adsb_graph* h) {
    ParsedGraph p{Graph(h), {}};
    p.original_ids.resize(p.graph.num_vertices());
    detail::check(adsb_graph_copy_original_ids(p.graph.handle(), p.original_ids.data()));
    return p;
}

// graph.hpp:93-136
inline ParsedGraph parse_edge_list(const std::string& text) {
    adsb_graph* h = nullptr;
    detail::check(adsb_graph_parse_text(text.data(), text.size(), &h));
    return parsed_from(h);
}
inline ParsedGraph parse_edge_list(std::istream& in) {
    std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
    return parse_edge_list(text);
}

struct ComponentLabels {  // graph.hpp:146-151
    std::vector<VertexId> label;
    VertexId num_components = 0;
    bool same_component(VertexId u, VertexId v) const noexcept { return label[u] == label[v]; }
};

inline ComponentLabels connected_components(const Graph& g, int device = -1) {
    ComponentLabels cc;
    cc.label.resize(g.num_vertices());
    detail::check(adsb_connected_components(g.handle(), device, cc.label.data(), &cc.num_components));
    return cc;
}
inline std::uint64_t eccentricity(const Graph& g, VertexId source, int device = -1) {
    std::uint64_t out = 0;
    detail::check(adsb_eccentricity(g.handle(), device, source, &out));
    return out;
}
inline std::uint64_t diameter_upper_bound(const Graph& g, int device = -1) {
    std::uint64_t out = 0;
    detail::check(adsb_diameter_upper_bound(g.handle(), device, &out));
    return out;
}

// engine.hpp:63-106
enum class Variant { sequential = ADSB_VARIANT_SEQUENTIAL, barrier = ADSB_VARIANT_BARRIER, local = ADSB_VARIANT_LOCAL,
                     shared = ADSB_VARIANT_SHARED, indexed = ADSB_VARIANT_INDEXED };

struct EngineConfig {
    unsigned threads = 1;
    Variant variant = Variant::local;
    unsigned frame_groups = 2;
    std::uint64_t check_interval = 1000;
    double latency_exponent = 1.33;
    std::uint64_t samples_per_frame = 1000;
    bool bounded_memory = false;
    unsigned reservation_block = 4;
    std::uint64_t queue_high_water = 64;
    std::uint64_t base_seed = 1;
    // GPU pipeline
    std::uint64_t epoch_samples = 0;
    std::uint64_t max_cycles = 0;
    int device = -1;
    adsb_comm* comm = nullptr;

    // engine.hpp:97-105 (the C ABI re-validates and throws the same messages)
    void validate() const {
        if (threads < 1) throw std::invalid_argument("threads must be >= 1");
        if (variant == Variant::shared && (frame_groups < 1 || frame_groups > threads))
            throw std::invalid_argument("frame groups must satisfy 1 <= F <= T");
        if (check_interval < 1) throw std::invalid_argument("check interval must be >= 1");
        if (!(latency_exponent > 0)) throw std::invalid_argument("xi must be > 0");
        if (samples_per_frame < 1) throw std::invalid_argument("samples per frame must be >= 1");
        if (reservation_block < 1) throw std::invalid_argument("reservation block must be >= 1");
    }

    adsb_config to_c() const {
        adsb_config c;
        adsb_config_init(&c);
        c.variant = static_cast<int32_t>(variant);
        c.threads = threads;
        c.frame_groups = frame_groups;
        c.check_interval = check_interval;
        c.latency_exponent = latency_exponent;
        c.samples_per_frame = samples_per_frame;
        c.epoch_samples = epoch_samples;
        c.base_seed = base_seed;
        c.max_cycles = max_cycles;
        c.device = device;
        c.comm = comm;
        c.bounded_memory = bounded_memory ? 1u : 0u;
        c.reservation_block = reservation_block;
        c.queue_high_water = queue_high_water;
        return c;
    }
};

struct QueueStats {  // engine.hpp:156-161 (per sampler team on the GPU)
    std::uint64_t max_depth = 0;
    double mean_depth = 0.0;
    std::uint64_t allocated = 0;
    bool high_water_exceeded = false;
};

struct RunResult {  // engine.hpp:163-171
    std::vector<std::uint64_t> data;
    std::uint64_t num = 0;
    std::uint64_t total_samples = 0;
    std::vector<std::uint64_t> per_thread_samples;
    std::uint64_t check_cycles = 0;
    std::uint64_t stop_epoch = 0;
    QueueStats queue;
};

// audit.hpp:36-80. Accepted for signature compatibility with estimate_bc
// (kadabra.hpp:308-309). The device pipelines have no per-thread event log to
// hand to it; their consistency replay is tests/test_gpu_parity.py's audit tests.
class AuditSink;

namespace kadabra {

enum class StopReason { eps_converged, omega_reached, capped };

inline const char* to_string(StopReason r) {
    return r == StopReason::eps_converged ? "eps_converged" : r == StopReason::omega_reached ? "omega_reached" : "capped";
}

struct BcResult {  // kadabra.hpp:295-304
    std::vector<double> scores;
    std::uint64_t tau = 0;
    StopReason reason = StopReason::eps_converged;
    std::uint64_t omega = 0;
    std::uint64_t diameter_bound = 0;
    double preprocess_seconds = 0.0;
    double ads_seconds = 0.0;
    RunResult run;
    adsb_stats device{};  // executed-algorithm counters
};

inline std::uint64_t compute_omega(std::uint64_t diameter_bound, double epsilon, double delta, double c = 0.5) {
    std::uint64_t out = 0;
    detail::check(adsb_compute_omega(diameter_bound, epsilon, delta, c, &out));
    return out;
}
inline double f_bound(double b, double delta_l, std::uint64_t omega, std::uint64_t tau) {
    double out = 0;
    detail::check(adsb_f_bound(b, delta_l, omega, tau, &out));
    return out;
}
inline double g_bound(double b, double delta_u, std::uint64_t omega, std::uint64_t tau) {
    double out = 0;
    detail::check(adsb_g_bound(b, delta_u, omega, tau, &out));
    return out;
}

// kadabra.hpp:308-348
inline BcResult estimate_bc(const Graph& g, double epsilon, double delta, const EngineConfig& config,
                            AuditSink* audit = nullptr) {
    (void)audit;
    config.validate();
    BcResult r;
    const adsb_config c = config.to_c();
    r.scores.resize(g.num_vertices());
    r.run.data.resize(g.num_vertices());
    detail::check(adsb_estimate_bc(g.handle(), epsilon, delta, &c, r.scores.data(), r.run.data.data(), &r.device));
    r.tau = r.device.tau;
    r.reason = static_cast<StopReason>(r.device.reason);
    r.omega = r.device.omega;
    r.diameter_bound = r.device.diameter_bound;
    r.preprocess_seconds = r.device.preprocess_seconds;
    r.ads_seconds = r.device.ads_seconds;
    r.run.num = r.device.tau;
    r.run.total_samples = r.device.total_samples;
    r.run.per_thread_samples = {r.device.total_samples};
    r.run.check_cycles = r.device.check_cycles;
    r.run.stop_epoch = r.device.stop_epoch;
    r.run.queue = {r.device.queue_max_depth, r.device.queue_mean_depth, r.device.queue_allocated,
                   r.device.queue_high_water_exceeded != 0};
    return r;
}

// Exact normalised BC on the device (Brandes, f64): the validation the
// reference runs with ApspOracle (tests/test_util.hpp:164-206), at C2's size.
inline std::vector<double> exact_bc(const Graph& g, int device = -1) {
    std::vector<double> bc(g.num_vertices());
    detail::check(adsb_exact_bc(g.handle(), device, bc.data(), nullptr));
    return bc;
}

}  // namespace kadabra
}  // namespace adsamp_b200
