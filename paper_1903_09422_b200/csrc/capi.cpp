// capi.cpp — the extern "C" boundary declared in include/adsb.h.
//
// Each entry point mirrors one reference function (paths relative to
// /root/reference/proj/include/adsamp/) and maps its exceptions onto status
// codes via adsb::guard (common.hpp).
#include <cmath>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>

#include "adsb.h"
#include "comm.hpp"
#include "device.cuh"
#include "engine.hpp"
#include "graph_host.hpp"

struct adsb_graph {
    adsb::HostGraph host;
    std::mutex mu;
    std::map<int, std::unique_ptr<adsb::DeviceContext>> devices;
};

namespace adsb {

namespace {
thread_local std::string g_last_error;

DeviceContext& context_for(const adsb_graph* cg, int requested) {
    auto* g = const_cast<adsb_graph*>(cg);
    const int dev = resolve_device(requested);
    std::lock_guard<std::mutex> lock(g->mu);
    auto it = g->devices.find(dev);
    if (it == g->devices.end()) it = g->devices.emplace(dev, make_device_context(g->host, dev)).first;
    return *it->second;
}

// The device runtime (streams, scratch, arenas) is shared by all graphs on a
// device: engine calls on one device are serialised.
struct Locked {
    DeviceContext& ctx;
    std::unique_lock<std::mutex> lock;
};
Locked locked_context(const adsb_graph* g, int requested) {
    DeviceContext& ctx = context_for(g, requested);
    return {ctx, std::unique_lock<std::mutex>(ctx.rt->mu)};
}

adsb_graph* wrap(HostGraph&& h) {
    auto* g = new adsb_graph;
    g->host = std::move(h);
    return g;
}

void need(const void* p, const char* what) {
    if (!p) invalid(std::string(what) + " must not be null");
}

// engine.hpp:97-105 EngineConfig::validate
void validate(const adsb_config& c) {
    if (c.threads < 1) invalid("threads must be >= 1");
    if (c.variant == ADSB_VARIANT_SHARED && (c.frame_groups < 1 || c.frame_groups > c.threads))
        invalid("frame groups must satisfy 1 <= F <= T");
    if (c.check_interval < 1) invalid("check interval must be >= 1");
    if (!(c.latency_exponent > 0)) invalid("xi must be > 0");
    if (c.samples_per_frame < 1) invalid("samples per frame must be >= 1");
    if (c.reservation_block < 1) invalid("reservation block must be >= 1");
    if (c.variant < ADSB_VARIANT_SEQUENTIAL || c.variant > ADSB_VARIANT_INDEXED) invalid("unknown variant");
    if (c.flags != 0) invalid("flags must be 0");
}
}  // namespace

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace adsb

using namespace adsb;

extern "C" {

const char* adsb_last_error(void) { return g_last_error.c_str(); }
int adsb_abi_version(void) { return ADSB_ABI_VERSION; }

void adsb_config_init(adsb_config* cfg) {
    if (!cfg) return;
    std::memset(cfg, 0, sizeof(*cfg));
    cfg->struct_size = sizeof(adsb_config);
    cfg->variant = ADSB_VARIANT_INDEXED;
    cfg->threads = 1;
    cfg->frame_groups = 2;
    cfg->check_interval = 1000;
    cfg->latency_exponent = 1.33;
    cfg->samples_per_frame = 1000;
    cfg->epoch_samples = 0;
    cfg->base_seed = 1;
    cfg->max_cycles = 0;
    cfg->device = -1;
    cfg->comm = nullptr;
    cfg->bounded_memory = 0;
    cfg->reservation_block = 4;
    cfg->queue_high_water = 64;
}

adsb_status adsb_graph_parse_text(const char* text, uint64_t len, adsb_graph** out) {
    return guard([&] {
        need(out, "out");
        need(text, "text");
        *out = wrap(parse_edge_list_text(text, len));
    });
}

adsb_status adsb_graph_parse_file(const char* path, adsb_graph** out) {
    return guard([&] {
        need(out, "out");
        need(path, "path");
        *out = wrap(parse_edge_list_file(path));
    });
}

adsb_status adsb_graph_save(const adsb_graph* g, const char* path) {
    return guard([&] {
        need(g, "graph");
        need(path, "path");
        save_graph_cache(g->host, path);
    });
}

adsb_status adsb_graph_load(const char* path, adsb_graph** out) {
    return guard([&] {
        need(out, "out");
        need(path, "path");
        *out = wrap(load_graph_cache(path));
    });
}

adsb_status adsb_graph_from_pairs(const uint64_t* pairs, uint64_t m, adsb_graph** out) {
    return guard([&] {
        need(out, "out");
        if (m) need(pairs, "pairs");
        *out = wrap(graph_from_pairs(pairs, m));
    });
}

adsb_status adsb_graph_from_edges(uint32_t n, const uint32_t* edges, uint64_t m, adsb_graph** out) {
    return guard([&] {
        need(out, "out");
        if (m) need(edges, "edges");
        *out = wrap(graph_from_edges(n, edges, m));
    });
}

adsb_status adsb_graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* neighbors,
                                adsb_graph** out) {
    return guard([&] {
        need(out, "out");
        need(offsets, "offsets");
        if (offsets[n]) need(neighbors, "neighbors");
        // With a GPU present, the current device's CSR replica is uploaded
        // range by range while the host copy is still being validated.
        int count = 0;
        if (std::getenv("ADSB_NO_EAGER_UPLOAD") || cudaGetDeviceCount(&count) != cudaSuccess || count == 0 ||
            offsets[n] >= 0xFFFFFFFFull) {
            cudaGetLastError();
            *out = wrap(graph_from_csr(n, offsets, neighbors));
            return;
        }
        const int dev = resolve_device(-1);
        auto up = begin_streaming_upload(n, offsets[n], dev);
        HostGraph h;
        try {
            h = graph_from_csr(n, offsets, neighbors, streaming_sink(*up));
        } catch (...) {
            abort_streaming_upload(std::move(up));
            throw;
        }
        auto ctx = finish_streaming_upload(std::move(up), h);
        adsb_graph* g = wrap(std::move(h));
        g->devices.emplace(dev, std::move(ctx));
        *out = g;
    });
}

void adsb_graph_destroy(adsb_graph* g) { delete g; }

adsb_status adsb_graph_info(const adsb_graph* g, uint32_t* n, uint64_t* nnz) {
    return guard([&] {
        need(g, "graph");
        if (n) *n = g->host.n;
        if (nnz) *nnz = g->host.nnz();
    });
}

adsb_status adsb_graph_copy_csr(const adsb_graph* g, uint64_t* offsets, uint32_t* neighbors) {
    return guard([&] {
        need(g, "graph");
        if (offsets) std::memcpy(offsets, g->host.offsets.data(), g->host.offsets.size() * sizeof(uint64_t));
        if (neighbors && g->host.nnz())
            std::memcpy(neighbors, g->host.nbrs.data(), g->host.nnz() * sizeof(uint32_t));
    });
}

adsb_status adsb_graph_copy_original_ids(const adsb_graph* g, uint64_t* out) {
    return guard([&] {
        need(g, "graph");
        need(out, "out");
        if (g->host.has_original_ids) {
            std::memcpy(out, g->host.original_ids.data(), g->host.original_ids.size() * sizeof(uint64_t));
        } else {  // constructed from dense ids: the identity
            for (uint32_t v = 0; v < g->host.n; ++v) out[v] = v;
        }
    });
}

adsb_status adsb_graph_serialize(const adsb_graph* g, char* buf, uint64_t* len) {
    return guard([&] {
        need(g, "graph");
        need(len, "len");
        const std::string s = serialize_edge_list(g->host);
        if (buf && *len >= s.size()) std::memcpy(buf, s.data(), s.size());
        *len = s.size();
    });
}

adsb_status adsb_connected_components(const adsb_graph* g, int device, uint32_t* labels,
                                      uint32_t* num_components) {
    return guard([&] {
        need(g, "graph");
        Locked L = locked_context(g, device);
        DeviceContext& ctx = L.ctx;
        const uint32_t c = device_components(ctx);
        if (num_components) *num_components = c;
        if (labels && g->host.n)
            ADSB_CUDA(cudaMemcpy(labels, ctx.labels.ptr, g->host.n * sizeof(uint32_t), cudaMemcpyDeviceToHost));
    });
}

adsb_status adsb_eccentricity(const adsb_graph* g, int device, uint32_t source, uint64_t* out) {
    return guard([&] {
        need(g, "graph");
        need(out, "out");
        Locked L = locked_context(g, device);
        *out = device_eccentricity(L.ctx, source);
    });
}

adsb_status adsb_diameter_upper_bound(const adsb_graph* g, int device, uint64_t* out) {
    return guard([&] {
        need(g, "graph");
        need(out, "out");
        Locked L = locked_context(g, device);
        *out = g->host.n == 0 ? 0 : device_diameter_bound(L.ctx);
    });
}

adsb_status adsb_compute_omega(uint64_t diameter_bound, double eps, double delta, double c, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        *out = compute_omega(diameter_bound, eps, delta, c);
    });
}

// kadabra.hpp:69-91
static void bound_domain(double b, double delta_v, uint64_t tau) {
    if (tau < 1) domain("tau must be >= 1");
    if (!(delta_v > 0.0 && delta_v < 1.0)) domain("per-vertex delta must lie in (0,1)");
    if (!(b >= 0.0 && b <= 1.0)) domain("b_tilde must lie in [0,1]");
}

adsb_status adsb_f_bound(double b, double delta_l, uint64_t omega, uint64_t tau, double* out) {
    return guard([&] {
        need(out, "out");
        bound_domain(b, delta_l, tau);
        *out = f_kernel(b, std::log(1.0 / delta_l), static_cast<double>(omega), static_cast<double>(tau));
    });
}

adsb_status adsb_g_bound(double b, double delta_u, uint64_t omega, uint64_t tau, double* out) {
    return guard([&] {
        need(out, "out");
        bound_domain(b, delta_u, tau);
        *out = g_kernel(b, std::log(1.0 / delta_u), static_cast<double>(omega), static_cast<double>(tau));
    });
}

// engine.hpp:110-116
adsb_status adsb_check_budget(uint64_t check_interval, uint32_t threads, double xi, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        if (check_interval < 1 || threads < 1 || !(xi > 0))
            invalid("check_budget: need N >= 1, T >= 1, xi > 0");
        const double v = static_cast<double>(check_interval) / std::pow(threads, xi);
        const auto rounded = std::llround(v);
        *out = rounded < 1 ? 1 : static_cast<uint64_t>(rounded);
    });
}

// engine.hpp:137-144 (the claim number k stands for the counter's fetch_add result)
adsb_status adsb_reserve_indices(uint64_t claim, uint32_t threads, uint32_t a, uint64_t* out) {
    return guard([&] {
        need(out, "out");
        if (threads < 1) invalid("threads must be >= 1");
        const uint64_t base = (claim / threads) * threads * (a + 1ull) + (claim % threads);
        for (uint32_t m = 0; m <= a; ++m) out[m] = base + static_cast<uint64_t>(m) * threads;
    });
}

// kadabra.hpp:133-151 with uniform deltas
adsb_status adsb_kadabra_check(const uint64_t* data, uint64_t n, uint64_t num, uint64_t omega, double eps,
                               double delta, int* stop) {
    return guard([&] {
        need(stop, "stop");
        if (num >= omega) {
            *stop = 1;
            return;
        }
        if (num < 1) domain("stopping check needs at least one sample");
        if (n) need(data, "data");
        const double delta_v = delta / (2.0 * static_cast<double>(n));
        const double log_inv = std::log(1.0 / delta_v);
        int ok = 1;
        for (uint64_t v = 0; v < n && ok; ++v) {
            const double b = static_cast<double>(data[v]) / static_cast<double>(num);
            if (f_kernel(b, log_inv, static_cast<double>(omega), static_cast<double>(num)) > eps) ok = 0;
            else if (g_kernel(b, log_inv, static_cast<double>(omega), static_cast<double>(num)) > eps) ok = 0;
        }
        *stop = ok;
    });
}

adsb_status adsb_estimate_bc(const adsb_graph* g, double epsilon, double delta, const adsb_config* cfg,
                             double* scores, uint64_t* counts, adsb_stats* stats) {
    return guard([&] {
        need(g, "graph");
        need(cfg, "config");
        if (cfg->struct_size != sizeof(adsb_config)) invalid("adsb_config.struct_size mismatch");
        validate(*cfg);
        if (g->host.n == 0) invalid("graph has no vertices");  // kadabra.hpp:310
        EngineOptions opt;
        opt.deterministic = cfg->variant == ADSB_VARIANT_INDEXED || cfg->variant == ADSB_VARIANT_SEQUENTIAL;
        opt.barrier = cfg->variant == ADSB_VARIANT_BARRIER;
        opt.spf = cfg->samples_per_frame;
        opt.epoch_samples = cfg->epoch_samples;
        opt.check_interval = cfg->check_interval;
        opt.bounded_memory = cfg->bounded_memory != 0;
        opt.reservation_block = cfg->reservation_block;
        opt.queue_high_water = cfg->queue_high_water;
        opt.seed = cfg->base_seed;
        opt.max_cycles = cfg->max_cycles;
        opt.nominal_threads = cfg->variant == ADSB_VARIANT_SEQUENTIAL ? 1 : cfg->threads;
        opt.comm = cfg->comm;
        int device = cfg->device;
        if (cfg->comm) device = cfg->comm->device;
        Locked L = locked_context(g, device);
        EngineOutput r = adsb::estimate_bc(L.ctx, epsilon, delta, opt);
        const uint32_t n = g->host.n;
        // r.counts points into the runtime's pinned buffer: copied out while the
        // runtime lock (L) is still held
        if (counts) {
            if (r.counts)  // fresh caller memory: page faults and widening spread over the host workers
                host_parallel_for(n, [&](uint64_t b, uint64_t e) { std::copy(r.counts + b, r.counts + e, counts + b); });
            else std::fill(counts, counts + n, uint64_t{0});
        }
        if (scores)  // kadabra.hpp:334-337
            host_parallel_for(n, [&](uint64_t b, uint64_t e) {
                for (uint64_t v = b; v < e; ++v)
                    scores[v] = r.tau == 0 || !r.counts ? 0.0 : static_cast<double>(r.counts[v]) / static_cast<double>(r.tau);
            });
        if (stats) {
            stats->tau = r.tau;
            stats->check_cycles = r.check_cycles;
            stats->stop_epoch = r.stop_epoch;
            stats->total_samples = r.total_samples;
            stats->omega = r.omega;
            stats->diameter_bound = r.diameter_bound;
            stats->reason = r.reason;
            stats->num_components = r.num_components;
            stats->preprocess_seconds = r.preprocess_seconds;
            stats->ads_seconds = r.ads_seconds;
            stats->edges_scanned = r.edges_scanned;
            stats->vertices_expanded = r.vertices_expanded;
            stats->kernel_launches = r.kernel_launches;
            stats->sampler_ms = r.sampler_ms;
            stats->rebuild_edges = r.rebuild_edges;
            stats->backtrack_edges = r.backtrack_edges;
            stats->store_fallbacks = r.store_fallbacks;
            stats->degenerate_steps = r.degenerate_steps;
            stats->queue_max_depth = r.queue_max_depth;
            stats->queue_mean_depth = r.queue_mean_depth;
            stats->queue_allocated = r.queue_allocated;
            stats->queue_high_water_exceeded = r.queue_high_water_exceeded ? 1u : 0u;
            stats->world = r.world;
        }
    });
}

adsb_status adsb_sample_frames(const adsb_graph* g, int device, uint64_t seed, uint64_t spf, uint64_t first,
                               uint64_t count, uint64_t* frame_offsets, uint32_t* incs, uint64_t cap) {
    return guard([&] {
        need(g, "graph");
        need(frame_offsets, "frame_offsets");
        if (cap) need(incs, "incs");
        if (g->host.n < 2) invalid("sampling needs at least two vertices");
        Locked L = locked_context(g, device);
        sample_frames(L.ctx, seed, spf, first, count, frame_offsets, incs, cap);
    });
}

adsb_status adsb_exact_bc(const adsb_graph* g, int device, double* bc, double* device_ms) {
    return guard([&] {
        need(g, "graph");
        need(bc, "bc");
        if (g->host.n == 0) invalid("graph is empty");
        Locked L = locked_context(g, device);
        const double ms = device_exact_bc(L.ctx, bc);
        if (device_ms) *device_ms = ms;
    });
}

adsb_status adsb_comm_unique_id(uint8_t id[128]) {
    return guard([&] {
        need(id, "id");
        static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
        ncclUniqueId uid;
        ADSB_NCCL(ncclGetUniqueId(&uid));
        std::memcpy(id, &uid, 128);
    });
}

adsb_status adsb_comm_init(int nranks, int rank, const uint8_t id[128], int device, adsb_comm** out) {
    return guard([&] {
        need(id, "id");
        need(out, "out");
        if (nranks < 1 || rank < 0 || rank >= nranks) invalid("rank out of range");
        const int dev = resolve_device(device);
        ADSB_CUDA(cudaSetDevice(dev));
        ncclUniqueId uid;
        std::memcpy(&uid, id, 128);
        auto c = std::make_unique<adsb_comm>();
        c->nranks = nranks;
        c->rank = rank;
        c->device = dev;
        ADSB_NCCL(ncclCommInitRank(&c->comm, nranks, uid, rank));
        *out = c.release();
    });
}

adsb_status adsb_comm_init_host(int nranks, int rank, int device, const adsb_host_collectives* ops, void* user,
                                adsb_comm** out) {
    return guard([&] {
        need(ops, "ops");
        need(out, "out");
        if (!ops->allreduce_u64 || !ops->allreduce_u32_sum || !ops->allgather_u64)
            invalid("every host collective must be set");
        if (nranks < 1 || rank < 0 || rank >= nranks) invalid("rank out of range");
        auto c = std::make_unique<adsb_comm>();
        c->host = *ops;
        c->user = user;
        c->nranks = nranks;
        c->rank = rank;
        c->device = resolve_device(device);
        *out = c.release();
    });
}

void adsb_comm_destroy(adsb_comm* comm) { delete comm; }

static adsb_status hand_out(std::vector<uint64_t>&& v, uint64_t** pairs, uint64_t* count) {
    need(pairs, "pairs");
    need(count, "count");
    *count = v.size() / 2;
    *pairs = static_cast<uint64_t*>(std::malloc(std::max<size_t>(1, v.size()) * sizeof(uint64_t)));
    if (!*pairs) throw std::bad_alloc();
    std::memcpy(*pairs, v.data(), v.size() * sizeof(uint64_t));
    return ADSB_OK;
}

adsb_status adsb_gen_gnm(uint32_t n, uint64_t m, uint64_t seed, int lcc, uint64_t** pairs, uint64_t* count) {
    return guard([&] {
        auto v = gen_gnm(n, m, seed);
        hand_out(lcc ? keep_lcc(v) : std::move(v), pairs, count);
    });
}

adsb_status adsb_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed,
                          int lcc, uint64_t** pairs, uint64_t* count) {
    return guard([&] {
        auto v = gen_rmat(scale, edge_factor, a, b, c, seed);
        hand_out(lcc ? keep_lcc(v) : std::move(v), pairs, count);
    });
}

adsb_status adsb_gen_ba(uint32_t n, uint32_t m_per, uint64_t seed, uint64_t** pairs, uint64_t* count) {
    return guard([&] { hand_out(gen_ba(n, m_per, seed), pairs, count); });
}

adsb_status adsb_gen_grid(uint32_t width, uint32_t height, double p_drop, uint64_t seed, int lcc,
                          uint64_t** pairs, uint64_t* count) {
    return guard([&] {
        auto v = gen_grid(width, height, p_drop, seed);
        hand_out(lcc ? keep_lcc(v) : std::move(v), pairs, count);
    });
}

adsb_status adsb_write_edge_list(const char* path, const uint64_t* pairs, uint64_t m) {
    return guard([&] {
        need(path, "path");
        FILE* f = std::fopen(path, "wb");
        if (!f) fail(ADSB_ERR_RUNTIME, std::string("cannot open '") + path + "' for writing");
        std::string buf;
        buf.reserve(1 << 22);
        char line[48];
        for (uint64_t i = 0; i < m; ++i) {
            const int k = std::snprintf(line, sizeof(line), "%llu %llu\n",
                                        static_cast<unsigned long long>(pairs[2 * i]),
                                        static_cast<unsigned long long>(pairs[2 * i + 1]));
            buf.append(line, static_cast<size_t>(k));
            if (buf.size() > (1 << 22)) {
                std::fwrite(buf.data(), 1, buf.size(), f);
                buf.clear();
            }
        }
        std::fwrite(buf.data(), 1, buf.size(), f);
        std::fclose(f);
    });
}

void adsb_free(void* p) { std::free(p); }

}  // extern "C"
