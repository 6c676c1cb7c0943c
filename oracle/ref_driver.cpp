// ref_driver.cpp — drives the UNMODIFIED reference headers
// (/root/reference/proj/include/adsamp/*.hpp, included by path at build time,
// never copied) so their outputs can pin the C restatement (oracle.c) and serve
// as the CPU baseline (`bench.py --impl reference`).
//
// TEST INFRASTRUCTURE ONLY. Built by oracle/Makefile into oracle/_ref/.
// The reference CLI (tools/adsamp_cli.cpp) needs CLI11, which is absent, so
// this driver stands in for `adsamp run` (adsamp_cli.cpp:74-123).
//
//   (--graph F: text edge list; --graph-bin F: dense pairs for Graph::from_edges)
//   ref_driver run    --graph F --eps E --delta D --seed S --variant V --spf K
//                     --threads T [--check-interval N] [--max-cycles C] [--counts OUT]
//   ref_driver frames --graph F --seed S --spf K --first P --count C --out OUT
//   ref_driver dub    --graph F

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "adsamp/engine.hpp"
#include "adsamp/graph.hpp"
#include "adsamp/harness.hpp"
#include "adsamp/kadabra.hpp"
#include "adsamp/rng.hpp"

using namespace adsamp;

namespace {

std::map<std::string, std::string> parse_flags(int argc, char** argv, int first) {
    std::map<std::string, std::string> f;
    for (int i = first; i + 1 < argc; i += 2) f[argv[i]] = argv[i + 1];
    return f;
}

std::string get(const std::map<std::string, std::string>& f, const char* k, const char* dflt) {
    auto it = f.find(k);
    return it == f.end() ? std::string(dflt) : it->second;
}

ParsedGraph load_text(const std::string& path) {
    std::ifstream in(path);
    if (!in) throw std::runtime_error("cannot open graph file '" + path + "'");
    return parse_edge_list(in);
}

// --graph-bin: u32 n, u64 m, m x (u32, u32) dense ids already in parse_edge_list's
// first-appearance order (oracle/gen.c or_write_dense_edges), built with the
// reference's own Graph::from_edges (graph.hpp:35-58) — the same CSR as parsing
// the text, without the single-threaded istringstream pass over GBs of text.
ParsedGraph load_bin(const std::string& path) {
    std::ifstream in(path, std::ios::binary);
    if (!in) throw std::runtime_error("cannot open graph file '" + path + "'");
    std::uint32_t n = 0;
    std::uint64_t m = 0;
    in.read(reinterpret_cast<char*>(&n), sizeof n);
    in.read(reinterpret_cast<char*>(&m), sizeof m);
    std::vector<std::pair<VertexId, VertexId>> edges(m);
    std::vector<std::uint32_t> buf(2 * m);
    in.read(reinterpret_cast<char*>(buf.data()), static_cast<std::streamsize>(buf.size() * sizeof(std::uint32_t)));
    if (!in) throw std::runtime_error("truncated graph file '" + path + "'");
    for (std::uint64_t i = 0; i < m; ++i) edges[i] = {buf[2 * i], buf[2 * i + 1]};
    std::vector<std::uint32_t>().swap(buf);
    ParsedGraph out;
    out.graph = Graph::from_edges(n, edges);
    return out;
}

ParsedGraph load(const std::map<std::string, std::string>& f) {
    auto it = f.find("--graph-bin");
    if (it != f.end()) return load_bin(it->second);
    auto jt = f.find("--graph");
    return load_text(jt == f.end() ? std::string() : jt->second);
}

std::uint64_t fnv1a(const std::vector<std::uint64_t>& v) {
    std::uint64_t h = 0xcbf29ce484222325ull;
    for (std::uint64_t x : v)
        for (int b = 0; b < 8; ++b) {
            h ^= (x >> (8 * b)) & 0xFF;
            h *= 0x100000001b3ull;
        }
    return h;
}

int cmd_run(const std::map<std::string, std::string>& f) {
    using clock = std::chrono::steady_clock;
    const auto tl0 = clock::now();
    const ParsedGraph parsed = load(f);
    const double load_s = std::chrono::duration<double>(clock::now() - tl0).count();
    const Graph& g = parsed.graph;
    EngineConfig cfg;
    cfg.variant = parse_variant(get(f, "--variant", "indexed"));
    cfg.threads = static_cast<unsigned>(std::stoul(get(f, "--threads", "1")));
    if (cfg.variant == Variant::sequential) cfg.threads = 1;
    cfg.frame_groups = std::min(2u, cfg.threads);
    cfg.check_interval = std::stoull(get(f, "--check-interval", "1000"));
    cfg.samples_per_frame = std::stoull(get(f, "--spf", "1000"));
    cfg.base_seed = std::stoull(get(f, "--seed", "1"));
    const double eps = std::stod(get(f, "--eps", "0.01"));
    const double delta = std::stod(get(f, "--delta", "0.1"));
    const std::uint64_t max_cycles = std::stoull(get(f, "--max-cycles", "0"));
    const int reps = std::stoi(get(f, "--reps", "1"));

    kadabra::BcResult r;
    std::string reason;
    std::string rep_times;
    // Capped runs: estimate_bc's preprocessing (kadabra.hpp:319-325) once per
    // process, then every rep runs the sampler wrapped in FixedCycleSampler
    // (harness.hpp:23-42); only ads_seconds is reported per rep.
    std::optional<ComponentLabels> cc;
    std::optional<kadabra::KadabraParams> params;
    double pre_s = 0.0;
    if (max_cycles != 0) {
        const auto t0 = clock::now();
        cc.emplace(connected_components(g));
        params.emplace(kadabra::KadabraParams::for_graph(g, eps, delta, 0.5, cfg.check_interval,
                                                         cfg.latency_exponent));
        pre_s = std::chrono::duration<double>(clock::now() - t0).count();
    }
    for (int rep = 0; rep < reps; ++rep) {
    if (max_cycles == 0) {
        r = kadabra::estimate_bc(g, eps, delta, cfg);
        reason = kadabra::to_string(r.reason);
    } else {
        kadabra::Sampler sampler(g, *cc, *params);
        FixedCycleSampler<kadabra::Sampler> capped(sampler, max_cycles);
        const auto t1 = clock::now();
        r.run = run(capped, cfg);
        const auto t2 = clock::now();
        r.tau = r.run.num;
        r.omega = params->omega;
        r.diameter_bound = params->diameter_bound;
        r.preprocess_seconds = pre_s;
        r.ads_seconds = std::chrono::duration<double>(t2 - t1).count();
        reason = "capped";
    }
    char buf[64];
    std::snprintf(buf, sizeof(buf), "%s[%.6f, %llu]", rep ? ", " : "", r.ads_seconds,
                  static_cast<unsigned long long>(r.run.total_samples));
    rep_times += buf;
    }
    const auto cpath = get(f, "--counts", "");
    if (!cpath.empty()) {
        std::ofstream out(cpath, std::ios::binary);
        out.write(reinterpret_cast<const char*>(r.run.data.data()),
                  static_cast<std::streamsize>(r.run.data.size() * sizeof(std::uint64_t)));
    }
    std::printf(
        "{\"n\": %u, \"m\": %llu, \"variant\": \"%s\", \"threads\": %u, \"spf\": %llu, "
        "\"tau\": %llu, \"check_cycles\": %llu, \"stop_epoch\": %llu, \"omega\": %llu, "
        "\"diameter_bound\": %llu, \"reason\": \"%s\", \"total_samples\": %llu, "
        "\"preprocess_s\": %.6f, \"ads_s\": %.6f, \"counts_fnv1a\": \"%016llx\", "
        "\"load_s\": %.3f, \"reps\": [%s]}\n",
        g.num_vertices(), static_cast<unsigned long long>(g.num_edges()), to_string(cfg.variant),
        cfg.threads, static_cast<unsigned long long>(cfg.samples_per_frame),
        static_cast<unsigned long long>(r.tau), static_cast<unsigned long long>(r.run.check_cycles),
        static_cast<unsigned long long>(r.run.stop_epoch), static_cast<unsigned long long>(r.omega),
        static_cast<unsigned long long>(r.diameter_bound), reason.c_str(),
        static_cast<unsigned long long>(r.run.total_samples), r.preprocess_seconds, r.ads_seconds,
        static_cast<unsigned long long>(fnv1a(r.run.data)), load_s, rep_times.c_str());
    return 0;
}

// Per-frame increments straight from kadabra::sample_path (kadabra.hpp:250-258)
// with the run_indexed stream keying (engine.hpp:595). Output: for each frame
// a u64 length followed by that many u32 vertex ids.
int cmd_frames(const std::map<std::string, std::string>& f) {
    const ParsedGraph parsed = load(f);
    const Graph& g = parsed.graph;
    const ComponentLabels cc = connected_components(g);
    kadabra::PathScratch scratch(g.num_vertices());
    const std::uint64_t seed = std::stoull(get(f, "--seed", "1"));
    const std::uint64_t spf = std::stoull(get(f, "--spf", "1"));
    const std::uint64_t first = std::stoull(get(f, "--first", "0"));
    const std::uint64_t count = std::stoull(get(f, "--count", "1"));
    std::ofstream out(get(f, "--out", "frames.bin"), std::ios::binary);
    std::vector<std::uint32_t> inc;
    for (std::uint64_t p = first; p < first + count; ++p) {
        SplitMix64 rng = stream_rng(seed, p);
        inc.clear();
        for (std::uint64_t i = 0; i < spf; ++i) kadabra::sample_path(g, cc, scratch, rng, inc);
        const std::uint64_t len = inc.size();
        out.write(reinterpret_cast<const char*>(&len), sizeof(len));
        out.write(reinterpret_cast<const char*>(inc.data()),
                  static_cast<std::streamsize>(len * sizeof(std::uint32_t)));
    }
    return 0;
}

int cmd_dub(const std::map<std::string, std::string>& f) {
    const ParsedGraph parsed = load(f);
    const Graph& g = parsed.graph;
    const ComponentLabels cc = connected_components(g);
    std::printf("{\"n\": %u, \"m\": %llu, \"components\": %u, \"diameter_bound\": %llu}\n",
                g.num_vertices(), static_cast<unsigned long long>(g.num_edges()), cc.num_components,
                static_cast<unsigned long long>(diameter_upper_bound(g)));
    return 0;
}

} // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_driver run|frames|dub [--flag value]...\n");
        return 2;
    }
    try {
        const auto flags = parse_flags(argc, argv, 2);
        const std::string cmd = argv[1];
        if (cmd == "run") return cmd_run(flags);
        if (cmd == "frames") return cmd_frames(flags);
        if (cmd == "dub") return cmd_dub(flags);
        std::fprintf(stderr, "unknown command '%s'\n", cmd.c_str());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
