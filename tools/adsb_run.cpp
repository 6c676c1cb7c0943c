// adsb_run.cpp — `adsamp run` (tools/adsamp_cli.cpp:74-123 in the reference)
// on the B200 engine, written against the C++ drop-in header only.
//
//   adsb_run --graph FILE [--variant indexed] [--threads 8] [--eps 0.01]
//            [--delta 0.1] [--seed 1] [--samples-per-frame 1000]
//            [--epoch-samples 0] [--output scores.csv]
//
// Output matches the reference CLI: a "vertex_id,score" file (original ids,
// %.10g) and the summary lines.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <string>

#include "adsamp_b200.hpp"

using namespace adsamp_b200;

int main(int argc, char** argv) {
    std::map<std::string, std::string> f;
    for (int i = 1; i + 1 < argc; i += 2) f[argv[i]] = argv[i + 1];
    auto get = [&](const char* k, const char* d) {
        auto it = f.find(k);
        return it == f.end() ? std::string(d) : it->second;
    };
    try {
        std::ifstream in(get("--graph", ""));
        if (!in) throw std::runtime_error("cannot open graph file '" + get("--graph", "") + "'");
        const ParsedGraph parsed = parse_edge_list(in);
        EngineConfig cfg;
        const std::string v = get("--variant", "indexed");
        cfg.variant = v == "sequential" ? Variant::sequential : v == "barrier" ? Variant::barrier
                    : v == "local" ? Variant::local : v == "shared" ? Variant::shared : Variant::indexed;
        cfg.threads = static_cast<unsigned>(std::stoul(get("--threads", "1")));
        cfg.frame_groups = std::min(2u, cfg.threads);
        cfg.samples_per_frame = std::stoull(get("--samples-per-frame", "1000"));
        cfg.epoch_samples = std::stoull(get("--epoch-samples", "0"));
        cfg.base_seed = std::stoull(get("--seed", "1"));
        const double eps = std::stod(get("--eps", "0.01"));
        const double delta = std::stod(get("--delta", "0.1"));
        const kadabra::BcResult r = kadabra::estimate_bc(parsed.graph, eps, delta, cfg);

        std::ostream* out = &std::cout;
        std::ofstream file;
        const std::string path = get("--output", "");
        if (!path.empty()) {
            file.open(path);
            out = &file;
        }
        *out << "vertex_id,score\n";
        char line[64];
        for (size_t i = 0; i < r.scores.size(); ++i) {
            std::snprintf(line, sizeof(line), "%llu,%.10g\n",
                          static_cast<unsigned long long>(parsed.original_ids[i]), r.scores[i]);
            *out << line;
        }
        std::cout << "vertices: " << parsed.graph.num_vertices() << "  edges: " << parsed.graph.num_edges() << "\n"
                  << "diameter_bound: " << r.diameter_bound << "  omega: " << r.omega << "\n"
                  << "tau: " << r.tau << "  reason: " << kadabra::to_string(r.reason) << "\n"
                  << "check_cycles: " << r.run.check_cycles << "  stop_epoch: " << r.run.stop_epoch << "\n"
                  << "preprocessing_seconds: " << r.preprocess_seconds << "\n"
                  << "ads_seconds: " << r.ads_seconds << "\n";
    } catch (const ParseError& e) {
        std::cerr << "parse error: " << e.what() << "\n";
        return 2;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
