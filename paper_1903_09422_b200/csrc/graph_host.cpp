// graph_host.cpp — edge-list ingestion and CSR construction (host).
//
// Semantics follow the reference exactly (paths relative to
// /root/reference/proj/include/adsamp/):
//   * graph.hpp:93-131  parse_edge_list — line-based; a line whose first char
//     outside " \t\r" is '%' or '#' is a comment; otherwise two ids read as
//     `istream >> uint64_t` would (skip whitespace, optional sign, decimal
//     digits, overflow fails), then no trailing token, then ids <= 2^32-1.
//     Dense ids follow first appearance (a then b, line by line), self-loop
//     lines included.
//   * graph.hpp:35-58   from_edges — self-loops dropped, both directions,
//     sorted, deduplicated, so every adjacency list is ascending.
// The CSR build is parallel (counting scatter + per-list sort/unique) rather
// than the reference's single global sort; the result is identical.
#include "graph_host.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <new>
#include <fstream>
#include <numeric>
#include <set>
#include <thread>
#include <unordered_map>

#include "common.hpp"
#include "rng.hpp"

namespace adsb {

unsigned host_threads() {
    const unsigned hw = std::thread::hardware_concurrency();
    return hw == 0 ? 1 : std::min(hw, 64u);
}

namespace {

struct HostBlockCache {
    std::mutex mu;
    std::map<size_t, std::vector<void*>> free;  // size class (power of two) -> blocks
    size_t cached = 0;
    int pinned = -1;  // -1 unknown, 0 malloc, 1 cudaHostAlloc
    static constexpr size_t kCap = size_t{8} << 30;  // page-locked bytes kept for reuse
};

HostBlockCache& host_cache() {
    static HostBlockCache* c = new HostBlockCache();  // never destroyed: blocks may outlive statics
    return *c;
}

// Size classes: multiples of 1/8 of the enclosing power of two (at most 12.5%
// slack: a 2.1 GB adjacency array must not round up to 4 GB of pinned memory).
size_t size_class(size_t bytes) {
    size_t p = kHostBlockMin;
    while (p < bytes) p <<= 1;
    const size_t step = std::max(kHostBlockMin, p / 8);
    return (bytes + step - 1) / step * step;
}

}  // namespace

void* host_block_alloc(size_t bytes) {
    HostBlockCache& c = host_cache();
    const size_t cls = size_class(bytes);
    std::lock_guard<std::mutex> lock(c.mu);
    auto it = c.free.find(cls);
    if (it != c.free.end() && !it->second.empty()) {
        void* p = it->second.back();
        it->second.pop_back();
        c.cached -= cls;
        return p;
    }
    if (c.pinned < 0) {
        int count = 0;
        c.pinned = cudaGetDeviceCount(&count) == cudaSuccess && count > 0 ? 1 : 0;
        cudaGetLastError();
    }
    void* p = nullptr;
    if (c.pinned == 1 && cudaHostAlloc(&p, cls, cudaHostAllocPortable) == cudaSuccess) return p;
    cudaGetLastError();
    p = std::malloc(cls);
    if (!p) throw std::bad_alloc();
    return p;
}

void host_block_free(void* p, size_t bytes) noexcept {
    if (!p) return;
    HostBlockCache& c = host_cache();
    const size_t cls = size_class(bytes);
    std::lock_guard<std::mutex> lock(c.mu);
    if (c.cached + cls <= HostBlockCache::kCap) {
        c.free[cls].push_back(p);
        c.cached += cls;
        return;
    }
    cudaPointerAttributes attr{};
    if (cudaPointerGetAttributes(&attr, p) == cudaSuccess && attr.type == cudaMemoryTypeHost) cudaFreeHost(p);
    else std::free(p);
    cudaGetLastError();
}

// Persistent host workers: spawning a std::thread per range cost ~40 us each
// (0.6 ms of C2's 1.75 ms graph_from_csr on 16 cores). run(T, f) calls f(i)
// for i in [0, T): i = 0 on the caller, the rest on pool workers. Calls are
// serialised; a call from inside a worker runs inline.
class HostPool {
  public:
    static HostPool& get() {
        static HostPool* pool = new HostPool();  // never destroyed (workers detach at exit)
        return *pool;
    }
    void run(unsigned T, const std::function<void(unsigned)>& f) {
        if (T <= 1 || in_worker()) {
            for (unsigned i = 0; i < T; ++i) f(i);
            return;
        }
        std::lock_guard<std::mutex> serial(run_mu_);
        ensure(T - 1);
        {
            std::lock_guard<std::mutex> lock(mu_);
            job_ = &f;
            active_ = T - 1;
            pending_ = T - 1;
            ++gen_;
        }
        cv_.notify_all();
        f(0);
        std::unique_lock<std::mutex> lock(mu_);
        done_cv_.wait(lock, [&] { return pending_ == 0; });
        job_ = nullptr;
    }

  private:
    static bool& in_worker() {
        static thread_local bool w = false;
        return w;
    }
    void ensure(unsigned workers) {
        while (threads_.size() < workers) {
            const unsigned id = static_cast<unsigned>(threads_.size());
            threads_.emplace_back([this, id] { loop(id); });
            threads_.back().detach();
        }
    }
    void loop(unsigned id) {
        in_worker() = true;
        uint64_t seen = 0;
        for (;;) {
            const std::function<void(unsigned)>* job;
            {
                std::unique_lock<std::mutex> lock(mu_);
                cv_.wait(lock, [&] { return gen_ != seen; });
                seen = gen_;
                if (id >= active_) continue;
                job = job_;
            }
            (*job)(id + 1);
            std::lock_guard<std::mutex> lock(mu_);
            if (--pending_ == 0) done_cv_.notify_one();
        }
    }
    std::mutex run_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    std::vector<std::thread> threads_;
    const std::function<void(unsigned)>* job_ = nullptr;
    unsigned active_ = 0, pending_ = 0;
    uint64_t gen_ = 0;
};

template <class F>
static void parallel_for(uint64_t count, F&& body) {
    const unsigned T = host_threads();
    if (count < 65536 || T == 1) {
        body(0, count);
        return;
    }
    const uint64_t chunk = (count + T - 1) / T;
    HostPool::get().run(T, [&](unsigned t) {
        const uint64_t b = t * chunk, e = std::min(count, b + chunk);
        if (b < e) body(b, e);
    });
}

void host_parallel_for(uint64_t count, const std::function<void(uint64_t, uint64_t)>& body) {
    parallel_for(count, body);
}

// parallel_for over vertices [0, n) with ranges of about equal adjacency
// volume (offsets: n+1 prefix sums).
template <class F>
static void parallel_for_weighted(uint64_t n, const uint64_t* offsets, F&& body) {
    const unsigned T = host_threads();
    const uint64_t total = offsets[n] + n;  // + n: every vertex costs something
    if (total < 262144 || T == 1) {
        body(0, n);
        return;
    }
    std::vector<uint64_t> cut(1, 0);
    uint64_t b = 0;
    for (unsigned t = 0; t < T && b < n; ++t) {
        uint64_t e = n;
        if (t + 1 < T) {
            const uint64_t target = total * (t + 1) / T;
            uint64_t lo = b, hi = n;  // first vertex u with offsets[u] + u >= target
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if (offsets[mid] + mid < target) lo = mid + 1;
                else hi = mid;
            }
            e = std::max(lo, b + 1);
        }
        cut.push_back(e);
        b = e;
    }
    HostPool::get().run(static_cast<unsigned>(cut.size() - 1), [&](unsigned t) { body(cut[t], cut[t + 1]); });
}


HostGraph graph_from_edges(uint32_t n, const uint32_t* edges, uint64_t m) {
    HostGraph g;
    g.n = n;
    // degree count and scatter on all host threads (relaxed atomic counters:
    // the order inside a list is irrelevant, every list is sorted next)
    std::atomic<bool> out_of_range{false};
    std::vector<uint64_t> deg(static_cast<size_t>(n) + 1, 0);
    parallel_for(m, [&](uint64_t b, uint64_t e) {
        bool bad = false;
        for (uint64_t i = b; i < e; ++i) {
            const uint32_t u = edges[2 * i], v = edges[2 * i + 1];
            if (u == v) continue;
            if (u >= n || v >= n) {
                bad = true;
                continue;
            }
            __atomic_fetch_add(&deg[u + 1], 1, __ATOMIC_RELAXED);
            __atomic_fetch_add(&deg[v + 1], 1, __ATOMIC_RELAXED);
        }
        if (bad) out_of_range = true;
    });
    if (out_of_range) invalid("edge endpoint out of range");
    for (uint32_t u = 0; u < n; ++u) deg[u + 1] += deg[u];
    std::vector<uint32_t, NoInitAlloc<uint32_t>> raw(deg[n]);
    {
        // each thread owns a vertex range of about equal volume and streams
        // the whole edge list, writing only its own lists (no shared cursors:
        // hub counters bounced between cores with atomics)
        std::vector<uint64_t> cur(deg.begin(), deg.end() - 1);
        parallel_for_weighted(n, deg.data(), [&](uint64_t vb, uint64_t ve) {
            for (uint64_t i = 0; i < m; ++i) {
                const uint32_t u = edges[2 * i], v = edges[2 * i + 1];
                if (u == v) continue;
                if (u >= vb && u < ve) raw[cur[u]++] = v;
                if (v >= vb && v < ve) raw[cur[v]++] = u;
            }
        });
    }
    // sort + unique each list in place; record the deduplicated degree
    std::vector<uint64_t> kept(static_cast<size_t>(n) + 1, 0);
    parallel_for_weighted(n, deg.data(), [&](uint64_t b, uint64_t e) {
        for (uint64_t u = b; u < e; ++u) {
            uint32_t* first = raw.data() + deg[u];
            uint32_t* last = raw.data() + deg[u + 1];
            std::sort(first, last);
            kept[u + 1] = static_cast<uint64_t>(std::unique(first, last) - first);
        }
    });
    for (uint32_t u = 0; u < n; ++u) kept[u + 1] += kept[u];
    g.nbrs.resize(kept[n]);
    parallel_for_weighted(n, kept.data(), [&](uint64_t b, uint64_t e) {
        for (uint64_t u = b; u < e; ++u)
            std::memcpy(g.nbrs.data() + kept[u], raw.data() + deg[u],
                        (kept[u + 1] - kept[u]) * sizeof(uint32_t));
    });
    g.offsets.assign(kept.begin(), kept.end());
    // original_ids stays empty: the identity (has_original_ids == false) is written on request
    return g;
}

HostGraph graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs) {
    return graph_from_csr(n, offsets, nbrs, nullptr);
}

HostGraph graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs, CsrChunkSink* sink) {
    if (offsets[0] != 0) invalid("offsets[0] must be 0");
    {
        // monotone offsets first (the weighted split below searches them), by equal vertex ranges
        const unsigned T = n >= (1u << 20) ? host_threads() : 1u;
        std::atomic<bool> decreasing{false};
        HostPool::get().run(T, [&](unsigned t) {
            const uint64_t b = static_cast<uint64_t>(n) * t / T, e = static_cast<uint64_t>(n) * (t + 1) / T;
            bool local = false;
            for (uint64_t u = b; u < e; ++u) local |= offsets[u + 1] < offsets[u];
            if (local) decreasing = true;
        });
        if (decreasing) invalid("offsets must be non-decreasing");
    }
    HostGraph g;
    g.n = n;
    g.offsets.resize(static_cast<size_t>(n) + 1);
    g.nbrs.resize(offsets[n]);
    std::atomic<bool> bad{false};
    // one parallel pass: copy each vertex range and check the Graph invariants
    // (ranges split by adjacency volume: hubs make vertex-count splits uneven)
    parallel_for_weighted(n, offsets, [&](uint64_t b, uint64_t e) {
        std::memcpy(g.offsets.data() + b, offsets + b, (e - b) * sizeof(uint64_t));
        std::memcpy(g.nbrs.data() + offsets[b], nbrs + offsets[b], (offsets[e] - offsets[b]) * sizeof(uint32_t));
        bool local_bad = false;
        for (uint64_t u = b; u < e; ++u) {
            uint64_t prev = UINT64_MAX;
            for (uint64_t i = offsets[u]; i < offsets[u + 1]; ++i) {
                const uint32_t v = nbrs[i];
                local_bad |= v >= n || v == u || (prev != UINT64_MAX && prev >= v);
                prev = v;
            }
        }
        if (local_bad) bad = true;
        else if (sink) sink->chunk(b, e, offsets[b], offsets[e], g);
    });
    g.offsets[n] = offsets[n];
    if (bad) invalid("CSR must have in-range, ascending, duplicate-free, loop-free adjacency");
    // original_ids stays empty: the identity (has_original_ids == false) is written on request
    return g;
}

namespace {

// First-appearance interning (graph.hpp:98-104). Dense small ids go through a
// direct table; anything else through a hash map.
struct Interner {
    std::vector<uint64_t> ids;
    std::unordered_map<uint64_t, uint32_t> map;
    std::vector<uint32_t> table;  // id -> dense+1 while ids stay below table.size()
    static constexpr uint64_t kTableLimit = uint64_t{1} << 27;

    uint32_t operator()(uint64_t id) {
        if (id < kTableLimit) {
            if (id >= table.size()) table.resize(std::min<uint64_t>(kTableLimit, std::max<uint64_t>(id + 1, 2 * table.size())), 0);
            uint32_t& slot = table[id];
            if (slot == 0) {
                ids.push_back(id);
                slot = static_cast<uint32_t>(ids.size());
            }
            return slot - 1;
        }
        auto [it, inserted] = map.try_emplace(id, static_cast<uint32_t>(ids.size()));
        if (inserted) ids.push_back(id);
        return it->second;
    }
};

bool is_space(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

// `istream >> uint64_t` (libstdc++ num_get): see file header.
bool get_u64(const char*& p, const char* e, uint64_t& out) {
    while (p < e && is_space(*p)) ++p;
    bool neg = false;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p == e || *p < '0' || *p > '9') return false;
    uint64_t v = 0;
    bool overflow = false;
    while (p < e && *p >= '0' && *p <= '9') {
        const uint64_t d = static_cast<uint64_t>(*p - '0');
        if (v > (UINT64_MAX - d) / 10) overflow = true;
        v = v * 10 + d;
        ++p;
    }
    if (overflow) return false;
    out = neg ? static_cast<uint64_t>(0 - v) : v;
    return true;
}

HostGraph finish(Interner& in, const std::vector<uint32_t>& edges) {
    if (in.ids.empty()) parse_error("no vertices found in edge list");
    HostGraph g = graph_from_edges(static_cast<uint32_t>(in.ids.size()), edges.data(), edges.size() / 2);
    g.original_ids = std::move(in.ids);
    g.has_original_ids = true;
    return g;
}

}  // namespace

namespace {

// One line-aligned chunk of an edge list, parsed independently.
struct ChunkParse {
    std::vector<uint64_t> ids;  // two per edge, in file order
    uint64_t lines = 0;         // lines in the chunk (blank and comment lines included)
    uint64_t err_line = 0;      // 1-based line (within the chunk) of the first error; 0 = none
    std::string err;            // its message without the "line N: " prefix
};

void parse_chunk(const char* p, const char* end, ChunkParse& r) {
    r.ids.reserve(static_cast<size_t>(end - p) / 6);
    while (p < end) {
        const char* nl = static_cast<const char*>(std::memchr(p, '\n', static_cast<size_t>(end - p)));
        const char* le = nl ? nl : end;
        ++r.lines;
        const char* q = p;
        while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
        if (q == le || *q == '%' || *q == '#') {
            p = nl ? nl + 1 : end;
            continue;
        }
        const char* c = p;
        uint64_t a = 0, b = 0;
        if (!get_u64(c, le, a) || !get_u64(c, le, b)) {
            r.err_line = r.lines;
            r.err = "expected two vertex ids";
            return;
        }
        while (c < le && is_space(*c)) ++c;
        if (c < le) {
            const char* te = c;
            while (te < le && !is_space(*te)) ++te;
            r.err_line = r.lines;
            r.err = "trailing token '" + std::string(c, te) + "'";
            return;
        }
        if (a > 0xFFFFFFFFull || b > 0xFFFFFFFFull) {
            r.err_line = r.lines;
            r.err = "vertex id exceeds 2^32-1";
            return;
        }
        r.ids.push_back(a);
        r.ids.push_back(b);
        p = nl ? nl + 1 : end;
    }
}

}  // namespace

// graph.hpp:93-131. Line-aligned chunks are parsed on all host threads; the
// first error in file order is reported with its global line number, and ids
// are interned in file order afterwards (first appearance fixes the dense
// numbering), so results and messages equal a sequential parse.
HostGraph parse_edge_list_text(const char* text, uint64_t len) {
    unsigned T = host_threads();
    if (len < (uint64_t{4} << 20)) T = 1;
    std::vector<uint64_t> cut(T + 1, len);
    cut[0] = 0;
    for (unsigned t = 1; t < T; ++t) {
        uint64_t pos = std::max(cut[t - 1], len * t / T);
        const char* nl = pos < len ? static_cast<const char*>(std::memchr(text + pos, '\n', len - pos)) : nullptr;
        cut[t] = nl ? static_cast<uint64_t>(nl - text) + 1 : len;
    }
    std::vector<ChunkParse> parts(T);
    if (T == 1) {
        parse_chunk(text, text + len, parts[0]);
    } else {
        HostPool::get().run(T, [&](unsigned t) { parse_chunk(text + cut[t], text + cut[t + 1], parts[t]); });
    }
    uint64_t lines_before = 0, total = 0;
    for (const ChunkParse& r : parts) {
        if (r.err_line) parse_error("line " + std::to_string(lines_before + r.err_line) + ": " + r.err);
        lines_before += r.lines;
        total += r.ids.size();
    }
    Interner in;
    std::vector<uint32_t> edges(total);
    uint64_t k = 0;
    for (ChunkParse& r : parts) {
        for (const uint64_t id : r.ids) edges[k++] = in(id);  // interning order fixes the dense numbering
        std::vector<uint64_t>().swap(r.ids);
    }
    return finish(in, edges);
}

HostGraph parse_edge_list_file(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    if (!f) fail(ADSB_ERR_RUNTIME, "cannot open graph file '" + path + "'");
    f.seekg(0, std::ios::end);
    const auto size = static_cast<uint64_t>(f.tellg());
    f.seekg(0, std::ios::beg);
    std::string buf(size, '\0');
    f.read(buf.data(), static_cast<std::streamsize>(size));
    return parse_edge_list_text(buf.data(), size);
}

HostGraph graph_from_pairs(const uint64_t* pairs, uint64_t m) {
    Interner in;
    std::vector<uint32_t> edges(2 * m);
    for (uint64_t i = 0; i < m; ++i) {
        const uint64_t a = pairs[2 * i], b = pairs[2 * i + 1];
        if (a > 0xFFFFFFFFull || b > 0xFFFFFFFFull)
            parse_error("line " + std::to_string(i + 1) + ": vertex id exceeds 2^32-1");
        edges[2 * i] = in(a);
        edges[2 * i + 1] = in(b);
    }
    return finish(in, edges);
}

// graph.hpp:140-144
std::string serialize_edge_list(const HostGraph& g) {
    std::string out;
    char line[32];
    for (uint32_t u = 0; u < g.n; ++u)
        for (uint64_t i = g.offsets[u]; i < g.offsets[u + 1]; ++i)
            if (u < g.nbrs[i]) {
                const int k = std::snprintf(line, sizeof(line), "%u %u\n", u, g.nbrs[i]);
                out.append(line, static_cast<size_t>(k));
            }
    return out;
}

// ---------------------------------------------------------------------------
// Generators
// ---------------------------------------------------------------------------

// G(n, m) exactly as the reference acceptance suite builds it
// (tests/acceptance.cpp:34-46): distinct unordered pairs drawn with
// next_below(n) until m are collected, emitted in sorted (u < v) order.
std::vector<uint64_t> gen_gnm(uint32_t n, uint64_t m, uint64_t seed) {
    if (n < 2) invalid("G(n,m) needs n >= 2");
    if (m > static_cast<uint64_t>(n) * (n - 1) / 2) invalid("G(n,m): m exceeds n(n-1)/2");
    SplitMix64 rng(seed);
    std::set<std::pair<uint32_t, uint32_t>> edges;
    while (edges.size() < m) {
        auto u = static_cast<uint32_t>(rng.next_below(n));
        auto v = static_cast<uint32_t>(rng.next_below(n));
        if (u == v) continue;
        if (u > v) std::swap(u, v);
        edges.insert({u, v});
    }
    std::vector<uint64_t> out;
    out.reserve(2 * m);
    for (auto [u, v] : edges) {
        out.push_back(u);
        out.push_back(v);
    }
    return out;
}

// R-MAT: edge i draws `scale` quadrant choices from stream reseed(seed, i),
// each from a 53-bit uniform, most significant bit first. Self-loops dropped,
// duplicates kept (from_edges collapses them).
std::vector<uint64_t> gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                               uint64_t seed) {
    if (scale < 1 || scale > 31) invalid("R-MAT scale must lie in [1, 31]");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0)) invalid("R-MAT probabilities invalid");
    const uint64_t m = static_cast<uint64_t>(edge_factor) << scale;
    std::vector<uint64_t> raw(2 * m);
    std::vector<uint8_t> loop(m);
    const double ab = a + b, abc = a + b + c;
    parallel_for(m, [&](uint64_t lo, uint64_t hi) {
        for (uint64_t i = lo; i < hi; ++i) {
            SplitMix64 rng(reseed(seed, i));
            uint64_t u = 0, v = 0;
            for (uint32_t bit = 0; bit < scale; ++bit) {
                const double r = static_cast<double>(rng.next() >> 11) * 0x1.0p-53;
                const uint64_t bu = r >= ab ? 1 : 0;
                const uint64_t bv = (r >= a && r < ab) || r >= abc ? 1 : 0;
                u = (u << 1) | bu;
                v = (v << 1) | bv;
            }
            raw[2 * i] = u;
            raw[2 * i + 1] = v;
            loop[i] = u == v;
        }
    });
    std::vector<uint64_t> out;
    out.reserve(2 * m);
    for (uint64_t i = 0; i < m; ++i)
        if (!loop[i]) {
            out.push_back(raw[2 * i]);
            out.push_back(raw[2 * i + 1]);
        }
    return out;
}

// Barabasi-Albert: K_{m+1} on 0..m (pairs i<j in lexicographic order), then
// each new vertex v picks m distinct targets uniformly from the endpoint list
// (degree-proportional), emitting (v, target) in pick order.
std::vector<uint64_t> gen_ba(uint32_t n, uint32_t m_per, uint64_t seed) {
    if (m_per < 1 || n <= m_per) invalid("BA needs 1 <= m < n");
    SplitMix64 rng(seed);
    std::vector<uint64_t> out;
    std::vector<uint32_t> endpoints;
    const uint64_t total = static_cast<uint64_t>(m_per) * (m_per + 1) / 2 +
                           static_cast<uint64_t>(n - m_per - 1) * m_per;
    out.reserve(2 * total);
    endpoints.reserve(2 * total);
    for (uint32_t i = 0; i <= m_per; ++i)
        for (uint32_t j = i + 1; j <= m_per; ++j) {
            out.push_back(i);
            out.push_back(j);
            endpoints.push_back(i);
            endpoints.push_back(j);
        }
    std::vector<uint32_t> picked(m_per);
    for (uint32_t v = m_per + 1; v < n; ++v) {
        uint32_t k = 0;
        while (k < m_per) {
            const uint32_t t = endpoints[rng.next_below(endpoints.size())];
            bool dup = false;
            for (uint32_t j = 0; j < k; ++j) dup |= picked[j] == t;
            if (!dup) picked[k++] = t;
        }
        for (uint32_t j = 0; j < m_per; ++j) {
            out.push_back(v);
            out.push_back(picked[j]);
            endpoints.push_back(v);
            endpoints.push_back(picked[j]);
        }
    }
    return out;
}

// width x height 4-neighbour lattice, vertex r*width+c; for each vertex in
// row-major order its right then its down edge, each dropped when
// next() < p_drop * 2^64 (threshold as tests/test_util.hpp:86).
std::vector<uint64_t> gen_grid(uint32_t width, uint32_t height, double p_drop, uint64_t seed) {
    if (width < 1 || height < 1) invalid("grid needs positive dimensions");
    if (!(p_drop >= 0.0 && p_drop < 1.0)) invalid("grid drop probability must lie in [0,1)");
    SplitMix64 rng(seed);
    const auto threshold = static_cast<uint64_t>(p_drop * 18446744073709551616.0);
    std::vector<uint64_t> out;
    out.reserve(4ull * width * height);
    for (uint32_t r = 0; r < height; ++r)
        for (uint32_t c = 0; c < width; ++c) {
            const uint64_t u = static_cast<uint64_t>(r) * width + c;
            if (c + 1 < width && rng.next() >= threshold) {
                out.push_back(u);
                out.push_back(u + 1);
            }
            if (r + 1 < height && rng.next() >= threshold) {
                out.push_back(u);
                out.push_back(u + width);
            }
        }
    return out;
}

std::vector<uint64_t> keep_lcc(const std::vector<uint64_t>& pairs) {
    const uint64_t m = pairs.size() / 2;
    uint64_t max_id = 0;
    for (uint64_t x : pairs) max_id = std::max(max_id, x);
    std::vector<uint32_t> parent(max_id + 1);
    std::iota(parent.begin(), parent.end(), 0u);
    auto find = [&](uint32_t x) {
        while (parent[x] != x) x = parent[x] = parent[parent[x]];
        return x;
    };
    std::vector<uint8_t> present(max_id + 1, 0);
    for (uint64_t i = 0; i < m; ++i) {
        const auto u = static_cast<uint32_t>(pairs[2 * i]), v = static_cast<uint32_t>(pairs[2 * i + 1]);
        if (u == v) continue;
        present[u] = present[v] = 1;
        const uint32_t ru = find(u), rv = find(v);
        if (ru != rv) parent[std::max(ru, rv)] = std::min(ru, rv);
    }
    std::vector<uint32_t> size(max_id + 1, 0);
    for (uint64_t x = 0; x <= max_id; ++x)
        if (present[x]) size[find(static_cast<uint32_t>(x))]++;
    uint32_t best = 0;
    for (uint64_t x = 0; x <= max_id; ++x)
        if (size[x] > size[best]) best = static_cast<uint32_t>(x);  // roots are component minima
    std::vector<uint64_t> out;
    out.reserve(pairs.size());
    for (uint64_t i = 0; i < m; ++i) {
        const auto u = static_cast<uint32_t>(pairs[2 * i]), v = static_cast<uint32_t>(pairs[2 * i + 1]);
        if (u == v || find(u) != best) continue;
        out.push_back(u);
        out.push_back(v);
    }
    return out;
}

}  // namespace adsb
