// graph_cache.cpp — binary CSR cache.
//
// The reference ingests only text (parse_edge_list, graph.hpp:93-131, a
// single-threaded istringstream pass: minutes for C5's 260M edges). A graph
// that went through that remap once can be saved as its CSR and loaded back
// with parallel reads, with the dense numbering, the ascending adjacency and
// the original ids preserved exactly:
//
//   header  "ADSBCSR1", u32 version, u32 flags (bit 0: original ids present),
//           u32 n, u32 reserved, u64 nnz, u64 checksum
//   body    offsets u64[n+1], neighbours u32[nnz], original ids u64[n] (flag)
//
// The checksum (over every body byte, computed in parallel chunks) catches a
// truncated or damaged file; loading then fails with ParseError.
#include <fcntl.h>
#include <unistd.h>

#include <atomic>
#include <cstring>
#include <string>
#include <vector>

#include "common.hpp"
#include "graph_host.hpp"

namespace adsb {
namespace {

constexpr char kMagic[8] = {'A', 'D', 'S', 'B', 'C', 'S', 'R', '1'};
constexpr uint32_t kVersion = 1;
constexpr uint64_t kChunk = uint64_t{1} << 22;  // bytes per checksum chunk

struct Header {
    char magic[8];
    uint32_t version;
    uint32_t flags;
    uint32_t n;
    uint32_t reserved;
    uint64_t nnz;
    uint64_t checksum;
};
static_assert(sizeof(Header) == 40, "cache header layout");

uint64_t mix(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// order-dependent hash of `bytes` (a multiple of 4) as u32 words, chunked so
// the chunks hash in parallel; `seed` chains the sections
uint64_t section_hash(const void* data, uint64_t bytes, uint64_t seed) {
    const uint64_t chunks = (bytes + kChunk - 1) / kChunk;
    std::vector<uint64_t> part(chunks);
    host_parallel_for(chunks, [&](uint64_t b, uint64_t e) {
        for (uint64_t c = b; c < e; ++c) {
            const auto* p = static_cast<const uint32_t*>(data) + c * (kChunk / 4);
            const uint64_t words = std::min<uint64_t>(kChunk, bytes - c * kChunk) / 4;
            uint64_t h = 0xcbf29ce484222325ull ^ c;
            for (uint64_t i = 0; i < words; ++i) h = (h ^ p[i]) * 0x100000001b3ull;
            part[c] = h;
        }
    });
    uint64_t h = mix(seed ^ bytes);
    for (uint64_t x : part) h = mix(h ^ x);
    return h;
}

uint64_t graph_hash(const HostGraph& g) {
    uint64_t h = section_hash(g.offsets.data(), g.offsets.size() * sizeof(uint64_t), g.n);
    h = section_hash(g.nbrs.data(), g.nbrs.size() * sizeof(uint32_t), h);
    if (g.has_original_ids) h = section_hash(g.original_ids.data(), g.original_ids.size() * sizeof(uint64_t), h);
    return h;
}

struct Fd {
    int fd = -1;
    ~Fd() {
        if (fd >= 0) ::close(fd);
    }
};

// pwrite/pread a section in parallel ranges
void io_section(int fd, void* data, uint64_t bytes, uint64_t file_off, bool write, const std::string& path) {
    constexpr uint64_t kPiece = uint64_t{64} << 20;
    const uint64_t pieces = (bytes + kPiece - 1) / kPiece;
    std::atomic<bool> ok{true};
    host_parallel_for(pieces, [&](uint64_t b, uint64_t e) {
        for (uint64_t k = b; k < e && ok.load(std::memory_order_relaxed); ++k) {
            uint64_t done = 0;
            const uint64_t len = std::min(kPiece, bytes - k * kPiece);
            auto* p = static_cast<char*>(data) + k * kPiece;
            while (done < len) {
                const ssize_t r = write ? ::pwrite(fd, p + done, len - done, static_cast<off_t>(file_off + k * kPiece + done))
                                        : ::pread(fd, p + done, len - done, static_cast<off_t>(file_off + k * kPiece + done));
                if (r <= 0) {
                    ok.store(false);
                    break;
                }
                done += static_cast<uint64_t>(r);
            }
        }
    });
    if (!ok.load()) {
        if (write) fail(ADSB_ERR_RUNTIME, "cannot write graph cache '" + path + "'");
        parse_error("graph cache '" + path + "' is truncated");
    }
}

}  // namespace

void save_graph_cache(const HostGraph& g, const std::string& path) {
    Header h{};
    std::memcpy(h.magic, kMagic, 8);
    h.version = kVersion;
    h.flags = g.has_original_ids ? 1u : 0u;
    h.n = g.n;
    h.nnz = g.nnz();
    h.checksum = graph_hash(g);
    const std::string tmp = path + ".tmp";
    Fd f;
    f.fd = ::open(tmp.c_str(), O_WRONLY | O_CREAT | O_TRUNC, 0644);
    if (f.fd < 0) fail(ADSB_ERR_RUNTIME, "cannot create graph cache '" + path + "'");
    if (::pwrite(f.fd, &h, sizeof h, 0) != static_cast<ssize_t>(sizeof h))
        fail(ADSB_ERR_RUNTIME, "cannot write graph cache '" + path + "'");
    uint64_t off = sizeof h;
    io_section(f.fd, const_cast<uint64_t*>(g.offsets.data()), g.offsets.size() * 8, off, true, path);
    off += g.offsets.size() * 8;
    io_section(f.fd, const_cast<uint32_t*>(g.nbrs.data()), g.nbrs.size() * 4, off, true, path);
    off += g.nbrs.size() * 4;
    if (g.has_original_ids)
        io_section(f.fd, const_cast<uint64_t*>(g.original_ids.data()), g.original_ids.size() * 8, off, true, path);
    if (::close(f.fd) != 0) {
        f.fd = -1;
        fail(ADSB_ERR_RUNTIME, "cannot write graph cache '" + path + "'");
    }
    f.fd = -1;
    if (std::rename(tmp.c_str(), path.c_str()) != 0) fail(ADSB_ERR_RUNTIME, "cannot rename graph cache '" + path + "'");
}

HostGraph load_graph_cache(const std::string& path) {
    Fd f;
    f.fd = ::open(path.c_str(), O_RDONLY);
    if (f.fd < 0) fail(ADSB_ERR_RUNTIME, "cannot open graph cache '" + path + "'");
    Header h{};
    if (::pread(f.fd, &h, sizeof h, 0) != static_cast<ssize_t>(sizeof h) || std::memcmp(h.magic, kMagic, 8) != 0)
        parse_error("'" + path + "' is not an adsb graph cache");
    if (h.version != kVersion) parse_error("graph cache '" + path + "' has version " + std::to_string(h.version));
    const off_t size = ::lseek(f.fd, 0, SEEK_END);
    const uint64_t want = sizeof h + (uint64_t{h.n} + 1) * 8 + h.nnz * 4 + ((h.flags & 1u) ? uint64_t{h.n} * 8 : 0);
    if (size < 0 || static_cast<uint64_t>(size) != want) parse_error("graph cache '" + path + "' is truncated");
    HostGraph g;
    g.n = h.n;
    g.offsets.resize(uint64_t{h.n} + 1);
    g.nbrs.resize(h.nnz);
    uint64_t off = sizeof h;
    io_section(f.fd, g.offsets.data(), g.offsets.size() * 8, off, false, path);
    off += g.offsets.size() * 8;
    io_section(f.fd, g.nbrs.data(), g.nbrs.size() * 4, off, false, path);
    off += g.nbrs.size() * 4;
    g.has_original_ids = (h.flags & 1u) != 0;
    if (g.has_original_ids) {
        g.original_ids.resize(h.n);
        io_section(f.fd, g.original_ids.data(), g.original_ids.size() * 8, off, false, path);
    } else {
        g.original_ids.clear();  // identity, written on request
    }
    if (graph_hash(g) != h.checksum) parse_error("graph cache '" + path + "' is damaged (checksum mismatch)");
    if (g.offsets[0] != 0 || g.offsets[h.n] != h.nnz) parse_error("graph cache '" + path + "' is damaged (offsets)");
    return g;
}

}  // namespace adsb
