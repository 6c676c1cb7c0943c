// graph_host.hpp — host-side graph ingestion with the reference's semantics.
//
//   parse_edge_list   graph.hpp:93-131  (first-appearance remap, comments, errors)
//   from_edges        graph.hpp:35-58   (drop self-loops, symmetrise, sort, dedup)
//
// The CSR built here is uploaded once per device (graph_device.cuh); all
// traversal work happens on the GPU.
#pragma once

#include <cstdint>
#include <functional>
#include <memory>
#include <string>
#include <utility>
#include <vector>

namespace adsb {

// Large host blocks (>= kHostBlockMin bytes) come from a process-wide cache:
// page-locked when a CUDA device is present (the device upload is then a
// direct DMA), plain malloc otherwise; freed blocks are kept for reuse
// (bounded), so building graphs repeatedly does not re-fault or re-pin pages.
constexpr size_t kHostBlockMin = size_t{256} << 10;
void* host_block_alloc(size_t bytes);
void host_block_free(void* p, size_t bytes) noexcept;

// Allocator that leaves trivially-constructible elements uninitialised on
// resize: large CSR arrays are filled by parallel copies right after.
template <class T>
struct NoInitAlloc : std::allocator<T> {
    using value_type = T;
    template <class U>
    struct rebind {
        using other = NoInitAlloc<U>;
    };
    NoInitAlloc() = default;
    template <class U>
    NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
    T* allocate(size_t count) {
        const size_t bytes = count * sizeof(T);
        if (bytes >= kHostBlockMin) return static_cast<T*>(host_block_alloc(bytes));
        return std::allocator<T>::allocate(count);
    }
    void deallocate(T* p, size_t count) noexcept {
        const size_t bytes = count * sizeof(T);
        if (bytes >= kHostBlockMin) host_block_free(p, bytes);
        else std::allocator<T>::deallocate(p, count);
    }
    template <class U>
    bool operator==(const NoInitAlloc<U>&) const noexcept { return true; }
    template <class U>
    bool operator!=(const NoInitAlloc<U>&) const noexcept { return false; }
    template <class U>
    void construct(U*) noexcept {}
    template <class U, class... A>
    void construct(U* p, A&&... a) {
        ::new (static_cast<void*>(p)) U(std::forward<A>(a)...);
    }
};

struct HostGraph {
    uint32_t n = 0;
    std::vector<uint64_t, NoInitAlloc<uint64_t>> offsets;  // n+1
    std::vector<uint32_t, NoInitAlloc<uint32_t>> nbrs;     // offsets[n], ascending per vertex
    std::vector<uint64_t> original_ids;  // dense -> id in the input (empty = identity when !has_original_ids)
    bool has_original_ids = false;

    uint64_t nnz() const { return nbrs.size(); }
    uint64_t degree(uint32_t u) const { return offsets[u + 1] - offsets[u]; }
};

// [0, count) split over the persistent host workers (inline when small)
void host_parallel_for(uint64_t count, const std::function<void(uint64_t, uint64_t)>& body);

HostGraph graph_from_edges(uint32_t n, const uint32_t* edges, uint64_t m);
HostGraph graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs);
// The same, calling chunk(b, e, g) from the worker that has just copied and
// validated vertices [b, e) into g (the device upload of that range can start
// while other ranges are still being validated). Throws after all workers
// finished if any range was invalid.
struct CsrChunkSink {
    // vertices [b, e), adjacency entries [nb, ne) of g
    virtual void chunk(uint64_t b, uint64_t e, uint64_t nb, uint64_t ne, const HostGraph& g) = 0;
    virtual ~CsrChunkSink() = default;
};
HostGraph graph_from_csr(uint32_t n, const uint64_t* offsets, const uint32_t* nbrs, CsrChunkSink* sink);
HostGraph parse_edge_list_text(const char* text, uint64_t len);
HostGraph parse_edge_list_file(const std::string& path);
HostGraph graph_from_pairs(const uint64_t* pairs, uint64_t m);
std::string serialize_edge_list(const HostGraph& g);
// binary CSR cache (graph_cache.cpp): exact round trip, parallel I/O, checksummed
void save_graph_cache(const HostGraph& g, const std::string& path);
HostGraph load_graph_cache(const std::string& path);

// Synthetic generators. Output: 2*m original ids.
std::vector<uint64_t> gen_gnm(uint32_t n, uint64_t m, uint64_t seed);
std::vector<uint64_t> gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                               uint64_t seed);
std::vector<uint64_t> gen_ba(uint32_t n, uint32_t m_per, uint64_t seed);
std::vector<uint64_t> gen_grid(uint32_t width, uint32_t height, double p_drop, uint64_t seed);
// keep only edges of the largest connected component (ties: the component
// holding the smallest id); self-loops dropped
std::vector<uint64_t> keep_lcc(const std::vector<uint64_t>& pairs);

unsigned host_threads();

}  // namespace adsb
