// device.cuh — device-resident CSR replica, preprocessing and scratch arenas.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <memory>
#include <atomic>
#include <mutex>
#include <string>
#include <vector>

#include "common.hpp"
#include "graph_host.hpp"

#define ADSB_CUDA(call)                                                                     \
    do {                                                                                    \
        cudaError_t _e = (call);                                                            \
        if (_e != cudaSuccess)                                                              \
            ::adsb::fail(ADSB_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

namespace adsb {

// RAII device allocation.
template <class T>
struct DevBuf {
    T* ptr = nullptr;
    size_t count = 0;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : ptr(o.ptr), count(o.count) { o.ptr = nullptr; o.count = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        reset();
        ptr = o.ptr;
        count = o.count;
        o.ptr = nullptr;
        o.count = 0;
        return *this;
    }
    ~DevBuf() { reset(); }
    void alloc(size_t n) {
        reset();
        if (n == 0) n = 1;
        ADSB_CUDA(cudaMalloc(reinterpret_cast<void**>(&ptr), n * sizeof(T)));
        count = n;
    }
    void reset() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        count = 0;
    }
    size_t bytes() const { return count * sizeof(T); }
};

// Pinned host staging.
template <class T>
struct PinnedBuf {
    T* ptr = nullptr;
    size_t count = 0;
    PinnedBuf() = default;
    PinnedBuf(PinnedBuf&& o) noexcept : ptr(o.ptr), count(o.count) { o.ptr = nullptr; o.count = 0; }
    PinnedBuf& operator=(PinnedBuf&& o) noexcept {
        if (ptr) cudaFreeHost(ptr);
        ptr = o.ptr;
        count = o.count;
        o.ptr = nullptr;
        o.count = 0;
        return *this;
    }
    explicit PinnedBuf(size_t n) {
        if (n == 0) n = 1;
        ADSB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&ptr), n * sizeof(T)));
        count = n;
    }
    PinnedBuf(const PinnedBuf&) = delete;
    PinnedBuf& operator=(const PinnedBuf&) = delete;
    ~PinnedBuf() {
        if (ptr) cudaFreeHost(ptr);
    }
};

// Reusable per-context scratch: buffers grow on demand and are kept between
// calls, so a steady-state estimate_bc performs no cudaMalloc/cudaFree (which
// would synchronise the device) and no pinned-host allocation.
enum class Scratch : int {
    kParent, kIsRoot, kRank, kCubTemp, kFlags, kDist, kFrontA, kFrontB, kLevelCounts, kBest,
    kTotal, kStats, kScal, kBaseMax, kStopIdx, kEvents, kSorted, kGathered, kFrameMax, kRunMax,
    kSortTemp, kEpochCnt, kDmax, kFlagDev, kTickets, kNcclScalar, kCtl, kRingCnt, kRingList, kRingLen, kEvents2, kScal2, kAudit, kMode, kCount
};

struct ScratchPool {
    DevBuf<uint8_t> dev[static_cast<int>(Scratch::kCount)];
    template <class T>
    T* get(Scratch id, size_t count) {
        DevBuf<uint8_t>& b = dev[static_cast<int>(id)];
        const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
        if (b.count < bytes) b.alloc(bytes + bytes / 4 + 256);
        return reinterpret_cast<T*>(b.ptr);
    }
    template <class T>
    size_t capacity(Scratch id) const { return dev[static_cast<int>(id)].count / sizeof(T); }
};

struct DeviceGraph {
    int device = 0;
    uint32_t n = 0;
    uint64_t nnz = 0;
    uint32_t max_degree = 0;
    DevBuf<uint32_t> offsets;  // n+1 (nnz < 2^32 on the device path)
    DevBuf<uint32_t> nbrs;     // nnz
    // search trees over the rows of high-degree vertices (hub_index.cuh), built
    // on the first estimate for this handle when the CSR misses L2: hub_ref[v] =
    // word offset of v's tree in hub_keys (meaningful only where hub_has_tree(deg v))
    DevBuf<uint32_t> hub_ref;
    DevBuf<uint32_t> hub_keys;
};

// Per-(graph, device) sampler scratch: one "slot" per concurrently running
// sample team. Each slot holds per-vertex state (16 B), a visit queue with
// the visited vertices' CSR ranges, and the t-side level boundaries.
struct SamplerArena {
    int kind = 1;            // SamplerKind (0 warp teams, 1 block teams)
    uint32_t hash_cap = 0;   // block teams: shared-memory hash capacity
    uint32_t block_threads = 256;
    bool vec4 = false;       // blocks sized for the vector kernels' dynamic shared memory
    int layout = 0;          // block teams' global state: 1 cleared (low-degree graphs), 0 tagged
    uint32_t slots = 0;      // warp teams; block teams: global-state regions
    uint32_t blocks = 0;     // block teams: resident blocks launched by the shared-memory kernels
    uint32_t n = 0;
    uint32_t level_cap = 0;
    DevBuf<unsigned long long> state;  // slots * n * 2 (meta, sigma)
    DevBuf<uint32_t> queue;            // slots * n
    DevBuf<uint2> qrange;              // slots * n (offset, degree)
    DevBuf<uint32_t> tlev;             // slots * level_cap
    DevBuf<uint32_t> dagq;             // block teams: slots * n t-side DAG lists (push rebuild, low-degree graphs)
    DevBuf<uint32_t> slot_tag;         // slots: generation tag of each region
    DevBuf<uint32_t> slot_busy;        // block teams: bitmap of regions lent to blocks
};

// Process-wide per-device runtime shared by every graph handle on that
// device: streams, events, the scratch pool, pinned staging and the sampler
// arenas. Creating a graph therefore costs only its CSR upload. Calls that use
// the runtime hold `mu` (one engine call per device at a time).
struct DeviceRuntime {
    int device = 0;
    std::mutex mu;
    std::unique_ptr<SamplerArena> arena[2];    // per SamplerKind
    int active = 1;                            // arena used by the current call
    ScratchPool pool;
    PinnedBuf<unsigned long long> pinned;      // 128 words of small host staging (level counts, flags, stats)
    PinnedBuf<uint32_t> host_counts;           // result download
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, ev_stat = nullptr;
    cudaEvent_t ev_samp[2] = {nullptr, nullptr}, ev_chk[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t> ev_launch;
    cudaStream_t stream = nullptr;   // sampling stream
    cudaStream_t stream2 = nullptr;  // check / collective stream
    // Device buffers of destroyed graphs, reused by the next graphs (avoids a
    // cudaFree + cudaMalloc pair, which synchronises the device, per handle).
    std::mutex spare_mu;
    std::vector<DevBuf<uint32_t>> spare;
};

// best-fit reuse of a spare buffer (within 2x of the request), else a fresh allocation
DevBuf<uint32_t> take_buffer(DeviceRuntime& rt, size_t count);
void give_buffer(DeviceRuntime& rt, DevBuf<uint32_t>&& b);

// Never destroyed: lives until process exit (CUDA tears its resources down then).
DeviceRuntime& device_runtime(int device);

struct DeviceContext {
    int device = 0;
    DeviceGraph graph;
    DevBuf<uint32_t> labels;  // component labels (reference numbering)
    bool labels_ready = false;
    bool dub_ready = false;   // the graph is immutable: labels and D_ub are computed once per handle
    bool hub_ready = false;   // hub search trees built (or found unnecessary)
    int use_smem = -1;        // block teams: -1 undecided, 0 global-store-only, 1 shared-memory table first
    uint64_t diameter_bound = 0;
    uint32_t num_components = 0;
    DeviceRuntime* rt = nullptr;
    ~DeviceContext();
};

int resolve_device(int requested);
std::unique_ptr<DeviceContext> make_device_context(const HostGraph& g, int device);
// Streaming construction (adsb_graph_from_csr): device buffers are taken
// first and each validated host range is uploaded as soon as its worker is
// done, so the copy overlaps validation of the other ranges.
struct StreamingUpload : CsrChunkSink {
    std::unique_ptr<DeviceContext> ctx;
    std::vector<uint32_t, NoInitAlloc<uint32_t>> off32;  // u32 offsets staging (page-locked when large)
    std::atomic<uint32_t> max_degree{0};
    std::unique_lock<std::mutex> lock;  // the device runtime (its stream) while uploading
    void chunk(uint64_t b, uint64_t e, uint64_t nb, uint64_t ne, const HostGraph& g) override;
};
std::unique_ptr<StreamingUpload> begin_streaming_upload(uint32_t n, uint64_t nnz, int device);
inline CsrChunkSink* streaming_sink(StreamingUpload& up) { return &up; }
std::unique_ptr<DeviceContext> finish_streaming_upload(std::unique_ptr<StreamingUpload> up, const HostGraph& g);
void abort_streaming_upload(std::unique_ptr<StreamingUpload> up);

// graph.hpp:153-175 connected_components: labels numbered by smallest member
// (exactly the reference's numbering); returns the component count.
uint32_t device_components(DeviceContext& ctx);
// graph.hpp:178-197 eccentricity
uint64_t device_eccentricity(DeviceContext& ctx, uint32_t source);
// graph.hpp:202-214 diameter_upper_bound (requires device_components first)
uint64_t device_diameter_bound(DeviceContext& ctx);

// search trees over high-degree adjacency rows (hub_index.cu), once per handle
void device_hub_index(DeviceContext& ctx);

// exact normalised BC (Brandes, f64; brandes.cu); returns the kernel time in ms
double device_exact_bc(DeviceContext& ctx, double* host_bc);

int num_sms(int device);

}  // namespace adsb
