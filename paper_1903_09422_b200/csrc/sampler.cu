// sampler.cu — K1 (deterministic frames) / K2 (epoch samples) path sampler.
//
// Replaces, bit for bit, kadabra.hpp:190-258 (sample_path_between /
// sample_path) driven by the stream keying of engine.hpp:595-610
// (paths relative to /root/reference/proj/include/adsamp/).
//
// One warp is one sampling team; a block holds 8 independent teams and the
// grid is sized to the resident warps (persistent kernel, dynamic tickets).
// Per sample the team runs a balanced bidirectional BFS (expand the side
// whose frontier has the smaller degree sum) instead of the reference's
// forward BFS, then rebuilds sigma_s on the t-side part of the shortest-path
// DAG, then performs the reference's sigma-weighted backtrack from t:
//
//   * sigma is u64 and wraps exactly as the reference's (sums mod 2^64 are
//     order independent, so any traversal yields the same wrapped values);
//   * predecessors are scanned in ascending id order (the CSR is sorted) and
//     chosen by a 65-bit warp prefix sum, equivalent to the sequential
//     `r -= sigma[p]` scan (kadabra.hpp:229-239);
//   * next_below draws are issued in the same order with the same bounds, so
//     the RNG stream is consumed identically and later samples of the same
//     frame stay in lockstep with the reference.
//
// Frontier expansion is warp-cooperative and load-balanced: 32 frontier
// vertices at a time, a warp prefix sum over their degrees, and every lane
// takes one adjacency entry of the flattened range (coalesced reads for hubs
// and for low-degree chunks alike). New vertices are claimed with one 64-bit
// CAS on their state word and appended with ballot/popc compaction.
#include <cstdlib>
#include <string>

#include "device.cuh"
#include "rng.hpp"
#include "sampler.cuh"

namespace adsb {

namespace {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kWarpsPerBlock = 8;
constexpr uint32_t kNone = 0xFFFFFFFFu;

__device__ __forceinline__ unsigned long long mk_meta(uint32_t tag, bool t_side, uint32_t dist) {
    return (static_cast<unsigned long long>(tag) << 32) | (t_side ? kSideT : 0ull) | dist;
}
__device__ __forceinline__ uint32_t tag_of(unsigned long long m) { return static_cast<uint32_t>(m >> 32); }
__device__ __forceinline__ bool is_t(unsigned long long m) { return (m & kSideT) != 0; }
__device__ __forceinline__ uint32_t dist_of(unsigned long long m) { return static_cast<uint32_t>(m & kDistMask); }

__device__ __forceinline__ unsigned long long shfl64(unsigned long long x, int src) {
    return __shfl_sync(kFull, x, src);
}

// owner lane of flattened edge e: number of lanes whose inclusive degree sum is <= e
__device__ __forceinline__ int owner_of(uint32_t incl, uint32_t e) {
    int lo = 0;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        const uint32_t c = __shfl_sync(kFull, incl, lo + s - 1);
        if (c <= e) lo += s;
    }
    return lo;
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t x, uint32_t lane) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, d);
        if (lane >= static_cast<uint32_t>(d)) x += y;
    }
    return x;
}

__device__ __forceinline__ unsigned long long warp_sum64(unsigned long long x) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) x += __shfl_xor_sync(kFull, x, d);
    return x;
}

struct Team {
    const uint32_t* __restrict__ off;
    const uint32_t* __restrict__ nbrs;
    unsigned long long* st;  // this slot: 2 words per vertex
    uint32_t* queue;         // s-side from the front, t-side from the back
    uint2* qrange;
    uint32_t* tlev;
    uint32_t n;
    uint32_t level_cap;
    uint32_t lane;
    uint32_t tag;
    unsigned long long edges;          // BFS expansion
    unsigned long long rebuild_edges;  // DAG sigma rebuild
    unsigned long long back_edges;     // backtrack scans
    unsigned long long verts;
    unsigned long long degenerate;
    bool error;

    __device__ unsigned long long* meta_ptr(uint32_t v) const { return st + 2ull * v; }
    __device__ unsigned long long* sigma_ptr(uint32_t v) const { return st + 2ull * v + 1; }
    __device__ unsigned long long ld_meta(uint32_t v) const { return __ldcg(meta_ptr(v)); }
    __device__ unsigned long long ld_sigma(uint32_t v) const { return __ldcg(sigma_ptr(v)); }
    __device__ ulonglong2 ld_state(uint32_t v) const {
        return __ldcg(reinterpret_cast<const ulonglong2*>(st + 2ull * v));
    }
    // t-side vertex j lives at queue[n-1-j]
    __device__ uint32_t tpos(uint32_t j) const { return n - 1 - j; }
};

// Expand one s-side level: frontier queue[lo, hi) at distance a; claims level
// a+1, accumulates sigma, detects the meeting with the t-ball (level b).
// Returns true when the frontiers met.
__device__ bool expand_s(Team& T, uint32_t lo, uint32_t hi, uint32_t a, uint32_t b, uint32_t& s_cnt,
                         unsigned long long& new_deg) {
    const unsigned long long new_meta = mk_meta(T.tag, false, a + 1);
    const uint32_t lt_mask = (1u << T.lane) - 1u;
    bool met = false;
    unsigned long long my_deg = 0;
    T.verts += hi - lo;
    for (uint32_t base = lo; base < hi; base += 32) {
        const uint32_t idx = base + T.lane;
        uint32_t o = 0, dg = 0;
        unsigned long long su = 0;
        if (idx < hi) {
            const uint2 r = T.qrange[idx];
            o = r.x;
            dg = r.y;
            su = T.ld_sigma(T.queue[idx]);
        }
        const uint32_t incl = warp_incl_scan(dg, T.lane);
        const uint32_t excl = incl - dg;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        T.edges += total;
        for (uint32_t e0 = 0; e0 < total; e0 += 32) {
            const uint32_t e = e0 + T.lane;
            const bool active = e < total;
            const int ow = owner_of(incl, active ? e : 0);
            const uint32_t o_o = __shfl_sync(kFull, o, ow);
            const uint32_t ex_o = __shfl_sync(kFull, excl, ow);
            const unsigned long long su_o = shfl64(su, ow);
            uint32_t v = 0;
            unsigned long long m = 0;
            bool won = false, add = false, hit_t = false;
            if (active) {
                v = T.nbrs[o_o + (e - ex_o)];
                m = T.ld_meta(v);
                if (tag_of(m) != T.tag) {
                    const unsigned long long prev = atomicCAS(T.meta_ptr(v), m, new_meta);
                    if (prev == m) won = true;
                    else m = prev;
                }
                if (!won) {
                    if (!is_t(m)) add = dist_of(m) == a + 1;
                    else hit_t = add = dist_of(m) == b;
                }
            }
            if (won) *T.sigma_ptr(v) = su_o;
            __syncwarp();
            if (add) atomicAdd(T.sigma_ptr(v), su_o);
            if (hit_t && !(m & kDag)) atomicOr(T.meta_ptr(v), kDag);
            met |= __any_sync(kFull, hit_t);
            const uint32_t ball = __ballot_sync(kFull, won);
            if (won) {
                const uint32_t pos = s_cnt + __popc(ball & lt_mask);
                const uint32_t vo = T.off[v];
                const uint32_t vd = T.off[v + 1] - vo;
                T.queue[pos] = v;
                T.qrange[pos] = make_uint2(vo, vd);
                my_deg += vd;
            }
            s_cnt += __popc(ball);
        }
    }
    new_deg = warp_sum64(my_deg);
    __syncwarp();
    return met;
}

// Expand one t-side level: frontier t-positions [lo, hi) at distance b;
// claims level b+1; on touching the s-ball (level a) accumulates sigma_s into
// the touching t-vertex and marks it as a DAG vertex.
__device__ bool expand_t(Team& T, uint32_t lo, uint32_t hi, uint32_t a, uint32_t b, uint32_t& t_cnt,
                         unsigned long long& new_deg) {
    const unsigned long long new_meta = mk_meta(T.tag, true, b + 1);
    const uint32_t lt_mask = (1u << T.lane) - 1u;
    bool met = false;
    unsigned long long my_deg = 0;
    T.verts += hi - lo;
    for (uint32_t base = lo; base < hi; base += 32) {
        const uint32_t j = base + T.lane;
        uint32_t u = 0, o = 0, dg = 0;
        if (j < hi) {
            const uint32_t q = T.tpos(j);
            u = T.queue[q];
            const uint2 r = T.qrange[q];
            o = r.x;
            dg = r.y;
        }
        const uint32_t incl = warp_incl_scan(dg, T.lane);
        const uint32_t excl = incl - dg;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        T.edges += total;
        for (uint32_t e0 = 0; e0 < total; e0 += 32) {
            const uint32_t e = e0 + T.lane;
            const bool active = e < total;
            const int ow = owner_of(incl, active ? e : 0);
            const uint32_t o_o = __shfl_sync(kFull, o, ow);
            const uint32_t ex_o = __shfl_sync(kFull, excl, ow);
            const uint32_t u_o = __shfl_sync(kFull, u, ow);
            uint32_t v = 0;
            bool won = false, hit_s = false;
            if (active) {
                v = T.nbrs[o_o + (e - ex_o)];
                unsigned long long m = T.ld_meta(v);
                if (tag_of(m) != T.tag) {
                    const unsigned long long prev = atomicCAS(T.meta_ptr(v), m, new_meta);
                    if (prev == m) won = true;
                    else m = prev;
                }
                if (!won && !is_t(m) && dist_of(m) == a) {
                    hit_s = true;
                    atomicAdd(T.sigma_ptr(u_o), T.ld_sigma(v));
                    atomicOr(T.meta_ptr(u_o), kDag);
                }
            }
            if (won) *T.sigma_ptr(v) = 0ull;
            met |= __any_sync(kFull, hit_s);
            const uint32_t ball = __ballot_sync(kFull, won);
            if (won) {
                const uint32_t q = T.tpos(t_cnt + __popc(ball & lt_mask));
                const uint32_t vo = T.off[v];
                const uint32_t vd = T.off[v + 1] - vo;
                T.queue[q] = v;
                T.qrange[q] = make_uint2(vo, vd);
                my_deg += vd;
            }
            t_cnt += __popc(ball);
        }
    }
    new_deg = warp_sum64(my_deg);
    __syncwarp();
    return met;
}

// sigma_s on the t-side DAG layer k-1, pulled from layer k: every vertex w of
// T_{k-1} sums sigma_s over its neighbours that are DAG vertices of T_k. The
// cost is T_{k-1}'s degree sum, i.e. exactly what expanding T_{k-1} cost
// (pushing from DAG_k instead would scan the hubs that sit in later layers).
__device__ void rebuild_level(Team& T, uint32_t lo, uint32_t hi, uint32_t k) {
    for (uint32_t base = lo; base < hi; base += 32) {
        const uint32_t j = base + T.lane;
        uint32_t w = 0, o = 0, dg = 0;
        if (j < hi) {
            const uint32_t q = T.tpos(j);
            w = T.queue[q];
            const uint2 r = T.qrange[q];
            o = r.x;
            dg = r.y;
        }
        const uint32_t incl = warp_incl_scan(dg, T.lane);
        const uint32_t excl = incl - dg;
        const uint32_t total = __shfl_sync(kFull, incl, 31);
        T.rebuild_edges += total;
        for (uint32_t e0 = 0; e0 < total; e0 += 32) {
            const uint32_t e = e0 + T.lane;
            const bool active = e < total;
            const int ow = owner_of(incl, active ? e : 0);
            const uint32_t o_o = __shfl_sync(kFull, o, ow);
            const uint32_t ex_o = __shfl_sync(kFull, excl, ow);
            const uint32_t w_o = __shfl_sync(kFull, w, ow);
            if (active) {
                const uint32_t v = T.nbrs[o_o + (e - ex_o)];
                const ulonglong2 sv = T.ld_state(v);
                if (tag_of(sv.x) == T.tag && is_t(sv.x) && dist_of(sv.x) == k && (sv.x & kDag)) {
                    atomicAdd(T.sigma_ptr(w_o), sv.y);
                    atomicOr(T.meta_ptr(w_o), kDag);
                }
            }
        }
    }
    __syncwarp();
}

template <bool kDet>
__device__ void emit(const SamplerParams& p, uint32_t lane, uint32_t v, uint64_t slot_pos,
                     uint32_t frame_local) {
    if (lane != 0) return;
    if (kDet) {
        if (slot_pos < p.ev_cap)
            p.events[slot_pos] = (static_cast<unsigned long long>(v) << 32) | frame_local;
    } else {
        atomicAdd(p.counts + v, 1u);
    }
}

// One sample: kadabra.hpp:250-258 (s, t draw + component check) and
// kadabra.hpp:190-244 (shortest-path count + sigma-weighted backtrack).
template <bool kDet>
__device__ void sample_one(const SamplerParams& p, Team& T, SplitMix64& rng, uint32_t frame_local) {
    const uint32_t n = p.n;
    const uint32_t s = static_cast<uint32_t>(rng.next_below(n));
    uint32_t t = static_cast<uint32_t>(rng.next_below(n - 1));
    if (t >= s) ++t;
    if (__ldg(p.label + s) != __ldg(p.label + t)) return;  // disconnected pair: empty sample

    T.tag += 1;
    if (T.tag == 0) {
        // Generation tags are u32 and persist across calls: after 2^32 samples
        // on this slot the tag wraps to 0, which zero-initialised words carry.
        // Clear the slot's state once and restart at 1.
        for (size_t i = T.lane; i < 2ull * p.slot_stride; i += 32) T.st[i] = 0ull;
        __syncwarp();
        T.tag = 1;
    }
    const uint32_t os = T.off[s], ds = T.off[s + 1] - os;
    const uint32_t ot = T.off[t], dt = T.off[t + 1] - ot;
    if (T.lane == 0) {
        *T.meta_ptr(s) = mk_meta(T.tag, false, 0);
        *T.sigma_ptr(s) = 1ull;
        *T.meta_ptr(t) = mk_meta(T.tag, true, 0);
        *T.sigma_ptr(t) = 0ull;
        T.queue[0] = s;
        T.qrange[0] = make_uint2(os, ds);
        T.queue[T.tpos(0)] = t;
        T.qrange[T.tpos(0)] = make_uint2(ot, dt);
        T.tlev[0] = 0;
        T.tlev[1] = 1;
    }
    __syncwarp();

    uint32_t s_lo = 0, s_hi = 1, s_cnt = 1;  // s frontier = queue[s_lo, s_hi)
    uint32_t t_lo = 0, t_hi = 1, t_cnt = 1;  // t frontier = t-positions [t_lo, t_hi)
    unsigned long long deg_s = ds, deg_t = dt;
    uint32_t a = 0, b = 0;
    for (;;) {
        bool met;
        unsigned long long nd = 0;
        if (deg_s <= deg_t) {
            met = expand_s(T, s_lo, s_hi, a, b, s_cnt, nd);
            if (met) break;
            s_lo = s_hi;
            s_hi = s_cnt;
            deg_s = nd;
            a += 1;
            if (s_lo == s_hi) { T.error = true; return; }
        } else {
            met = expand_t(T, t_lo, t_hi, a, b, t_cnt, nd);
            if (met) break;
            t_lo = t_hi;
            t_hi = t_cnt;
            deg_t = nd;
            b += 1;
            if (b + 2 > T.level_cap || t_lo == t_hi) { T.error = true; return; }
            if (T.lane == 0) T.tlev[b + 1] = t_hi;
            __syncwarp();
        }
    }
    const uint32_t d = a + b + 1;  // d(s, t)

    // sigma_s on the t-side DAG layers b-1 .. 0 (layer b was filled by the meeting)
    for (uint32_t k = b; k >= 1; --k) rebuild_level(T, T.tlev[k - 1], T.tlev[k], k);

    // Backtrack from t (kadabra.hpp:227-242), d-1 interior vertices.
    if (d < 2) return;
    uint64_t ev_pos = 0;
    if (kDet) {
        if (T.lane == 0) ev_pos = atomicAdd(p.ev_cursor, static_cast<unsigned long long>(d - 1));
        ev_pos = shfl64(ev_pos, 0);
    }
    uint32_t cur = t;
    ulonglong2 cs = T.ld_state(t);
    uint32_t ds_cur = d;
    for (uint32_t step = 0; ds_cur > 1; ++step) {
        unsigned long long r = rng.next_below(cs.y);
        // predecessor rule for cur (see file header)
        bool want_t;
        uint32_t want_dist;
        if (is_t(cs.x)) {
            const uint32_t k = dist_of(cs.x);
            want_t = k < b;
            want_dist = k < b ? k + 1 : a;
        } else {
            want_t = false;
            want_dist = dist_of(cs.x) - 1;
        }
        const uint32_t beg = T.off[cur], end = T.off[cur + 1];
        uint32_t chosen = kNone, first_pred = kNone;
        ulonglong2 chosen_state = make_ulonglong2(0, 0), first_state = make_ulonglong2(0, 0);
        for (uint32_t base = beg; base < end; base += 32) {
            const uint32_t i = base + T.lane;
            uint32_t q = 0;
            ulonglong2 sq = make_ulonglong2(0, 0);
            unsigned long long val = 0;
            if (i < end) {
                q = T.nbrs[i];
                sq = T.ld_state(q);
                const bool cand = tag_of(sq.x) == T.tag && is_t(sq.x) == want_t &&
                                  dist_of(sq.x) == want_dist && (!want_t || (sq.x & kDag));
                val = cand ? sq.y : 0ull;
            }
            T.back_edges += min(32u, end - base);
            if (first_pred == kNone) {
                const uint32_t cb = __ballot_sync(kFull, i < end && tag_of(sq.x) == T.tag && is_t(sq.x) == want_t &&
                                                             dist_of(sq.x) == want_dist && (!want_t || (sq.x & kDag)));
                if (cb) {
                    const int f = __ffs(cb) - 1;
                    first_pred = __shfl_sync(kFull, q, f);
                    first_state.x = shfl64(sq.x, f);
                    first_state.y = shfl64(sq.y, f);
                }
            }
            // 65-bit inclusive prefix sum (lo + carry count)
            unsigned long long lo = val;
            uint32_t hi = 0;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const unsigned long long olo = __shfl_up_sync(kFull, lo, dd);
                const uint32_t ohi = __shfl_up_sync(kFull, hi, dd);
                if (T.lane >= static_cast<uint32_t>(dd)) {
                    const unsigned long long nlo = lo + olo;
                    hi += ohi + (nlo < lo ? 1u : 0u);
                    lo = nlo;
                }
            }
            const uint32_t ball = __ballot_sync(kFull, hi > 0 || r < lo);
            if (ball) {
                const int f = __ffs(ball) - 1;
                chosen = __shfl_sync(kFull, q, f);
                chosen_state.x = shfl64(sq.x, f);
                chosen_state.y = shfl64(sq.y, f);
                break;
            }
            r -= shfl64(lo, 31);
        }
        if (chosen == kNone) {
            // sigma(cur) and all predecessor sigmas are 0 mod 2^64: reference UB
            // (oracle.c documents the rule); take the first predecessor
            if (first_pred == kNone) { T.error = true; return; }
            chosen = first_pred;
            chosen_state = first_state;
            T.degenerate += 1;
        }
        emit<kDet>(p, T.lane, chosen, ev_pos + step, frame_local);
        cur = chosen;
        cs = chosen_state;
        ds_cur = is_t(cs.x) ? d - dist_of(cs.x) : dist_of(cs.x);
    }
}

template <bool kDet>
__global__ void __launch_bounds__(256) sampler_kernel(SamplerParams p) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t slot = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
    if (slot >= p.slots) return;
    Team T;
    T.off = p.off;
    T.nbrs = p.nbrs;
    T.n = p.n;
    T.st = p.state + 2ull * p.slot_stride * slot;
    T.queue = p.queue + static_cast<size_t>(p.slot_stride) * slot;
    T.qrange = p.qrange + static_cast<size_t>(p.slot_stride) * slot;
    T.tlev = p.tlev + static_cast<size_t>(p.level_cap) * slot;
    T.level_cap = p.level_cap;
    T.lane = lane;
    T.tag = p.slot_tag[slot];
    T.edges = 0;
    T.rebuild_edges = 0;
    T.back_edges = 0;
    T.verts = 0;
    T.degenerate = 0;
    T.error = false;
    unsigned long long samples = 0;
    for (;;) {
        unsigned long long item = 0;
        if (lane == 0) item = atomicAdd(p.ticket, 1ull);
        item = shfl64(item, 0);
        if (item >= p.num_items) break;
        const uint64_t local = item * p.world + p.rank;  // frame (or sample) index within the batch
        SplitMix64 rng(reseed(p.seed, p.first + local));
        for (uint64_t i = 0; i < p.spf; ++i) {
            sample_one<kDet>(p, T, rng, static_cast<uint32_t>(local));
            ++samples;
        }
    }
    if (lane == 0) {
        p.slot_tag[slot] = T.tag;
        atomicAdd(p.stats + kStatEdges, T.edges + T.rebuild_edges + T.back_edges);
        atomicAdd(p.stats + kStatRebuildEdges, T.rebuild_edges);
        atomicAdd(p.stats + kStatBacktrackEdges, T.back_edges);
        atomicAdd(p.stats + kStatVertices, T.verts);
        atomicAdd(p.stats + kStatSamples, samples);
        if (T.error) atomicAdd(p.stats + kStatErrors, 1ull);
        if (T.degenerate) atomicAdd(p.stats + kStatDegenerate, T.degenerate);
    }
}

}  // namespace

int sampler_warps_per_sm(bool deterministic) {
    int blocks = 0;
    if (deterministic)
        ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, sampler_kernel<true>, 256, 0));
    else
        ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, sampler_kernel<false>, 256, 0));
    return blocks * kWarpsPerBlock;
}

void launch_sampler_warp(bool deterministic, const SamplerParams& p, cudaStream_t stream) {
    const unsigned blocks = (p.slots + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (deterministic)
        sampler_kernel<true><<<blocks, 256, 0, stream>>>(p);
    else
        sampler_kernel<false><<<blocks, 256, 0, stream>>>(p);
    ADSB_CUDA(cudaGetLastError());
}

SamplerKind sampler_kind() {
    const char* e = std::getenv("ADSB_SAMPLER");
    if (e && std::string(e) == "warp") return SamplerKind::kWarp;
    return SamplerKind::kBlock;
}

void launch_sampler(SamplerKind kind, bool deterministic, const SamplerParams& p, cudaStream_t stream) {
    if (kind == SamplerKind::kWarp) launch_sampler_warp(deterministic, p, stream);
    else launch_sampler_cta(deterministic, p, stream);
}

}  // namespace adsb
