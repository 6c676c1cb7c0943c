// sampler_cta.cu — block-per-sample K1/K2 sampler with shared-memory state.
//
// Same contract as sampler.cu (bit-exact kadabra.hpp:190-258 under the
// engine.hpp:595-610 keying; paths relative to /root/reference/proj/include/
// adsamp/), restructured for B200's memory hierarchy:
//
//   * one thread block (256 threads) owns one sample at a time (persistent
//     grid, dynamic tickets);
//   * the per-sample visited set (vertex -> side/dist/dag, sigma) lives in a
//     shared-memory open-addressing hash table, cleared per sample; the CSR is
//     the only global data a sample reads (L2-resident for C1-C3);
//   * every BFS level first PROBES its frontier's adjacency for the other
//     side's ball and only CLAIMS new vertices when the frontiers did not meet,
//     so the large meeting level (typically >90% of the scanned adjacency)
//     performs no insertions at all and only the two pre-meeting balls occupy
//     the table (C2: mean 121 vertices, C3: 673);
//   * frontier adjacency is flattened across the whole block: a block scan over
//     the frontier degrees, then each thread takes edges e = tid, tid+256, ...
//     and finds its owner vertex by binary search in the scan (hubs and
//     low-degree frontiers are balanced alike);
//   * a sample whose balls outgrow the table is redone with the per-block
//     dense global state (stamped 16-byte words, as sampler.cu), which is also
//     the only path for graphs whose balls are routinely large (grid, C5).
//
// The sigma-weighted backtrack (kadabra.hpp:227-242) is performed by warp 0
// with a 65-bit warp prefix sum over the ascending-neighbour candidates.
#include <cub/block/block_scan.cuh>

#include "device.cuh"
#include "rng.hpp"
#include "sampler.cuh"

namespace adsb {

namespace {

constexpr int kBT = 256;
constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kMetaT = 1u << 31;
constexpr uint32_t kMetaDag = 1u << 30;
constexpr uint32_t kMetaDist = (1u << 30) - 1;
constexpr uint32_t kSmemLevels = 64;

__device__ __forceinline__ bool m_is_t(uint32_t m) { return (m & kMetaT) != 0; }
__device__ __forceinline__ uint32_t m_dist(uint32_t m) { return m & kMetaDist; }

using BlockScan = cub::BlockScan<uint32_t, kBT>;

struct Shared {
    typename BlockScan::TempStorage scan_tmp;
    uint32_t scan[kBT];               // inclusive degree scan of the current chunk
    uint32_t cbase[kBT];              // off(u) - exclusive(u): nbr index = cbase[owner] + e
    uint32_t cslot[kBT];              // store slot of the chunk's frontier vertex
    unsigned long long cval[kBT];     // per-vertex payload (sigma of u)
    unsigned long long item;
    unsigned long long degsum;
    uint32_t s_cnt, t_cnt;            // queue fill: s-side from 0 up, t-side from the top down
    uint32_t inserted;                // hash reservations this sample
    uint32_t overflow;
    uint32_t tlev_small[kSmemLevels]; // t-level boundaries (shared-memory store)
};

// ---------------------------------------------------------------------------
// Stores: where a sample's per-vertex state lives
// ---------------------------------------------------------------------------

// Shared-memory open-addressing table: km = key << 32 | meta, sig = sigma.
// Empty slots have key 0xFFFFFFFF and sigma 0 (sigma is zeroed with the key,
// so concurrent claimers and adders never race on initialisation).
struct SmemStore {
    unsigned long long* km;
    unsigned long long* sig;
    uint32_t* qv;      // queue: vertex ids
    uint32_t* qdeg;    // queue: degrees (for the side-balancing heuristic)
    uint32_t* tlev;
    uint32_t mask;
    uint32_t shift;
    uint32_t qcap;
    uint32_t limit;    // max insertions (<= capacity/2 keeps probing short and finite)
    uint32_t level_cap;
    Shared* sh;

    __device__ uint32_t home(uint32_t v) const {
        return static_cast<uint32_t>((static_cast<unsigned long long>(v) * 0x9E3779B97F4A7C15ull) >> shift) & mask;
    }
    __device__ void begin(uint32_t tid) {
        for (uint32_t i = tid; i <= mask; i += kBT) {
            km[i] = ~0ull;
            sig[i] = 0ull;
        }
    }
    __device__ uint32_t find(uint32_t v, uint32_t& meta) const {
        uint32_t h = home(v);
        for (;;) {
            const unsigned long long x = km[h];
            const uint32_t k = static_cast<uint32_t>(x >> 32);
            if (k == v) {
                meta = static_cast<uint32_t>(x);
                return h;
            }
            if (k == kEmptyKey) return kNone;
            h = (h + 1) & mask;
        }
    }
    // returns the slot (kNone on overflow); inserted tells whether this call created it
    __device__ uint32_t claim(uint32_t v, uint32_t new_meta, bool& inserted, uint32_t& meta) {
        inserted = false;
        uint32_t h = home(v);
        bool reserved = false;
        for (;;) {
            unsigned long long x = km[h];
            uint32_t k = static_cast<uint32_t>(x >> 32);
            if (k == v) {
                meta = static_cast<uint32_t>(x);
                return h;
            }
            if (k == kEmptyKey) {
                if (!reserved) {
                    if (atomicAdd(&sh->inserted, 1u) >= limit) {
                        sh->overflow = 1;
                        return kNone;
                    }
                    reserved = true;
                }
                const unsigned long long want = (static_cast<unsigned long long>(v) << 32) | new_meta;
                const unsigned long long prev = atomicCAS(&km[h], x, want);
                if (prev == x) {
                    inserted = true;
                    meta = new_meta;
                    return h;
                }
                if (static_cast<uint32_t>(prev >> 32) == v) {
                    meta = static_cast<uint32_t>(prev);
                    return h;
                }
            }
            h = (h + 1) & mask;
        }
    }
    __device__ void zero_sigma(uint32_t) {}
    __device__ void add_sigma(uint32_t slot, unsigned long long x) { atomicAdd(&sig[slot], x); }
    __device__ void set_dag(uint32_t slot) { atomicOr(&km[slot], static_cast<unsigned long long>(kMetaDag)); }
    __device__ unsigned long long sigma(uint32_t slot) const { return sig[slot]; }
    __device__ bool queue_ok(uint32_t s_cnt, uint32_t t_cnt) const { return s_cnt + t_cnt <= qcap; }
    __device__ uint32_t tpos(uint32_t j) const { return qcap - 1 - j; }
};

// Per-block dense global state (stamped with a per-block generation tag).
struct GlobalStore {
    unsigned long long* st;  // 2 words per vertex: (tag << 32 | meta), sigma
    uint32_t* qv;
    uint32_t* qdeg;
    uint32_t* tlev;
    uint32_t tag;
    uint32_t qcap;
    uint32_t level_cap;

    __device__ void begin(uint32_t) {}
    __device__ uint32_t find(uint32_t v, uint32_t& meta) const {
        const unsigned long long x = __ldcg(st + 2ull * v);
        if (static_cast<uint32_t>(x >> 32) != tag) return kNone;
        meta = static_cast<uint32_t>(x);
        return v;
    }
    __device__ uint32_t claim(uint32_t v, uint32_t new_meta, bool& inserted, uint32_t& meta) {
        inserted = false;
        unsigned long long x = __ldcg(st + 2ull * v);
        if (static_cast<uint32_t>(x >> 32) != tag) {
            const unsigned long long want = (static_cast<unsigned long long>(tag) << 32) | new_meta;
            const unsigned long long prev = atomicCAS(st + 2ull * v, x, want);
            if (prev == x) {
                inserted = true;
                meta = new_meta;
                return v;
            }
            x = prev;
        }
        meta = static_cast<uint32_t>(x);
        return v;
    }
    __device__ void zero_sigma(uint32_t slot) { st[2ull * slot + 1] = 0ull; }
    __device__ void add_sigma(uint32_t slot, unsigned long long x) { atomicAdd(st + 2ull * slot + 1, x); }
    __device__ void set_dag(uint32_t slot) { atomicOr(st + 2ull * slot, static_cast<unsigned long long>(kMetaDag)); }
    __device__ unsigned long long sigma(uint32_t slot) const { return __ldcg(st + 2ull * slot + 1); }
    __device__ bool queue_ok(uint32_t, uint32_t) const { return true; }
    __device__ uint32_t tpos(uint32_t j) const { return qcap - 1 - j; }
};

struct Ctx {
    const uint32_t* __restrict__ off;
    const uint32_t* __restrict__ nbrs;
    uint32_t tid;
    uint32_t lane;
    uint32_t warp;
    Shared* sh;
    unsigned long long edges, rebuild_edges, back_edges, verts;
};

// Visit the flattened adjacency of queue entries [lo, hi) (t-side entries when
// t_list). prep(slot) gives the per-vertex payload; body(slot_u, payload, v)
// runs once per adjacency entry. Ends with a block barrier.
template <class Store, class Prep, class Body>
__device__ void for_edges(Ctx& C, Store& S, uint32_t lo, uint32_t hi, bool t_list, unsigned long long& counter,
                          Prep prep, Body body) {
    Shared& sh = *C.sh;
    for (uint32_t base = lo; base < hi; base += kBT) {
        const uint32_t i = base + C.tid;
        uint32_t deg = 0, o = 0, slot = 0;
        unsigned long long val = 0;
        if (i < hi) {
            const uint32_t q = t_list ? S.tpos(i) : i;
            const uint32_t u = S.qv[q];
            o = C.off[u];
            deg = C.off[u + 1] - o;
            uint32_t meta;
            slot = S.find(u, meta);
            val = prep(slot, meta, deg);
        }
        uint32_t incl, total;
        BlockScan(sh.scan_tmp).InclusiveSum(deg, incl, total);
        sh.scan[C.tid] = incl;
        sh.cbase[C.tid] = o - (incl - deg);
        sh.cslot[C.tid] = slot;
        sh.cval[C.tid] = val;
        __syncthreads();
        counter += C.tid == 0 ? total : 0;
        for (uint32_t e = C.tid; e < total; e += kBT) {
            uint32_t l = 0, r = kBT - 1;  // first k with scan[k] > e
            while (l < r) {
                const uint32_t mid = (l + r) >> 1;
                if (sh.scan[mid] > e) r = mid;
                else l = mid + 1;
            }
            const uint32_t v = C.nbrs[sh.cbase[l] + e];
            body(sh.cslot[l], sh.cval[l], v);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ unsigned long long shfl64(unsigned long long x, int src) {
    return __shfl_sync(kFull, x, src);
}

// Result of the BFS phase: distance split d = a + b + 1.
struct Meet {
    uint32_t a, b;
    bool ok;
};

template <class Store>
__device__ Meet bfs(Ctx& C, Store& S, uint32_t s, uint32_t t) {
    Shared& sh = *C.sh;
    if (C.tid == 0) {
        bool ins;
        uint32_t m;
        const uint32_t ss = S.claim(s, 0u, ins, m);
        const uint32_t tt = S.claim(t, kMetaT, ins, m);
        S.zero_sigma(ss);
        S.zero_sigma(tt);
        S.add_sigma(ss, 1ull);
        S.qv[0] = s;
        S.qdeg[0] = C.off[s + 1] - C.off[s];
        S.qv[S.tpos(0)] = t;
        S.qdeg[S.tpos(0)] = C.off[t + 1] - C.off[t];
        S.tlev[0] = 0;
        S.tlev[1] = 1;
        sh.s_cnt = 1;
        sh.t_cnt = 1;
    }
    __syncthreads();
    uint32_t s_lo = 0, s_hi = 1, t_lo = 0, t_hi = 1, a = 0, b = 0;
    unsigned long long deg_s = C.off[s + 1] - C.off[s], deg_t = C.off[t + 1] - C.off[t];
    for (;;) {
        if (deg_s <= deg_t) {
            // ---- s-side level a: probe for the t-ball (meeting level fills sigma of T_b)
            C.verts += C.tid == 0 ? s_hi - s_lo : 0;
            bool met = false;
            for_edges(C, S, s_lo, s_hi, false, C.edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.sigma(slot); },
                      [&](uint32_t, unsigned long long su, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && m_is_t(m) && m_dist(m) == b) {
                              S.add_sigma(sl, su);
                              if (!(m & kMetaDag)) S.set_dag(sl);
                              met = true;
                          }
                      });
            if (__syncthreads_or(met)) return {a, b, true};
            // ---- no meeting: claim level a+1, then accumulate its sigma
            if (C.tid == 0) sh.degsum = 0;
            __syncthreads();
            unsigned long long my_deg = 0;
            const uint32_t meta_new = a + 1;
            for_edges(C, S, s_lo, s_hi, false, C.edges,
                      [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                      [&](uint32_t, unsigned long long, uint32_t v) {
                          bool ins;
                          uint32_t m;
                          const uint32_t sl = S.claim(v, meta_new, ins, m);
                          if (ins) {
                              S.zero_sigma(sl);
                              const uint32_t pos = atomicAdd(&sh.s_cnt, 1u);
                              const uint32_t dg = C.off[v + 1] - C.off[v];
                              if (S.queue_ok(pos + 1, sh.t_cnt)) {
                                  S.qv[pos] = v;
                                  S.qdeg[pos] = dg;
                              } else {
                                  sh.overflow = 1;
                              }
                              my_deg += dg;
                          }
                      });
            if (my_deg) atomicAdd(&sh.degsum, my_deg);
            if (sh.overflow) return {a, b, false};
            for_edges(C, S, s_lo, s_hi, false, C.edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.sigma(slot); },
                      [&](uint32_t, unsigned long long su, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && !m_is_t(m) && m_dist(m) == a + 1) S.add_sigma(sl, su);
                      });
            s_lo = s_hi;
            s_hi = sh.s_cnt;
            deg_s = sh.degsum;
            a += 1;
            if (s_lo == s_hi) return {a, b, false};
        } else {
            // ---- t-side level b: probe for the s-ball
            C.verts += C.tid == 0 ? t_hi - t_lo : 0;
            bool met = false;
            for_edges(C, S, t_lo, t_hi, true, C.edges,
                      [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                      [&](uint32_t su_slot, unsigned long long, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && !m_is_t(m) && m_dist(m) == a) {
                              S.add_sigma(su_slot, S.sigma(sl));
                              S.set_dag(su_slot);
                              met = true;
                          }
                      });
            if (__syncthreads_or(met)) return {a, b, true};
            if (C.tid == 0) sh.degsum = 0;
            __syncthreads();
            unsigned long long my_deg = 0;
            const uint32_t meta_new = kMetaT | (b + 1);
            for_edges(C, S, t_lo, t_hi, true, C.edges,
                      [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                      [&](uint32_t, unsigned long long, uint32_t v) {
                          bool ins;
                          uint32_t m;
                          const uint32_t sl = S.claim(v, meta_new, ins, m);
                          if (ins) {
                              S.zero_sigma(sl);
                              const uint32_t j = atomicAdd(&sh.t_cnt, 1u);
                              const uint32_t dg = C.off[v + 1] - C.off[v];
                              if (S.queue_ok(sh.s_cnt, j + 1)) {
                                  S.qv[S.tpos(j)] = v;
                                  S.qdeg[S.tpos(j)] = dg;
                              } else {
                                  sh.overflow = 1;
                              }
                              my_deg += dg;
                          }
                      });
            if (my_deg) atomicAdd(&sh.degsum, my_deg);
            __syncthreads();
            if (sh.overflow) return {a, b, false};
            t_lo = t_hi;
            t_hi = sh.t_cnt;
            deg_t = sh.degsum;
            b += 1;
            if (b + 2 > S.level_cap) {
                if (C.tid == 0) sh.overflow = 1;
                return {a, b, false};
            }
            if (C.tid == 0) S.tlev[b + 1] = t_hi;
            __syncthreads();
            if (t_lo == t_hi) return {a, b, false};
        }
    }
}

// sigma_s on the t-side DAG layers (pull; see sampler.cu rebuild_level)
template <class Store>
__device__ void rebuild(Ctx& C, Store& S, uint32_t b) {
    for (uint32_t k = b; k >= 1; --k) {
        for_edges(C, S, S.tlev[k - 1], S.tlev[k], true, C.rebuild_edges,
                  [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                  [&](uint32_t w_slot, unsigned long long, uint32_t v) {
                      uint32_t m;
                      const uint32_t sl = S.find(v, m);
                      if (sl != kNone && m_is_t(m) && m_dist(m) == k && (m & kMetaDag)) {
                          S.add_sigma(w_slot, S.sigma(sl));
                          S.set_dag(w_slot);
                      }
                  });
    }
}

// Backtrack by warp 0 (kadabra.hpp:227-242). Returns false on an inconsistent
// state (every predecessor sigma wrapped to 0), which the reference leaves
// undefined.
template <bool kDet, class Store>
__device__ bool backtrack(Ctx& C, Store& S, const SamplerParams& p, SplitMix64& rng, uint32_t t, Meet mt,
                          uint32_t frame_local) {
    const uint32_t d = mt.a + mt.b + 1;
    if (d < 2) return true;
    uint64_t ev_pos = 0;
    if (kDet) {
        if (C.lane == 0) ev_pos = atomicAdd(p.ev_cursor, static_cast<unsigned long long>(d - 1));
        ev_pos = shfl64(ev_pos, 0);
    }
    uint32_t cur = t, cmeta = 0;
    uint32_t cslot = S.find(t, cmeta);
    unsigned long long csig = S.sigma(cslot);
    uint32_t ds_cur = d;
    for (uint32_t step = 0; ds_cur > 1; ++step) {
        unsigned long long r = rng.next_below(csig);
        bool want_t;
        uint32_t want_dist;
        if (m_is_t(cmeta)) {
            const uint32_t k = m_dist(cmeta);
            want_t = k < mt.b;
            want_dist = k < mt.b ? k + 1 : mt.a;
        } else {
            want_t = false;
            want_dist = m_dist(cmeta) - 1;
        }
        const uint32_t beg = C.off[cur], end = C.off[cur + 1];
        uint32_t chosen = kNone, chosen_meta = 0;
        unsigned long long chosen_sig = 0;
        for (uint32_t base = beg; base < end; base += 32) {
            const uint32_t i = base + C.lane;
            uint32_t q = 0, m = 0;
            unsigned long long val = 0;
            if (i < end) {
                q = C.nbrs[i];
                const uint32_t sl = S.find(q, m);
                if (sl != kNone && m_is_t(m) == want_t && m_dist(m) == want_dist && (!want_t || (m & kMetaDag)))
                    val = S.sigma(sl);
            }
            C.back_edges += C.lane == 0 ? min(32u, end - base) : 0;
            unsigned long long lo = val;
            uint32_t hi = 0;
#pragma unroll
            for (int dd = 1; dd < 32; dd <<= 1) {
                const unsigned long long olo = __shfl_up_sync(kFull, lo, dd);
                const uint32_t ohi = __shfl_up_sync(kFull, hi, dd);
                if (C.lane >= static_cast<uint32_t>(dd)) {
                    const unsigned long long nlo = lo + olo;
                    hi += ohi + (nlo < lo ? 1u : 0u);
                    lo = nlo;
                }
            }
            const uint32_t ball = __ballot_sync(kFull, hi > 0 || r < lo);
            if (ball) {
                const int f = __ffs(ball) - 1;
                chosen = __shfl_sync(kFull, q, f);
                chosen_meta = __shfl_sync(kFull, m, f);
                chosen_sig = shfl64(val, f);
                break;
            }
            r -= shfl64(lo, 31);
        }
        if (chosen == kNone) return false;
        if (C.lane == 0) {
            if (kDet) {
                if (ev_pos + step < p.ev_cap)
                    p.events[ev_pos + step] = (static_cast<unsigned long long>(chosen) << 32) | frame_local;
            } else {
                atomicAdd(p.counts + chosen, 1u);
            }
        }
        cur = chosen;
        cmeta = chosen_meta;
        csig = chosen_sig;
        ds_cur = m_is_t(cmeta) ? d - m_dist(cmeta) : m_dist(cmeta);
    }
    return true;
}

// Whole sample with one store. Returns 0 ok, 1 overflow (redo with the global
// store), 2 inconsistent state.
template <bool kDet, class Store>
__device__ int run_sample(Ctx& C, Store& S, const SamplerParams& p, SplitMix64& rng, uint32_t s, uint32_t t,
                          uint32_t frame_local) {
    Shared& sh = *C.sh;
    S.begin(C.tid);
    if (C.tid == 0) {
        sh.inserted = 0;
        sh.overflow = 0;
    }
    __syncthreads();
    const Meet mt = bfs(C, S, s, t);
    if (!mt.ok) return sh.overflow ? 1 : 2;
    rebuild(C, S, mt.b);
    int rc = 0;
    if (C.warp == 0) rc = backtrack<kDet>(C, S, p, rng, t, mt, frame_local) ? 0 : 2;
    rc = __syncthreads_or(rc) ? 2 : 0;
    return rc;
}

template <bool kDet>
__global__ void __launch_bounds__(kBT) sampler_cta_kernel(SamplerParams p) {
    extern __shared__ unsigned long long dyn[];
    __shared__ Shared sh;
    Ctx C;
    C.off = p.off;
    C.nbrs = p.nbrs;
    C.tid = threadIdx.x;
    C.lane = threadIdx.x & 31;
    C.warp = threadIdx.x >> 5;
    C.sh = &sh;
    C.edges = C.rebuild_edges = C.back_edges = C.verts = 0;
    const uint32_t slot = blockIdx.x;

    SmemStore sm;
    const uint32_t H = p.hash_cap;
    sm.km = dyn;
    sm.sig = dyn + H;
    sm.qcap = H / 2;
    sm.qv = reinterpret_cast<uint32_t*>(dyn + 2 * H);
    sm.qdeg = sm.qv + sm.qcap;
    sm.tlev = sh.tlev_small;
    sm.mask = H - 1;
    sm.shift = 64 - (31 - __clz(H));
    sm.limit = H / 2;
    sm.level_cap = kSmemLevels;
    sm.sh = &sh;

    GlobalStore gs;
    gs.st = p.state + 2ull * p.n * slot;
    gs.qv = p.queue + static_cast<size_t>(p.n) * slot;
    gs.qdeg = reinterpret_cast<uint32_t*>(p.qrange + static_cast<size_t>(p.n) * slot);
    gs.tlev = p.tlev + static_cast<size_t>(p.level_cap) * slot;
    gs.tag = p.slot_tag[slot];
    gs.qcap = p.n;
    gs.level_cap = p.level_cap;

    unsigned long long samples = 0, fallbacks = 0, errors = 0;
    for (;;) {
        if (C.tid == 0) sh.item = atomicAdd(p.ticket, 1ull);
        __syncthreads();
        const unsigned long long item = sh.item;
        __syncthreads();
        if (item >= p.num_items) break;
        const uint64_t local = item * p.world + p.rank;
        SplitMix64 rng(reseed(p.seed, p.first + local));
        for (uint64_t i = 0; i < p.spf; ++i) {
            ++samples;
            const uint32_t s = static_cast<uint32_t>(rng.next_below(p.n));
            uint32_t t = static_cast<uint32_t>(rng.next_below(p.n - 1));
            if (t >= s) ++t;
            if (__ldg(p.label + s) != __ldg(p.label + t)) continue;
            int rc = 1;
            if (p.use_smem) rc = run_sample<kDet>(C, sm, p, rng, s, t, static_cast<uint32_t>(local));
            if (rc == 1) {
                fallbacks += p.use_smem ? 1 : 0;
                gs.tag += 1;
                rc = run_sample<kDet>(C, gs, p, rng, s, t, static_cast<uint32_t>(local));
            }
            if (rc != 0) ++errors;
        }
    }
    // per-thread counters: reduce across the block once
    atomicAdd(p.stats + kStatEdges, C.edges + C.rebuild_edges + C.back_edges);
    atomicAdd(p.stats + kStatRebuildEdges, C.rebuild_edges);
    atomicAdd(p.stats + kStatBacktrackEdges, C.back_edges);
    atomicAdd(p.stats + kStatVertices, C.verts);
    if (C.tid == 0) {
        p.slot_tag[slot] = gs.tag;
        atomicAdd(p.stats + kStatSamples, samples);
        atomicAdd(p.stats + kStatFallbacks, fallbacks);
        if (errors) atomicAdd(p.stats + kStatErrors, errors);
    }
}

}  // namespace

size_t sampler_cta_smem_bytes(uint32_t hash_cap) {
    return static_cast<size_t>(hash_cap) * 16 + static_cast<size_t>(hash_cap / 2) * 8;
}

int sampler_cta_blocks_per_sm(uint32_t hash_cap) {
    const size_t dyn = sampler_cta_smem_bytes(hash_cap);
    static bool configured = false;
    if (!configured) {
        ADSB_CUDA(cudaFuncSetAttribute(sampler_cta_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        ADSB_CUDA(cudaFuncSetAttribute(sampler_cta_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    int blocks = 0;
    ADSB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, sampler_cta_kernel<true>, kBT, dyn));
    return blocks;
}

void launch_sampler_cta(bool deterministic, const SamplerParams& p, cudaStream_t stream) {
    const size_t dyn = sampler_cta_smem_bytes(p.hash_cap);
    sampler_cta_blocks_per_sm(p.hash_cap);  // sets the dynamic smem attribute once
    if (deterministic)
        sampler_cta_kernel<true><<<p.slots, kBT, dyn, stream>>>(p);
    else
        sampler_cta_kernel<false><<<p.slots, kBT, dyn, stream>>>(p);
    ADSB_CUDA(cudaGetLastError());
}

}  // namespace adsb
