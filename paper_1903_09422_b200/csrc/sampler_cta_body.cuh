// sampler_cta_body.cuh — body of the block-team sampler, included once per
// block size by sampler_cta.cu inside a namespace that defines kBT.
// (Not a standalone header.)


constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr uint32_t kMaxHubs = 32;
#ifndef ADSB_HUB_PROBE
#define ADSB_HUB_PROBE 1
#endif
#ifndef ADSB_PROBE_PREFETCH
#define ADSB_PROBE_PREFETCH 1
#endif
#ifndef ADSB_VEC_FALLBACK
#define ADSB_VEC_FALLBACK 1  // vector kernels: fallback samples read adjacency as 16-byte vectors too
#endif
#ifndef ADSB_CLAIM_PREFETCH
#define ADSB_CLAIM_PREFETCH 1  // ... and prefetch a vector's four state words in claim passes
#endif
constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr uint32_t kEmptyKey = 0xFFFFFFFFu;
constexpr uint32_t kMetaT = 1u << 31;
constexpr uint32_t kMetaDag = 1u << 30;
constexpr uint32_t kMetaDist = (1u << 30) - 1;
constexpr uint32_t kSmemLevels = 64;
constexpr uint32_t kSmallStep = 64;  // backtrack steps with deg(cur) <= this run on warp 0 alone

__device__ __forceinline__ bool m_is_t(uint32_t m) { return (m & kMetaT) != 0; }
__device__ __forceinline__ uint32_t m_dist(uint32_t m) { return m & kMetaDist; }


struct Shared {
    uint32_t wtot[kBT / 32];          // block scan: per-warp totals
    uint32_t scan[kBT];               // inclusive degree scan of the current chunk
    uint32_t cbase[kBT];              // off(u) - exclusive(u): nbr index = cbase[owner] + e
    uint32_t cslot[kBT];              // store slot of the chunk's frontier vertex
    unsigned long long cval[kBT];     // per-vertex payload (sigma of u)
    unsigned long long item;
    unsigned long long tick[2];       // next work item, double-buffered by loop parity
    uint32_t tflag[2];                // fused: the previous sample completed its epoch
    unsigned long long done_old;      // thread 0 (fused): Done counter before the last sample's increment
    unsigned long long spare_tick;    // thread 0 (fused, ADSB_TICKET_PAIR): second ticket of the last fetch
    // block statistics: adjacency counters per warp (each written only by its
    // lane 0 with plain adds: no 64-bit shared atomics, which are CAS loops on sm_100)
    unsigned long long st_edges[kBT / 32], st_rebuild[kBT / 32], st_back[kBT / 32];
    unsigned long long st_verts, st_degen;  // thread 0 adds
    unsigned long long n_samples, n_fallbacks, n_errors;
    uint32_t g_region, g_tag;         // fallback: borrowed global region and its tag
    uint32_t pending;                 // thread 0 (fused): done_old belongs to an unprocessed completion
    uint32_t recorded, last_d;        // thread 0: increments recorded / last distance (fused audit)
    uint32_t lvl_cnt[3];              // per BFS level (slot = level % 3): vertices claimed,
    uint32_t lvl_deg[3];              //   their adjacency total (< 2^32: u32 offsets),
    uint32_t lvl_ins[3];              //   hash reservations (shared-memory store),
    uint32_t lvl_met[3];              //   whether the frontiers met (any thread sets it)
    uint32_t s_cnt, t_cnt;            // queue fill: s-side from 0 up, t-side from the top down
    uint32_t dag_cnt;                 // push rebuild: fill of the t-side DAG list
    uint32_t overflow;
    uint32_t tlev_small[kSmemLevels]; // t-level boundaries (shared-memory store)
    uint32_t slev_small[kSmemLevels]; // s-level boundaries (shared-memory store)
    unsigned long long wlo[kBT / 32]; // backtrack: per-warp 65-bit candidate sums
    uint32_t whi[kBT / 32];
    uint32_t first;                   // backtrack: first thread whose prefix exceeds r
    uint32_t ch, chm;                 // backtrack: chosen predecessor and its meta
    unsigned long long chs;           // backtrack: chosen predecessor's sigma
    uint32_t bch, bchm;               // backtrack, block rounds: chosen predecessor and meta
    unsigned long long bchs;          //   and its sigma
    unsigned long long ev_pos;
    unsigned long long fold_epoch;    // fused mode: epoch being folded
    uint32_t fold_len, fold_max, flag;
    // probe passes: frontier hubs searched against the other side's level list
    // instead of scanned (for_edges_tok, kMaxHubs per chunk)
    uint32_t n_hub[2];
    uint32_t hub_o[kMaxHubs], hub_e[kMaxHubs], hub_slot[kMaxHubs];
    uint32_t hub_tree[kMaxHubs];      // word offset of the hub's search tree (kNone: none)
    unsigned long long hub_val[kMaxHubs];
    const uint32_t* hub_ref;          // SamplerParams::hub_ref / hub_keys (nullptr: no trees)
    const uint32_t* hub_keys;
};

// ---------------------------------------------------------------------------
// Stores: where a sample's per-vertex state lives
// ---------------------------------------------------------------------------

// Shared-memory open-addressing table: km = key << 32 | meta, sig = sigma.
// Empty slots have key 0xFFFFFFFF and sigma 0 (sigma is zeroed with the key,
// so concurrent claimers and adders never race on initialisation).
template <bool kVec>
struct SmemStoreT {
    static constexpr uint32_t kLoadBatch = ADSB_LOAD_BATCH;
    static constexpr bool kVec4 = kVec;  // flattened adjacency read as 16-byte vectors
    static constexpr bool kTrees = kVec; // hub searches go through the search trees (hub_index.cuh)
    // vectorised reads: each chunk vertex's adjacency range [off(u), off(u+1))
    // as lo[kBT] then hi[kBT], in dynamic shared memory (vector kernels only:
    // a larger static block would shrink the L1 the scalar kernels prefetch into)
    uint32_t* crange;
    // Entry = one u32: (vertex + 1) << 8 | meta8 (bit 7 t-side, bit 6 DAG,
    // bits 0-5 distance); 0 = empty. Needs n < 2^24 - 1 and distances <= 63
    // (larger graphs use the global store; a deeper level overflows to it).
    // Sigma sits in its own u64 array: 12 B per entry plus 2 B of queue.
    static constexpr uint32_t kMaxDist = 62;  // levels a+1, b+1 stay <= 63
    unsigned long long* sig;
    uint32_t* km;
    uint32_t* qv;      // queue: vertex ids
    uint32_t* tlev;
    uint32_t* slev;
    uint32_t cap;      // table entries (any size: slots come from a multiply-high)
    uint32_t qcap;
    uint32_t limit;    // max insertions (<= capacity/2 keeps probing short and finite)
    uint32_t level_cap;
    Shared* sh;
    uint32_t* ins_ctr;  // this level's reservation counter (Shared::lvl_ins slot)
    uint32_t ins_base;  // reservations made before this level (same in every thread)
#if ADSB_SMEM_FILTER
    // Membership filter of the claimed vertices (kFbBits bits, one hash): a
    // probe whose bit is clear skips the table walk. The meeting level's
    // probes, the bulk of a sample's adjacency, almost all miss.
    uint32_t* fb;
    static constexpr uint32_t kFbLog = 15, kFbWords = (1u << kFbLog) / 32;
    static __device__ __forceinline__ uint32_t fbh(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - kFbLog); }
#endif

    static __device__ __forceinline__ uint32_t decode(uint32_t w) {
        return ((w & 0x80u) ? kMetaT : 0u) | ((w & 0x40u) ? kMetaDag : 0u) | (w & 0x3Fu);
    }
    static __device__ __forceinline__ uint32_t encode(uint32_t v, uint32_t meta) {
        return ((v + 1u) << 8) | ((meta & kMetaT) ? 0x80u : 0u) | (m_dist(meta) & 0x3Fu);
    }
    __device__ void set_level(uint32_t* ctr, uint32_t base) {
        ins_ctr = ctr;
        ins_base = base;
    }
    __device__ uint32_t home(uint32_t v) const {
        return __umulhi(v * 0x9E3779B1u, cap);  // Fibonacci hash scaled onto [0, cap)
    }
    __device__ void clear_all(uint32_t tid) {
        for (uint32_t i = tid; i < cap; i += kBT) {
            km[i] = 0u;
            sig[i] = 0ull;
        }
#if ADSB_SMEM_FILTER
        for (uint32_t i = tid; i < kFbWords; i += kBT) fb[i] = 0u;
#endif
    }
    __device__ void begin(uint32_t tid) {
#ifdef ADSB_DEBUG_CHECKS
        for (uint32_t i = tid; i < cap; i += kBT)
            ADSB_DCHECK(km[i] == 0u && sig[i] == 0ull, "hash table not clean at sample start");
#endif
    }
    // Reset exactly the slots this sample inserted (the queue lists them) so
    // the next sample starts from an empty table without touching all of it.
    template <class CtxT>
    __device__ void end(CtxT& C, Shared& s) {
        __syncthreads();
        const uint32_t ns = min(s.s_cnt, qcap), nt = min(s.t_cnt, qcap);
        if (s.overflow) {
            clear_all(C.tid);
        } else {
            // pass 1 resolves every slot (and zeroes sigma) while the table is
            // intact; pass 2 empties the keys without further probing
            for (uint32_t i = C.tid; i < ns + nt; i += kBT) {
                const uint32_t q = i < ns ? i : tpos(i - ns);
                uint32_t m;
                const uint32_t h = find(qv[q], m);
                if (h != kNone) sig[h] = 0ull;
                qv[q] = h;
            }
            __syncthreads();
            for (uint32_t i = C.tid; i < ns + nt; i += kBT) {
                const uint32_t h = qv[i < ns ? i : tpos(i - ns)];
                if (h != kNone) km[h] = 0u;
            }
#if ADSB_SMEM_FILTER
            for (uint32_t i = C.tid; i < kFbWords; i += kBT) fb[i] = 0u;
#endif
        }
        __syncthreads();
    }
    __device__ uint32_t find(uint32_t v, uint32_t& meta) const {
#if ADSB_SMEM_FILTER
        {
            const uint32_t f = fbh(v);
            if (!(fb[f >> 5] & (1u << (f & 31)))) return kNone;
        }
#endif
        const uint32_t key = v + 1u;
        uint32_t h = home(v);
        for (;;) {
            const uint32_t w = km[h];
            if ((w >> 8) == key) {
                meta = decode(w);
                return h;
            }
            if (w == 0u) return kNone;
            h = h + 1 < cap ? h + 1 : 0u;
        }
    }
    // returns the slot (kNone on overflow); inserted tells whether this call
    // created it. kReserve = false: the caller guarantees capacity (room_for),
    // so no reservation counter is touched.
    template <bool kReserve = true>
    __device__ uint32_t claim(uint32_t v, uint32_t new_meta, bool& inserted, uint32_t& meta) {
        inserted = false;
        meta = ~0u;  // on overflow: matches no side/level test
        const uint32_t key = v + 1u;
        uint32_t h = home(v);
        bool reserved = !kReserve;
        for (;;) {
            const uint32_t w = km[h];
            if ((w >> 8) == key) {
                meta = decode(w);
                return h;
            }
            if (w == 0u) {
                if (!reserved) {
                    if (atomicAdd(ins_ctr, 1u) + ins_base >= limit) {
                        sh->overflow = 1;
                        return kNone;
                    }
                    reserved = true;
                }
                const uint32_t prev = atomicCAS(&km[h], 0u, encode(v, new_meta));
                if (prev == 0u) {
                    inserted = true;
                    meta = new_meta;
#if ADSB_SMEM_FILTER
                    const uint32_t f = fbh(v);
                    atomicOr(fb + (f >> 5), 1u << (f & 31));
#endif
                    return h;
                }
                if ((prev >> 8) == key) {
                    meta = decode(prev);
                    return h;
                }
            }
            h = h + 1 < cap ? h + 1 : 0u;
        }
    }
    __device__ static constexpr bool pre_zeroed() { return true; }  // claim and sigma accumulation share one pass
    static constexpr bool kSpeculativeClaims = false;  // meeting-level claims would overflow the table
    __device__ void zero_sigma(uint32_t) {}
    // 64-bit shared-memory atomics are CAS loops on sm_100; sigma (mod 2^64)
    // is added as two native 32-bit atomics with the carry of the low word
    // (each wrap of the low word is seen by exactly one adder). Sigma is only
    // read after a barrier, never while adds are in flight.
    __device__ void add_sigma(uint32_t slot, unsigned long long x) {
        uint32_t* w = reinterpret_cast<uint32_t*>(&sig[slot]);
        const uint32_t xl = static_cast<uint32_t>(x), xh = static_cast<uint32_t>(x >> 32);
        uint32_t carry = 0;
        if (xl) {
            const uint32_t old = atomicAdd(w, xl);
            carry = old + xl < old ? 1u : 0u;
        }
        if (xh | carry) atomicAdd(w + 1, xh + carry);
    }
    __device__ void set_dag(uint32_t slot) { atomicOr(&km[slot], 0x40u); }
    __device__ void prefetch(uint32_t) const {}
    static constexpr bool kBatchClaims = false;
    static constexpr bool kSlotIsVertex = false;
    __device__ unsigned long long claim_issue(uint32_t, uint32_t) { return ~0ull; }
    template <bool kReserve = true>
    __device__ uint32_t claim_tok(uint32_t v, uint32_t new_meta, unsigned long long, bool& inserted, uint32_t& meta) {
        return claim<kReserve>(v, new_meta, inserted, meta);
    }
    static constexpr bool kHasDagQueue = false;
    uint32_t* dq = nullptr;
    __device__ bool set_dag_first(uint32_t slot) { return !(atomicOr(&km[slot], 0x40u) & 0x40u); }
    __device__ unsigned long long sigma(uint32_t slot) const { return sig[slot]; }
    __device__ bool queue_ok(uint32_t s_cnt, uint32_t t_cnt) const { return s_cnt + t_cnt <= qcap; }
    __device__ uint32_t tpos(uint32_t j) const { return qcap - 1 - j; }
    // A one-pass (speculative) level is safe when it cannot claim more vertices
    // than the table has left: the level claims at most its adjacency count.
    __device__ bool room_for(unsigned long long edges) const {
        return ins_base < limit && edges <= limit - ins_base;
    }
    // insertions the table still takes after `used`
    __device__ uint32_t table_room(uint32_t used) const { return used < limit ? limit - used : 0u; }
};
using SmemStore = SmemStoreT<false>;

// Per-team dense global state, 2 words per vertex, in one of two layouts
// chosen per graph (SamplerParams::clear_layout; the engine zeroes the arena
// when a graph switches it):
//  * tagged (hub-heavy graphs): word 0 = tag << 32 | meta with a per-sample
//    generation tag, never cleared. A claim loads the word and CASes it
//    against the stale value, so the many edges into an already-claimed hub
//    are plain loads. The claimer zeroes sigma; an s-side level accumulates
//    sigma in a second pass (skipped on the meeting level, the biggest one).
//  * cleared (low-degree graphs, e.g. lattices): word 0 = present << 32 |
//    meta, and a region is all-zero between samples: each sample zeroes the
//    words it claimed (both queue ends) at its end. A claim is ONE CAS
//    against 0 with no load first, and sigma is already zero, so an s-side
//    level claims and accumulates in one pass. Measured on C4: -22% with the
//    push rebuild; on C3/C5 the blind CAS and one-pass sums cost 15-35%
//    (same-address atomics on hubs, sums on the meeting level).
// kU: adjacency loads kept in flight per thread by for_edges.
#ifndef ADSB_BT_PREFETCH
#define ADSB_BT_PREFETCH 0  // backtrack: prefetch the candidates offsets into L1 (measured neutral)
#endif
#ifndef ADSB_PF_DIST
#define ADSB_PF_DIST 1  // adjacency prefetch distance (rounds of kBT edges) in for_edges
#endif
#ifndef ADSB_FALLBACK_FILTER
#define ADSB_FALLBACK_FILTER 1
#endif
#ifndef ADSB_SPEC_SIGMA
#define ADSB_SPEC_SIGMA 0  // measured neutral (C4 -0.1%)
#endif
#ifndef ADSB_TICKET_PAIR
#define ADSB_TICKET_PAIR 0
#endif
#ifndef ADSB_LP_MIN_ROUNDS
#define ADSB_LP_MIN_ROUNDS 8  // level_pick only for steps of more than this many kBT-wide rounds
#endif
#ifndef ADSB_LEVEL_PICK
#define ADSB_LEVEL_PICK 1
#endif
#ifndef ADSB_LOWDEG_PREFETCH
#define ADSB_LOWDEG_PREFETCH 1
#endif
#ifndef ADSB_LOWDEG_COUNT
#define ADSB_LOWDEG_COUNT 1
#endif
// 16-byte compare-and-swap on a (meta, sigma) state entry (ATOMG.E.CAS.128).
__device__ __forceinline__ ulonglong2 cas128(unsigned long long* p, ulonglong2 cmp, ulonglong2 val) {
    ulonglong2 old;
    asm volatile(
        "{\n\t.reg .b128 c, n, o;\n\t"
        "mov.b128 c, {%2, %3};\n\t"
        "mov.b128 n, {%4, %5};\n\t"
        "atom.global.cas.b128 o, [%6], c, n;\n\t"
        "mov.b128 {%0, %1}, o;\n\t}"
        : "=l"(old.x), "=l"(old.y)
        : "l"(cmp.x), "l"(cmp.y), "l"(val.x), "l"(val.y), "l"(p)
        : "memory");
    return old;
}
__device__ __forceinline__ ulonglong2 ldcg2(const unsigned long long* p) {
    return __ldcg(reinterpret_cast<const ulonglong2*>(p));
}
template <uint32_t kU, bool kBatch = false, bool kTr = false>
struct GlobalStoreT {
    static constexpr uint32_t kLoadBatch = kU;
    // fallback samples of the vector kernels: 16-byte adjacency reads and hub search trees too
    static constexpr bool kVec4 = kTr && ADSB_VEC_FALLBACK;
    static constexpr bool kTrees = kTr;
    uint32_t* crange;  // vectorised reads: row ranges of the chunk (the dynamic shared memory's tail)
    static constexpr bool kBatchClaims = kBatch;  // global-store-only kernels
    static constexpr bool kSlotIsVertex = true;   // find() returns the vertex as its slot
    static constexpr uint32_t kMaxDist = kMetaDist - 1;
    static constexpr unsigned long long kPresent = 1ull << 32;
    unsigned long long* st;  // 2 words per vertex: (tag or present << 32 | meta), sigma
    uint32_t* qv;
    uint32_t* tlev;
    uint32_t* slev;    // s-level boundaries (backtrack by level list)
    uint32_t* dq;      // t-side DAG lists, level by level (push rebuild)
    uint32_t tag;
    uint32_t qcap;
    uint32_t level_cap;
    bool clear;        // cleared layout (see above)
    // Fallback samples of the shared-memory kernels: a membership filter of
    // the claimed vertices (2^18 bits, one hash) in the idle table memory. A
    // clear bit proves "not claimed", so probes skip the global load, and
    // levels probe before they claim (room_for is false) as with the table:
    // the meeting level, the biggest, then claims nothing.
    uint32_t* filt;
    static constexpr uint32_t kFiltLog = 18;
    __device__ static uint32_t fhash(uint32_t v) { return (v * 0x9E3779B1u) >> (32 - kFiltLog); }
    __device__ void fset(uint32_t v) {
        if (filt) {
            const uint32_t h = fhash(v);
            atomicOr(filt + (h >> 5), 1u << (h & 31));
        }
    }
    __device__ bool fmiss(uint32_t v) const {
        if (!filt) return false;
        const uint32_t h = fhash(v);
        return !(filt[h >> 5] & (1u << (h & 31)));
    }

    __device__ void begin(uint32_t) {}
    // Cleared layout: zero the state of every vertex this sample claimed
    // (both queue ends, meeting-level claims included). The caller's next
    // barrier orders these stores before the region's next claims.
    template <class CtxT>
    __device__ void end(CtxT& C, Shared& s) {
        if (clear) {
            __syncthreads();
            const uint32_t ns = s.s_cnt, nt = s.t_cnt;
            // 4 queue loads in flight per thread, then their 4 stores (the
            // clear is ~6% of a C4 sample: one dependent load per store before)
            for (uint32_t i0 = C.tid; i0 < ns + nt; i0 += 4 * kBT) {
                uint32_t v[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint32_t i = i0 + k * kBT;
                    v[k] = i < ns + nt ? __ldcg(qv + (i < ns ? i : tpos(i - ns))) : kNone;
                }
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if (v[k] != kNone) __stcg(reinterpret_cast<ulonglong2*>(st) + v[k], make_ulonglong2(0ull, 0ull));
            }
            __syncthreads();
        }
    }
    __device__ uint32_t find(uint32_t v, uint32_t& meta) const {
        if (fmiss(v)) return kNone;
        const unsigned long long x = __ldcg(st + 2ull * v);
        if (clear ? x == 0ull : static_cast<uint32_t>(x >> 32) != tag) return kNone;
        meta = static_cast<uint32_t>(x);
        return v;
    }
    template <bool kReserve = true>
    __device__ uint32_t claim(uint32_t v, uint32_t new_meta, bool& inserted, uint32_t& meta) {
        inserted = false;
        if (clear) {
            const unsigned long long prev = atomicCAS(st + 2ull * v, 0ull, kPresent | new_meta);
            inserted = prev == 0ull;
            meta = inserted ? new_meta : static_cast<uint32_t>(prev);
            if (inserted) fset(v);
            return v;
        }
        // tagged: one 16-byte load, then one 16-byte CAS that stamps the word and
        // zeroes sigma together, so adders that see the stamp never race with
        // an initialisation (a losing CAS returns the winner's stamped entry)
        ulonglong2 x = ldcg2(st + 2ull * v);
        while (static_cast<uint32_t>(x.x >> 32) != tag) {
            const unsigned long long want = (static_cast<unsigned long long>(tag) << 32) | new_meta;
            const ulonglong2 prev = cas128(st + 2ull * v, x, make_ulonglong2(want, 0ull));
            if (prev.x == x.x && prev.y == x.y) {
                inserted = true;
                meta = new_meta;
                fset(v);
                return v;
            }
            x = prev;
        }
        meta = static_cast<uint32_t>(x.x);
        return v;
    }
    // Batched low-degree claims: the CAS is issued early (claim_issue) and
    // its old word decoded later (claim_tok); otherwise claim_tok claims.
    __device__ unsigned long long claim_issue(uint32_t v, uint32_t new_meta) {
        if (clear) return atomicCAS(st + 2ull * v, 0ull, kPresent | new_meta);
        return ~0ull;
    }
    template <bool kReserve = true>
    __device__ uint32_t claim_tok(uint32_t v, uint32_t new_meta, unsigned long long tok, bool& inserted,
                                  uint32_t& meta) {
        if (tok == ~0ull) return claim<kReserve>(v, new_meta, inserted, meta);
        inserted = tok == 0ull;
        meta = inserted ? new_meta : static_cast<uint32_t>(tok);
        if (inserted) fset(v);
        return v;
    }
    // Claims and sigma sums share one pass when sigma is zero at the claim: the
    // cleared layout, and the tagged layout of a fallback sample (the 16-byte
    // claim zeroes it). Global-only tagged kernels keep the second pass: their
    // one-pass levels claim speculatively on the meeting level, the biggest,
    // whose sums the second pass skips.
    __device__ bool pre_zeroed() const { return clear || filt != nullptr; }
    static constexpr bool kSpeculativeClaims = true;  // no capacity limit: probe and claim in one pass
    __device__ void zero_sigma(uint32_t) {}  // every claim leaves sigma zero
    __device__ void add_sigma(uint32_t slot, unsigned long long x) { atomicAdd(st + 2ull * slot + 1, x); }
    __device__ void set_dag(uint32_t slot) { atomicOr(st + 2ull * slot, static_cast<unsigned long long>(kMetaDag)); }
    __device__ void prefetch(uint32_t v) const { asm volatile("prefetch.global.L2 [%0];" ::"l"(st + 2ull * v)); }
    static constexpr bool kHasDagQueue = true;
    __device__ bool set_dag_first(uint32_t slot) {
        return !(atomicOr(st + 2ull * slot, static_cast<unsigned long long>(kMetaDag)) & kMetaDag);
    }
    __device__ unsigned long long sigma(uint32_t slot) const { return __ldcg(st + 2ull * slot + 1); }
    __device__ bool queue_ok(uint32_t, uint32_t) const { return true; }
    __device__ uint32_t tpos(uint32_t j) const { return qcap - 1 - j; }
    __device__ bool room_for(unsigned long long) const { return filt == nullptr; }
    __device__ void set_level(uint32_t*, uint32_t) {}
    __device__ uint32_t table_room(uint32_t) const { return 0xFFFFFFFFu; }  // no capacity limit
};

// CSR reads carry an L2 eviction-priority hint: evict_last when the CSR fits
// in a fraction of L2 (SamplerParams::csr_hint = 1), so the per-sample state
// streaming through L2 (C4: ~10 GB per 1k samples) does not evict it.
#ifndef ADSB_POL_HOIST
#define ADSB_POL_HOIST 1  // the L2 policy is created once per kernel, not per CSR load
#endif
__device__ __forceinline__ unsigned long long csr_policy(float frac) {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, %1;" : "=l"(pol) : "f"(frac));
    return pol;
}
__device__ __forceinline__ uint32_t ld_csr_pol(const uint32_t* p, unsigned long long pol) {
    uint32_t v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ uint32_t ld_csr(const uint32_t* p, float frac) { return ld_csr_pol(p, csr_policy(frac)); }
__device__ __forceinline__ uint4 ld_csr4_pol(const uint4* p, unsigned long long pol) {
    uint4 v;
    asm("ld.global.nc.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
        : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
        : "l"(p), "l"(pol));
    return v;
}
struct Ctx {
    const uint32_t* __restrict__ off;
    const uint32_t* __restrict__ nbrs;
    float csr_hint;
#if ADSB_POL_HOIST
    unsigned long long pol;
    __device__ __forceinline__ uint32_t O(size_t i) const { return ld_csr_pol(off + i, pol); }
    __device__ __forceinline__ uint32_t N(size_t i) const { return ld_csr_pol(nbrs + i, pol); }
    // the 16-byte vector holding adjacency entries 4g .. 4g+3 (cudaMalloc aligns nbrs)
    __device__ __forceinline__ uint4 N4(size_t g) const { return ld_csr4_pol(reinterpret_cast<const uint4*>(nbrs) + g, pol); }
#else
    __device__ __forceinline__ uint32_t O(size_t i) const { return ld_csr(off + i, csr_hint); }
    __device__ __forceinline__ uint32_t N(size_t i) const { return ld_csr(nbrs + i, csr_hint); }
    __device__ __forceinline__ uint4 N4(size_t g) const {
        return ld_csr4_pol(reinterpret_cast<const uint4*>(nbrs) + g, csr_policy(csr_hint));
    }
#endif
    uint32_t tid;
    uint32_t lane;
    uint32_t warp;
    uint32_t hub_factor;
    Shared* sh;
    uint32_t n;
    bool low_degree;
};

// Inclusive prefix sum over the block (warp shuffles + per-warp totals, one
// barrier). sh.wtot is rewritten only after the caller's next barrier.
__device__ __forceinline__ uint32_t block_inclusive_sum(Ctx& C, uint32_t x, uint32_t& total) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, x, d);
        if (C.lane >= static_cast<uint32_t>(d)) x += y;
    }
    if (C.lane == 31) C.sh->wtot[C.warp] = x;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (uint32_t w = 0; w < kBT / 32; ++w) {
        const uint32_t t = C.sh->wtot[w];
        pre += w < C.warp ? t : 0u;
        tot += t;
    }
    total = tot;
    return x + pre;
}

// Visit the flattened adjacency of queue entries [lo, hi) (t-side entries when
// t_list). prep(slot) gives the per-vertex payload; body(slot_u, payload, v)
// runs once per adjacency entry. Ends with a block barrier.
// for_edges_tok: issue(v) runs for a low-degree vertex's (up to 4)
// neighbours before any body, and its token is passed to body(.., v, tok):
// claims issue their compare-and-swaps together (ADSB_LOWDEG_BATCH) instead
// of one dependent round trip per neighbour.
#ifndef ADSB_LOWDEG_BATCH
#define ADSB_LOWDEG_BATCH 1
#endif
#ifndef ADSB_LEAN_LOOP
#define ADSB_LEAN_LOOP 0
#endif
constexpr unsigned long long kNoTok = ~0ull;
// Probe passes may pass the other side's last level [l_lo, l_hi) (t-side
// queue entries when l_t): a frontier vertex whose adjacency is much longer
// than that list (deg > |L| log2 deg, SamplerParams::hub_factor) is not scanned; instead every list
// vertex is binary-searched in its ascending adjacency (the same edges, found
// in |L| log deg reads: C5's meeting probes are dominated by a few hubs
// against ~1k-vertex levels). body runs once per found edge, as for scanned ones.
// Position of the first entry >= v in the ascending row [o, e) whose search
// tree starts at `tree` (hub_index.cuh): one 8-key node (one sector) per
// level, then inside one 32-entry block of the row one parallel step over its
// four 8-entry groups and a search inside one group.
__device__ __forceinline__ uint32_t tree_lower_bound(const Ctx& C, const uint32_t* __restrict__ tree, uint32_t o,
                                                     uint32_t e, uint32_t v) {
    if (v > __ldg(tree + 7)) return e;
    uint32_t pos = 0;
    for (int k = static_cast<int>(__ldg(tree)); k >= 0; --k) {
        const uint4* node = reinterpret_cast<const uint4*>(tree + __ldg(tree + 1 + k)) + 2u * pos;
        const uint4 a = __ldg(node), b = __ldg(node + 1);
        const uint32_t c = (a.x < v) + (a.y < v) + (a.z < v) + (a.w < v) + (b.x < v) + (b.y < v) + (b.z < v) + (b.w < v);
        pos = pos * kHubFan + c;  // c <= 7: v <= the row's maximum, so every visited node holds a key >= v
    }
    uint32_t l = o + pos * kHubLeaf, r = min(l + kHubLeaf, e);
    const uint32_t k0 = l + 7 < r ? C.N(l + 7) : 0xFFFFFFFFu;
    const uint32_t k1 = l + 15 < r ? C.N(l + 15) : 0xFFFFFFFFu;
    const uint32_t k2 = l + 23 < r ? C.N(l + 23) : 0xFFFFFFFFu;
    l += 8u * ((k0 < v) + (k1 < v) + (k2 < v));
    r = min(l + 8u, r);
    while (l < r) {
        const uint32_t mid = (l + r) >> 1;
        if (C.N(mid) < v) l = mid + 1;
        else r = mid;
    }
    return l;
}
__device__ __forceinline__ bool hub_search(const Ctx& C, uint32_t o, uint32_t e, uint32_t v) {
    uint32_t l = o, r = e;
    while (l < r) {
        const uint32_t mid = (l + r) >> 1;
        if (C.N(mid) < v) l = mid + 1;
        else r = mid;
    }
    return l < e && C.N(l) == v;
}
__device__ __forceinline__ bool hub_search_tree(const Ctx& C, uint32_t o, uint32_t e, uint32_t v, uint32_t tree) {
    if (tree == kNone) return hub_search(C, o, e, v);
    const uint32_t l = tree_lower_bound(C, C.sh->hub_keys + tree, o, e, v);
    return l < e && C.N(l) == v;
}
// dependent loads of one search in a row of deg entries: log2(deg), or with a
// search tree one node per 3 bits above the 32-entry block, plus the block
__device__ __forceinline__ uint32_t search_cost(uint32_t deg, bool trees) {
    const uint32_t bits = 32u - __clz(deg);
    return trees && hub_has_tree(deg) ? (bits + 4u) / 3u : bits;
}
// adjacency entries one search reads, for the edges_scanned statistic: a
// binary search reads one entry per step; a tree search reads an 8-key node per
// level (copies of row entries), the three group ends of the leaf block and
// three steps inside a group, plus the final comparison
__device__ __forceinline__ uint32_t search_reads(uint32_t deg, bool trees) {
    if (!(trees && hub_has_tree(deg))) return 32u - __clz(deg);
    uint32_t n = (deg + kHubLeaf - 1) / kHubLeaf, levels = 1;
    while (n > kHubFan) {
        n = (n + kHubFan - 1) / kHubFan;
        ++levels;
    }
    return kHubFan * levels + 7u;
}
// factor in quarters: deg > (factor / 4) |L| cost(deg)
__device__ __forceinline__ bool is_hub(uint32_t deg, uint32_t list, uint32_t factor, bool trees = false) {
    return ADSB_HUB_PROBE && list && factor &&
           4ull * deg > static_cast<unsigned long long>(factor) * list * search_cost(deg, trees);
}
// The chunk's hubs against the level list: pair (h, j) per thread, one binary
// search each. The hub list is complete (filled before the chunk's scan barrier).
template <class Store, class Body>
__device__ __forceinline__ void hub_phase(Ctx& C, Store& S, Shared& sh, uint32_t par, uint32_t l_lo, uint32_t l_hi,
                                          bool l_t, Body& body) {
    if (l_hi <= l_lo) return;
    const uint32_t nh = min(sh.n_hub[par], kMaxHubs);
    if (nh == 0) return;
    const uint32_t L = l_hi - l_lo;
    const uint32_t pairs = nh * L;
    for (uint32_t pi = C.tid; pi < pairs; pi += kBT) {
        const uint32_t h = pi / L, j = pi - h * L;
        const uint32_t q = l_lo + j;
        const uint32_t v = S.qv[l_t ? S.tpos(q) : q];
        bool hit;
        if constexpr (Store::kTrees) hit = hub_search_tree(C, sh.hub_o[h], sh.hub_e[h], v, sh.hub_tree[h]);
        else hit = hub_search(C, sh.hub_o[h], sh.hub_e[h], v);
        if (hit) body(sh.hub_slot[h], sh.hub_val[h], v, kNoTok);
    }
}

template <class Store, class Prep, class Issue, class Body>
__device__ void for_edges_tok(Ctx& C, Store& S, uint32_t lo, uint32_t hi, bool t_list, unsigned long long* counter,
                              Prep prep, Issue issue, Body body, uint32_t l_lo = 0, uint32_t l_hi = 0,
                              bool l_t = false, bool touch_all = false) {
    Shared& sh = *C.sh;
    ADSB_PHASE_ADD(6, 1);
    if (C.low_degree) {
        // Low-degree graphs (max degree <= 32, e.g. the grid): one thread per
        // frontier vertex walks its whole adjacency; no scan, no chunk
        // barriers, one barrier per level. Imbalance is bounded by the max degree.
        unsigned long long mine = 0;
#if ADSB_LOWDEG_PREFETCH
        // Software pipeline over this thread's frontier vertices: the next
        // vertex id is loaded and its CSR offsets prefetched while this one is
        // processed, and the state words of this vertex's neighbours are
        // prefetched into L2 before the first claim or probe touches them.
        uint32_t i = lo + C.tid;
        uint32_t u_next = i < hi ? S.qv[t_list ? S.tpos(i) : i] : 0u;
        for (; i < hi; i += kBT) {
            const uint32_t u = u_next;
            const bool more = i + kBT < hi;
            if (more) u_next = S.qv[t_list ? S.tpos(i + kBT) : i + kBT];
            ADSB_DCHECK(u < C.n);
            const uint32_t o = C.O(u), e = C.O(u + 1);
            uint32_t meta;
            const uint32_t slot = S.find(u, meta);
            const unsigned long long val = prep(slot, meta, e - o);
            mine += e - o;
            for (uint32_t j0 = o; j0 < e; j0 += 4) {
                uint32_t vv[4];
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k) vv[k] = j0 + k < e ? C.N(j0 + k) : kNone;
                // batched claims only in the global-store-only kernels (the
                // extra registers would spill in the shared-memory kernels)
                if constexpr (ADSB_LOWDEG_BATCH && Store::kBatchClaims) {
                    unsigned long long tok[4];
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k) tok[k] = vv[k] != kNone ? issue(vv[k]) : kNoTok;
                    if (more && j0 == o) asm volatile("prefetch.global.L2 [%0];" ::"l"(C.off + u_next));
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k)
                        if (vv[k] != kNone) body(slot, val, vv[k], tok[k]);
                } else {
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k)
                        if (vv[k] != kNone) S.prefetch(vv[k]);
                    if (more && j0 == o) asm volatile("prefetch.global.L2 [%0];" ::"l"(C.off + u_next));
#pragma unroll
                    for (uint32_t k = 0; k < 4; ++k)
                        if (vv[k] != kNone) body(slot, val, vv[k], kNoTok);
                }
            }
        }
#else
        for (uint32_t i = lo + C.tid; i < hi; i += kBT) {
            const uint32_t q = t_list ? S.tpos(i) : i;
            const uint32_t u = S.qv[q];
            ADSB_DCHECK(u < C.n);
            const uint32_t o = C.O(u), e = C.O(u + 1);
            uint32_t meta;
            const uint32_t slot = S.find(u, meta);
            const unsigned long long val = prep(slot, meta, e - o);
            mine += e - o;
            for (uint32_t j0 = o; j0 < e; j0 += 4) {
                uint32_t vv[4];
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k) vv[k] = j0 + k < e ? C.N(j0 + k) : kNone;
#pragma unroll
                for (uint32_t k = 0; k < 4; ++k)
                    if (vv[k] != kNone) body(slot, val, vv[k], kNoTok);
            }
        }
#endif
        const uint32_t wm = __reduce_add_sync(kFull, static_cast<uint32_t>(mine));
        if (C.lane == 0 && wm) counter[C.warp] += wm;
        __syncthreads();
        return;
    }
    if (l_hi > l_lo) {  // probe pass with a level list: hub counters start at 0
        if (C.tid == 0) sh.n_hub[0] = sh.n_hub[1] = 0;
        __syncthreads();
    }
    if constexpr (Store::kVec4) {
    // Vectorised flattening: each frontier vertex's adjacency [o, e) is covered
    // by the 16-byte vectors floor(o/4) .. ceil(e/4)-1; the block scans vector
    // counts and thread t takes vectors t, t+kBT, ... of the chunk, so one load
    // brings 4 ids (a hub row: 4 real edges per load; entries of the vector
    // outside [o, e) are skipped). 4x the bytes in flight per load instruction.
    for (uint32_t base = lo; base < hi; base += kBT) {
        ADSB_PHASE_MARK(f0);
        const uint32_t i = base + C.tid;
        uint32_t nv = 0, o = 0, e = 0, slot = 0;
        unsigned long long val = 0;
        const uint32_t par = ((base - lo) / kBT) & 1u;
        if (C.tid == 0) sh.n_hub[par ^ 1u] = 0;
        uint32_t scanned = 0;
        if (i < hi) {
            const uint32_t q = t_list ? S.tpos(i) : i;
            const uint32_t u = S.qv[q];
            ADSB_DCHECK(u < C.n);
            o = C.O(u);
            e = C.O(u + 1);
            nv = e > o ? ((e + 3) >> 2) - (o >> 2) : 0u;
            uint32_t meta;
            slot = S.find(u, meta);
            val = prep(slot, meta, e - o);
            scanned = e - o;
            const bool trees = Store::kTrees && sh.hub_ref != nullptr;
            if (is_hub(e - o, l_hi - l_lo, C.hub_factor, trees)) {
                const uint32_t h = atomicAdd(&sh.n_hub[par], 1u);
                if (h < kMaxHubs) {
                    sh.hub_o[h] = o;
                    sh.hub_e[h] = e;
                    sh.hub_slot[h] = slot;
                    sh.hub_val[h] = val;
                    if constexpr (Store::kTrees)
                        sh.hub_tree[h] = trees && hub_has_tree(e - o) ? __ldg(sh.hub_ref + u) : kNone;
                    nv = 0;
                    scanned = (l_hi - l_lo) * search_reads(e - o, trees);  // searches, not scans
                }
            }
        }
        const uint32_t wdeg = __reduce_add_sync(kFull, scanned);
        if (C.lane == 0 && wdeg) counter[C.warp] += wdeg;
        uint32_t total;
        const uint32_t incl = block_inclusive_sum(C, nv, total);
        sh.scan[C.tid] = incl;
        sh.cbase[C.tid] = (o >> 2) - (incl - nv);
        S.crange[C.tid] = o;
        S.crange[kBT + C.tid] = e;
        sh.cslot[C.tid] = slot;
        sh.cval[C.tid] = val;
        __syncthreads();
        ADSB_PHASE_MARK(f1);
        ADSB_PHASE_ADD(8, f1 - f0);
        ADSB_PHASE_ADD(12, total);
        ADSB_PHASE_ADD(13, 1);
        const uint32_t populated = min(hi - base, static_cast<uint32_t>(kBT));
        uint32_t ow = 0, o_end = 0, o_base = 0, r_lo = 0, r_hi = 0, o_slot = 0;
        unsigned long long o_val = 0;
        bool have = false;
        for (uint32_t j = C.tid; j < total; j += kBT) {
            if (!have || j >= o_end) {
                uint32_t l = have ? ow + 1 : 0, r = populated - 1;
                while (l < r) {
                    const uint32_t mid = (l + r) >> 1;
                    if (sh.scan[mid] > j) r = mid;
                    else l = mid + 1;
                }
                ow = l;
                o_end = sh.scan[ow];
                o_base = sh.cbase[ow];
                r_lo = S.crange[ow];
                r_hi = S.crange[kBT + ow];
                o_slot = sh.cslot[ow];
                o_val = sh.cval[ow];
                have = true;
            }
            const uint32_t g = o_base + j;
            const uint4 x = C.N4(g);
            if (j + ADSB_PF_DIST * kBT < o_end)
                asm volatile("prefetch.global.L1 [%0];" ::"l"(reinterpret_cast<const uint4*>(C.nbrs) + g + ADSB_PF_DIST * kBT));
            const uint32_t e0 = g * 4u;
            // touch_all (claim passes on a global region): every entry's state
            // word is read, so the vector's four go to L2 together before the
            // first is used instead of one dependent HBM round trip each
            if constexpr (Store::kSlotIsVertex && ADSB_CLAIM_PREFETCH) {
                if (touch_all) {
                    if (e0 >= r_lo && e0 < r_hi) S.prefetch(x.x);
                    if (e0 + 1 >= r_lo && e0 + 1 < r_hi) S.prefetch(x.y);
                    if (e0 + 2 >= r_lo && e0 + 2 < r_hi) S.prefetch(x.z);
                    if (e0 + 3 >= r_lo && e0 + 3 < r_hi) S.prefetch(x.w);
                } else if (ADSB_PROBE_PREFETCH && S.filt != nullptr) {
                    // probe passes read the state word only of entries the
                    // membership filter lets through: those go to L2 together
                    if (e0 >= r_lo && e0 < r_hi && !S.fmiss(x.x)) S.prefetch(x.x);
                    if (e0 + 1 >= r_lo && e0 + 1 < r_hi && !S.fmiss(x.y)) S.prefetch(x.y);
                    if (e0 + 2 >= r_lo && e0 + 2 < r_hi && !S.fmiss(x.z)) S.prefetch(x.z);
                    if (e0 + 3 >= r_lo && e0 + 3 < r_hi && !S.fmiss(x.w)) S.prefetch(x.w);
                }
            }
#pragma unroll 1
            for (uint32_t k = 0; k < 4; ++k) {
                const uint32_t idx = e0 + k;
                if (idx < r_lo || idx >= r_hi) continue;
                const uint32_t v = k == 0 ? x.x : k == 1 ? x.y : k == 2 ? x.z : x.w;
                ADSB_DCHECK(v < C.n);
                body(o_slot, o_val, v, kNoTok);
            }
        }
        hub_phase(C, S, sh, par, l_lo, l_hi, l_t, body);
        ADSB_PHASE_MARK(f2);
        __syncthreads();
        ADSB_PHASE_MARK(f3);
        ADSB_PHASE_ADD(9, f2 - f1);
        ADSB_PHASE_ADD(11, f3 - f2);
    }
    } else {
    for (uint32_t base = lo; base < hi; base += kBT) {
        ADSB_PHASE_MARK(f0);
        const uint32_t i = base + C.tid;
        uint32_t deg = 0, o = 0, slot = 0;
        unsigned long long val = 0;
        const uint32_t par = ((base - lo) / kBT) & 1u;
        if (C.tid == 0) sh.n_hub[par ^ 1u] = 0;
        uint32_t hub_reads = 0;
        if (i < hi) {
            const uint32_t q = t_list ? S.tpos(i) : i;
            const uint32_t u = S.qv[q];
            ADSB_DCHECK(u < C.n);
            o = C.O(u);
            deg = C.O(u + 1) - o;
            uint32_t meta;
            slot = S.find(u, meta);
            val = prep(slot, meta, deg);
            const bool trees = Store::kTrees && sh.hub_ref != nullptr;
            if (is_hub(deg, l_hi - l_lo, C.hub_factor, trees)) {
                const uint32_t h = atomicAdd(&sh.n_hub[par], 1u);
                if (h < kMaxHubs) {
                    sh.hub_o[h] = o;
                    sh.hub_e[h] = o + deg;
                    sh.hub_slot[h] = slot;
                    sh.hub_val[h] = val;
                    if constexpr (Store::kTrees)
                        sh.hub_tree[h] = trees && hub_has_tree(deg) ? __ldg(sh.hub_ref + u) : kNone;
                    hub_reads = (l_hi - l_lo) * search_reads(deg, trees);
                    deg = 0;
                }
            }
        }
        {
            const uint32_t wr = __reduce_add_sync(kFull, hub_reads);
            if (C.lane == 0 && wr) counter[C.warp] += wr;
        }
        uint32_t total;
        const uint32_t incl = block_inclusive_sum(C, deg, total);
        sh.scan[C.tid] = incl;
        sh.cbase[C.tid] = o - (incl - deg);
        sh.cslot[C.tid] = slot;
        sh.cval[C.tid] = val;
        __syncthreads();
        ADSB_PHASE_MARK(f1);
        ADSB_PHASE_ADD(8, f1 - f0);
        ADSB_PHASE_ADD(12, total);
        ADSB_PHASE_ADD(13, 1);
        if (C.tid == 0) *counter += total;
        // Owner of edge e = first chunk entry k with scan[k] > e. A thread's
        // edges e, e+kBT, ... have non-decreasing owners, so it keeps the
        // current owner's row in registers and searches again (over the
        // remaining populated entries only) when e passes that owner's end:
        // O(1) per edge inside hub adjacency lists.
        const uint32_t populated = min(hi - base, static_cast<uint32_t>(kBT));
        uint32_t ow = 0, o_end = 0, o_base = 0;
        bool have = false;
        // kBatch adjacency loads in flight per thread before any body runs:
        // all loads are issued into registers first, then one non-unrolled
        // loop runs the body on vv[0] and shifts the batch down (the body is
        // instantiated once: unrolled copies overflow the instruction cache;
        // staging through shared memory would wait on each load in turn).
        // Owner indices pack into one register (8 bits each).
        constexpr uint32_t kBatch = Store::kLoadBatch;
        constexpr uint32_t kOwnerBits = kBT <= 256 ? 8 : 16;
        static_assert(kBT <= 65536 && kBatch * kOwnerBits <= 32, "owner indices pack into 32 bits");
#if ADSB_LEAN_LOOP
        if constexpr (kBatch == 1) {
            // One load per iteration: the owner's row (end, base, slot, payload)
            // stays in registers until the edge index leaves it, so a hub row
            // costs no shared-memory reads per edge.
            uint32_t o_slot = 0;
            unsigned long long o_val = 0;
            for (uint32_t e = C.tid; e < total; e += kBT) {
                if (!have || e >= o_end) {
                    uint32_t l = have ? ow + 1 : 0, r = populated - 1;
                    while (l < r) {
                        const uint32_t mid = (l + r) >> 1;
                        if (sh.scan[mid] > e) r = mid;
                        else l = mid + 1;
                    }
                    ow = l;
                    o_end = sh.scan[ow];
                    o_base = sh.cbase[ow];
                    o_slot = sh.cslot[ow];
                    o_val = sh.cval[ow];
                    have = true;
                }
                const uint32_t v = C.N(o_base + e);
                if (e + ADSB_PF_DIST * kBT < o_end)
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(C.nbrs + o_base + e + ADSB_PF_DIST * kBT));
                ADSB_DCHECK(v < C.n);
                body(o_slot, o_val, v, kNoTok);
            }
        } else
#endif
        for (uint32_t e0 = C.tid; e0 < total; e0 += kBT * kBatch) {
            uint32_t owners = 0, cnt = 0;
            uint32_t vv[kBatch];
#pragma unroll
            for (uint32_t k = 0; k < kBatch; ++k) {
                const uint32_t e = e0 + k * kBT;
                if (e < total) {
                    if (!have || e >= o_end) {
                        uint32_t l = have ? ow + 1 : 0, r = populated - 1;
                        while (l < r) {
                            const uint32_t mid = (l + r) >> 1;
                            if (sh.scan[mid] > e) r = mid;
                            else l = mid + 1;
                        }
                        ow = l;
                        o_end = sh.scan[ow];
                        o_base = sh.cbase[ow];
                        have = true;
                    }
                    vv[k] = C.N(o_base + e);
                    // pull this thread's next adjacency id into L1 while the
                    // body runs (same row: the common case inside hub lists)
                    if (k + 1 == kBatch && e + ADSB_PF_DIST * kBT < o_end)
                        asm volatile("prefetch.global.L1 [%0];" ::"l"(C.nbrs + o_base + e + ADSB_PF_DIST * kBT));
                    owners |= ow << (kOwnerBits * k);
                    cnt = k + 1;
                }
            }
#pragma unroll 1
            for (uint32_t k = 0; k < cnt; ++k) {
                const uint32_t v = vv[0];
                ADSB_DCHECK(v < C.n);
                const uint32_t w = owners & ((1u << kOwnerBits) - 1u);
                owners >>= kOwnerBits;
                body(sh.cslot[w], sh.cval[w], v, kNoTok);
#pragma unroll
                for (uint32_t j = 0; j + 1 < kBatch; ++j) vv[j] = vv[j + 1];
            }
        }
        hub_phase(C, S, sh, par, l_lo, l_hi, l_t, body);
        ADSB_PHASE_MARK(f2);
        __syncthreads();
        ADSB_PHASE_MARK(f3);
        ADSB_PHASE_ADD(9, f2 - f1);
        ADSB_PHASE_ADD(11, f3 - f2);
    }
    }
}

template <class Store, class Prep, class Body>
__device__ __forceinline__ void for_edges(Ctx& C, Store& S, uint32_t lo, uint32_t hi, bool t_list,
                                          unsigned long long* counter, Prep prep, Body body, uint32_t l_lo = 0,
                                          uint32_t l_hi = 0, bool l_t = false, bool touch_all = false) {
    for_edges_tok(C, S, lo, hi, t_list, counter, prep, [](uint32_t) { return kNoTok; },
                  [&](uint32_t su, unsigned long long val, uint32_t v, unsigned long long) { body(su, val, v); },
                  l_lo, l_hi, l_t, touch_all);
}

__device__ __forceinline__ unsigned long long shfl64(unsigned long long x, int src) {
    return __shfl_sync(kFull, x, src);
}

// Next positions of a per-level counter for the converged lanes of a warp:
// one shared atomic per group instead of one per lane (the counter is the
// same address for the whole block).
__device__ __forceinline__ uint32_t aggregated_inc(uint32_t* ctr) {
    namespace cg = cooperative_groups;
    const cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(ctr, g.size());
    return g.shfl(base, 0) + g.thread_rank();
}

// One shared atomic per warp for the level's adjacency total.
__device__ __forceinline__ void add_degsum(Ctx& C, uint32_t my_deg, uint32_t slot) {
    const uint32_t w = __reduce_add_sync(kFull, my_deg);
    if (C.lane == 0 && w) atomicAdd(&C.sh->lvl_deg[slot], w);
}

// Adjacency total of queue entries [lo, hi) (a newly claimed level), for the
// side-balancing choice. One parallel pass after the level's barrier: the
// offset loads overlap (4 in flight per thread) instead of stalling each claim.
template <class Store>
__device__ uint32_t level_degrees(Ctx& C, Store& S, uint32_t lo, uint32_t hi, bool t_list, uint32_t slot) {
    ADSB_PHASE_MARK(ld0);
    uint32_t my = 0;
    for (uint32_t i0 = lo + C.tid; i0 < hi; i0 += 4 * kBT) {
        uint32_t v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t i = i0 + k * kBT;
            v[k] = i < hi ? S.qv[t_list ? S.tpos(i) : i] : kNone;
        }
        uint32_t lo_off[4], hi_off[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            lo_off[k] = v[k] != kNone ? C.O(v[k]) : 0u;
            hi_off[k] = v[k] != kNone ? C.O(v[k] + 1) : 0u;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) my += hi_off[k] - lo_off[k];
    }
    add_degsum(C, my, slot);
    __syncthreads();
    ADSB_PHASE_ADD(10, clock64() - ld0);
    return C.sh->lvl_deg[slot];
}

// Result of the BFS phase: distance split d = a + b + 1.
struct Meet {
    uint32_t a, b;
    int status;  // 0 met, 1 store overflow (redo on the global store), 2 inconsistent,
                 // 3 table full at a claim pass (continue on the global store from BfsState)
};

// Loop state of bfs() between levels: what a sample carries from the
// shared-memory table to a global region when the table fills up at a claim
// pass (the completed levels are copied; that level's claims are redone).
struct BfsState {
    uint32_t s_lo, s_hi, t_lo, t_hi, a, b, used;
    unsigned long long deg_s, deg_t;
};

#ifndef ADSB_MIGRATE
#define ADSB_MIGRATE 1
#endif
#ifndef ADSB_PREDICT_QUARTERS
#define ADSB_PREDICT_QUARTERS 4  // migrate before a claim pass over more than this / 4 x the table's room (0: never)
#endif

template <class Store>
__device__ Meet bfs(Ctx& C, Store& S, uint32_t s, uint32_t t, BfsState* io = nullptr) {
    Shared& sh = *C.sh;
    // io != nullptr on entry with io->used == ~0u: resume a migrated sample at
    // the claim pass of its current level (the probe found no meeting there);
    // on a claim-pass overflow of the table the state is written to io.
    const bool resume = io != nullptr && io->used == ~0u;
    // Level L = a + b uses counter slot L % 3; thread 0 zeroes slot (L+1) % 3
    // as level L starts: every thread read that slot (as level L-2's) before
    // level L-1's barriers, and level L+1 writes it only after level L's.
    // So a level needs no barrier of its own before it starts claiming.
    S.set_level(&sh.lvl_ins[2], 0);
    if (C.tid == 0) {
        for (int i = 0; i < 3; ++i) sh.lvl_cnt[i] = sh.lvl_deg[i] = sh.lvl_ins[i] = sh.lvl_met[i] = 0;
    }
    if (!resume && C.tid == 0) {
        bool ins;
        uint32_t m;
        const uint32_t ss = S.claim(s, 0u, ins, m);
        const uint32_t tt = S.claim(t, kMetaT, ins, m);
        S.zero_sigma(ss);
        S.zero_sigma(tt);
        S.add_sigma(ss, 1ull);
        S.qv[0] = s;
        S.qv[S.tpos(0)] = t;
        S.tlev[0] = 0;
        S.tlev[1] = 1;
        S.slev[0] = 0;
        S.slev[1] = 1;
        sh.s_cnt = 1;
        sh.t_cnt = 1;
    }
    __syncthreads();
    uint32_t s_lo = 0, s_hi = 1, t_lo = 0, t_hi = 1, a = 0, b = 0;
    uint32_t used = sh.lvl_ins[2];  // reservations so far (s and t)
    // Side balancing needs only an estimate of each frontier's work (any
    // choice gives the same distances, sigma and DAG). Low-degree graphs on a
    // store without a capacity limit use the frontier size and skip the
    // per-level degree pass (a dependent offset load plus a barrier per level).
    const bool by_count = ADSB_LOWDEG_COUNT && C.low_degree && S.room_for(~0ull);
    unsigned long long deg_s = by_count ? 1ull : C.O(s + 1) - C.O(s);
    unsigned long long deg_t = by_count ? 1ull : C.O(t + 1) - C.O(t);
    bool skip_next = false;
    if (resume) {
        s_lo = io->s_lo, s_hi = io->s_hi, t_lo = io->t_lo, t_hi = io->t_hi, a = io->a, b = io->b, used = 0;
        deg_s = io->deg_s, deg_t = io->deg_t;
        skip_next = true;
    }
    auto migrate = [&](uint32_t used_now) -> Meet {
        if (io) *io = BfsState{s_lo, s_hi, t_lo, t_hi, a, b, used_now, deg_s, deg_t};
        return {a, b, io ? 3 : 1};
    };
    // A claim pass over more adjacency than the table has room left (nearly
    // always) fills it: migrate before the pass instead of after (the level's
    // claims run once, on the region). A wrong guess only costs the sample the
    // slower store. Only the table has a capacity (table_room), and only a
    // sample that can migrate (io) and is not already resumed takes this exit.
    auto predicted = [&](unsigned long long deg) {
        return ADSB_PREDICT_QUARTERS != 0 && io != nullptr && !resume &&
               4ull * deg > static_cast<unsigned long long>(ADSB_PREDICT_QUARTERS) * S.table_room(used);
    };
    for (;;) {
        const bool skip_probe = skip_next;  // first level of a resumed sample: its probe already ran
        skip_next = false;
        if (a >= Store::kMaxDist || b >= Store::kMaxDist) return {a, b, 1};  // deeper than the store encodes
        const uint32_t cur = (a + b) % 3, nxt = (a + b + 1) % 3;
        if (C.tid == 0) sh.lvl_cnt[nxt] = sh.lvl_deg[nxt] = sh.lvl_ins[nxt] = sh.lvl_met[nxt] = 0;
        S.set_level(&sh.lvl_ins[cur], used);
        if (deg_s <= deg_t && S.room_for(deg_s)) {
            // ---- s-side level a, one pass: claim level a+1 and detect the meeting.
            // Claims made on the meeting level are harmless (never predecessors).
            if (C.tid == 0) sh.st_verts += s_hi - s_lo;
            for_edges_tok(C, S, s_lo, s_hi, false, sh.st_edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.sigma(slot); },
                      [&](uint32_t v) { return S.claim_issue(v, a + 1); },
                      [&](uint32_t, unsigned long long su, uint32_t v, unsigned long long tok) {
                          bool ins;
                          uint32_t m;
                          const uint32_t sl = S.template claim_tok<false>(v, a + 1, tok, ins, m);
                          if (ins) {
                              S.zero_sigma(sl);
                              if (S.pre_zeroed()) S.add_sigma(sl, su);
                              const uint32_t pos = s_hi + aggregated_inc(&sh.lvl_cnt[cur]);
                              ADSB_DCHECK(pos + t_hi < S.qcap);
                              S.qv[pos] = v;
                          } else if (m_is_t(m) && m_dist(m) == b) {
                              S.add_sigma(sl, su);
                              if (!(m & kMetaDag)) S.set_dag(sl);
                              sh.lvl_met[cur] = 1u;  // read after for_edges' closing barrier
                          } else if (S.pre_zeroed() && !m_is_t(m) && m_dist(m) == a + 1) {
                              S.add_sigma(sl, su);
                          }
                      });
            const bool met = sh.lvl_met[cur] != 0;  // for_edges ended with a barrier
            const uint32_t added = sh.lvl_cnt[cur];
            if (met) {
                if (C.tid == 0) sh.s_cnt = s_hi + added;  // the table clear walks the queue
                return {a, b, 0};
            }
            if (!S.pre_zeroed())
            for_edges(C, S, s_lo, s_hi, false, sh.st_edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.sigma(slot); },
                      [&](uint32_t, unsigned long long su, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && !m_is_t(m) && m_dist(m) == a + 1) S.add_sigma(sl, su);
                      });
            s_lo = s_hi;
            s_hi += added;
            used += added;  // one-pass claims reserve nothing: occupancy grew by the inserts
            a += 1;
            if (C.tid == 0) {
                sh.s_cnt = s_hi;
                if (a + 2 <= S.level_cap) S.slev[a + 1] = s_hi;  // read only after later barriers
            }
            if (s_lo == s_hi) return {a, b, 2};
            deg_s = by_count ? s_hi - s_lo : level_degrees(C, S, s_lo, s_hi, false, cur);
        } else if (deg_s > deg_t && S.room_for(deg_t)) {
            // ---- t-side level b, one pass: claim level b+1 and detect the meeting
            if (C.tid == 0) sh.st_verts += t_hi - t_lo;
            const uint32_t meta_new = kMetaT | (b + 1);
            for_edges_tok(C, S, t_lo, t_hi, true, sh.st_edges,
                      [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                      [&](uint32_t v) { return S.claim_issue(v, meta_new); },
                      [&](uint32_t su_slot, unsigned long long, uint32_t v, unsigned long long tok) {
                          bool ins;
                          uint32_t m;
                          const uint32_t sl = S.template claim_tok<false>(v, meta_new, tok, ins, m);
                          if (ins) {
                              S.zero_sigma(sl);
                              const uint32_t j = t_hi + aggregated_inc(&sh.lvl_cnt[cur]);
                              ADSB_DCHECK(j + s_hi < S.qcap);
                              S.qv[S.tpos(j)] = v;
                          } else if (!m_is_t(m) && m_dist(m) == a) {
                              S.add_sigma(su_slot, S.sigma(sl));
                              S.set_dag(su_slot);
                              sh.lvl_met[cur] = 1u;  // read after for_edges' closing barrier
                          }
                      });
            const bool met = sh.lvl_met[cur] != 0;
            const uint32_t added = sh.lvl_cnt[cur];
            if (met) {
                if (C.tid == 0) sh.t_cnt = t_hi + added;
                return {a, b, 0};
            }
            t_lo = t_hi;
            t_hi += added;
            used += added;  // one-pass claims reserve nothing: occupancy grew by the inserts
            b += 1;
            if (C.tid == 0) {
                sh.t_cnt = t_hi;
                if (b + 2 <= S.level_cap) S.tlev[b + 1] = t_hi;  // read only after later barriers
            }
            if (b + 2 > S.level_cap) return {a, b, 1};
            if (t_lo == t_hi) return {a, b, 2};
            deg_t = by_count ? t_hi - t_lo : level_degrees(C, S, t_lo, t_hi, true, cur);
        } else if (deg_s <= deg_t) {
            // ---- s-side level a: probe for the t-ball (meeting level fills sigma of T_b);
            // hubs of the frontier are searched for T_b's vertices instead of scanned
            if (C.tid == 0) sh.st_verts += s_hi - s_lo;
            if (!skip_probe) {
            for_edges(C, S, s_lo, s_hi, false, sh.st_edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.sigma(slot); },
                      [&](uint32_t, unsigned long long su, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && m_is_t(m) && m_dist(m) == b) {
                              S.add_sigma(sl, su);
                              if (!(m & kMetaDag)) S.set_dag(sl);
                              sh.lvl_met[cur] = 1u;  // read after for_edges' closing barrier
                          }
                      },
                      t_lo, t_hi, true);
            if (sh.lvl_met[cur]) return {a, b, 0};  // for_edges ended with a barrier
            if (predicted(deg_s)) return migrate(used);
            }
            // ---- no meeting: claim level a+1, then accumulate its sigma
            const uint32_t meta_new = a + 1;
            for_edges(C, S, s_lo, s_hi, false, sh.st_edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.pre_zeroed() ? S.sigma(slot) : 0ull; },
                      [&](uint32_t, unsigned long long su, uint32_t v) {
                          bool ins;
                          uint32_t m;
                          const uint32_t sl = S.claim(v, meta_new, ins, m);
                          if (S.pre_zeroed() && sl != kNone && (ins || (!m_is_t(m) && m_dist(m) == a + 1)))
                              S.add_sigma(sl, su);
                          if (ins) {
                              S.zero_sigma(sl);
                              const uint32_t pos = s_hi + aggregated_inc(&sh.lvl_cnt[cur]);
                              if (S.queue_ok(pos + 1, t_hi)) S.qv[pos] = v;
                              else sh.overflow = 1;
                          }
                      },
                      0, 0, false, true);
            __syncthreads();  // counters and overflow final before any thread reads them
            const uint32_t added = sh.lvl_cnt[cur];
            if (C.tid == 0) sh.s_cnt = min(s_hi + added, S.qcap);
            if (sh.overflow) return migrate(used);
            if (!S.pre_zeroed())
            for_edges(C, S, s_lo, s_hi, false, sh.st_edges,
                      [&](uint32_t slot, uint32_t, uint32_t) { return S.sigma(slot); },
                      [&](uint32_t, unsigned long long su, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && !m_is_t(m) && m_dist(m) == a + 1) S.add_sigma(sl, su);
                      });
            s_lo = s_hi;
            s_hi += added;
            used += sh.lvl_ins[cur];
            a += 1;
            if (C.tid == 0 && a + 2 <= S.level_cap) S.slev[a + 1] = s_hi;
            if (s_lo == s_hi) return {a, b, 2};
            deg_s = by_count ? s_hi - s_lo : level_degrees(C, S, s_lo, s_hi, false, cur);
        } else {
            // ---- t-side level b: probe for the s-ball (hubs searched for S_a's vertices)
            if (C.tid == 0) sh.st_verts += t_hi - t_lo;
            if (!skip_probe) {
            for_edges(C, S, t_lo, t_hi, true, sh.st_edges,
                      [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                      [&](uint32_t su_slot, unsigned long long, uint32_t v) {
                          uint32_t m;
                          const uint32_t sl = S.find(v, m);
                          if (sl != kNone && !m_is_t(m) && m_dist(m) == a) {
                              S.add_sigma(su_slot, S.sigma(sl));
                              S.set_dag(su_slot);
                              sh.lvl_met[cur] = 1u;  // read after for_edges' closing barrier
                          }
                      },
                      s_lo, s_hi, false);
            if (sh.lvl_met[cur]) return {a, b, 0};  // for_edges ended with a barrier
            if (predicted(deg_t)) return migrate(used);
            }
            const uint32_t meta_new = kMetaT | (b + 1);
            for_edges(C, S, t_lo, t_hi, true, sh.st_edges,
                      [&](uint32_t, uint32_t, uint32_t) { return 0ull; },
                      [&](uint32_t, unsigned long long, uint32_t v) {
                          bool ins;
                          uint32_t m;
                          const uint32_t sl = S.claim(v, meta_new, ins, m);
                          if (ins) {
                              S.zero_sigma(sl);
                              const uint32_t j = t_hi + aggregated_inc(&sh.lvl_cnt[cur]);
                              if (S.queue_ok(s_hi, j + 1)) S.qv[S.tpos(j)] = v;
                              else sh.overflow = 1;
                          }
                      },
                      0, 0, false, true);
            __syncthreads();
            const uint32_t added = sh.lvl_cnt[cur];
            if (C.tid == 0) sh.t_cnt = min(t_hi + added, S.qcap);
            if (sh.overflow) return migrate(used);
            t_lo = t_hi;
            t_hi += added;
            used += sh.lvl_ins[cur];
            b += 1;
            if (C.tid == 0 && b + 2 <= S.level_cap) S.tlev[b + 1] = t_hi;
            if (b + 2 > S.level_cap) return {a, b, 1};
            if (t_lo == t_hi) return {a, b, 2};
            deg_t = by_count ? t_hi - t_lo : level_degrees(C, S, t_lo, t_hi, true, cur);
        }
    }
}

// sigma_s on the t-side DAG layers (pull; see sampler.cu rebuild_level)
template <class Store>
__device__ void rebuild(Ctx& C, Store& S, uint32_t b) {
    for (uint32_t k = b; k >= 1; --k) {
        for_edges(C, S, S.tlev[k - 1], S.tlev[k], true, C.sh->st_rebuild,
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

// Push form for low-degree graphs on the global store: only the t-side DAG
// is walked. The DAG vertices of T_b are listed first (one pass over T_b);
// then each listed vertex x of T_k adds sigma(x) to its T_{k-1} neighbours
// and lists the ones it flags first. A lattice's DAG is ~20% of its t-ball,
// which the pull form reads whole. Same sums mod 2^64, same flags.
#ifndef ADSB_PUSH_BATCH
#define ADSB_PUSH_BATCH 0
#endif
#ifndef ADSB_KARY
#define ADSB_KARY 0  // measured slower (spills): C2 +2%, C5 +5%
#endif
#ifndef ADSB_PUSH_REBUILD
#define ADSB_PUSH_REBUILD 1
#endif
template <class Store>
__device__ void rebuild_push(Ctx& C, Store& S, uint32_t b) {
    Shared& sh = *C.sh;
    if (C.tid == 0) sh.dag_cnt = 0;
    __syncthreads();
    for (uint32_t j = S.tlev[b] + C.tid; j < S.tlev[b + 1]; j += kBT) {
        const uint32_t v = __ldcg(S.qv + S.tpos(j));
        uint32_t m;
        const bool dag = S.find(v, m) != kNone && (m & kMetaDag);
        if (dag) S.dq[aggregated_inc(&sh.dag_cnt)] = v;
    }
    __syncthreads();
    uint32_t lo = 0, hi = sh.dag_cnt;
    unsigned long long scanned = 0;
    for (uint32_t k = b; k >= 1; --k) {
        for (uint32_t i = lo + C.tid; i < hi; i += kBT) {
            const uint32_t x = __ldcg(S.dq + i);
            const unsigned long long sx = S.sigma(x);
            const uint32_t o = C.O(x), e = C.O(x + 1);
            scanned += e - o;
            for (uint32_t j0 = o; j0 < e; j0 += 4) {
                uint32_t ww[4];
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) ww[q] = j0 + q < e ? C.N(j0 + q) : kNone;
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q)
                    if (ww[q] != kNone) S.prefetch(ww[q]);
#if ADSB_PUSH_BATCH
                // all state loads first (no atomics between them), then the updates
                uint32_t mm[4];
                bool hit[4];
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) hit[q] = ww[q] != kNone && S.find(ww[q], mm[q]) != kNone;
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) {
                    if (!hit[q] || !m_is_t(mm[q]) || m_dist(mm[q]) != k - 1) continue;
                    S.add_sigma(ww[q], sx);
                    if (!(mm[q] & kMetaDag) && S.set_dag_first(ww[q])) S.dq[aggregated_inc(&sh.dag_cnt)] = ww[q];
                }
#else
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) {
                    if (ww[q] == kNone) continue;
                    uint32_t m;
                    if (S.find(ww[q], m) == kNone || !m_is_t(m) || m_dist(m) != k - 1) continue;
                    S.add_sigma(ww[q], sx);
                    if (!(m & kMetaDag) && S.set_dag_first(ww[q])) S.dq[aggregated_inc(&sh.dag_cnt)] = ww[q];
                }
#endif
            }
        }
        __syncthreads();
        lo = hi;
        hi = sh.dag_cnt;
    }
    const uint32_t wm = __reduce_add_sync(kFull, static_cast<uint32_t>(scanned));
    if (C.lane == 0 && wm) sh.st_rebuild[C.warp] += wm;
    __syncthreads();
}

__device__ __forceinline__ void add65(unsigned long long& lo, uint32_t& hi, unsigned long long xlo, uint32_t xhi) {
    const unsigned long long n = lo + xlo;
    hi += xhi + (n < lo ? 1u : 0u);
    lo = n;
}

// First lane (in lane order) among the candidates `cb` at which the running
// `r -= val` scan stops (r < val), or -1 with r reduced by the chunk's total.
// Warp-uniform; cost is one 64-bit shuffle per candidate.
__device__ __forceinline__ int pick_candidate(uint32_t cb, unsigned long long val, unsigned long long& r) {
    for (uint32_t bits = cb; bits; bits &= bits - 1) {
        const int j = __ffs(bits) - 1;
        const unsigned long long x = __shfl_sync(kFull, val, j);
        if (r < x) return j;
        r -= x;
    }
    return -1;
}

// Block-wide backtrack (kadabra.hpp:227-242). Every step scans N(cur) in
// ascending order, kBT entries per round: each thread tests one neighbour
// against the predecessor rule, a 65-bit block prefix sum over the
// candidates' sigma (warp shuffles + per-warp totals) finds the first
// neighbour with r < prefix — exactly the reference's sequential
// `r -= sigma[p]` scan. All threads draw the same r from their copy of the
// stream. Returns false on an inconsistent state (every predecessor sigma
// wrapped to 0), which the reference leaves undefined.
// Hub steps: the predecessors of cur are exactly the vertices of one BFS
// level list (s-level want_dist, or t-level want_dist with the DAG flag)
// that are adjacent to cur. When that list is much shorter than N(cur), each
// thread takes list entries and binary-searches them in cur's ascending
// adjacency; the position found is the reference's scan order
// (kadabra.hpp:231-241), so the candidates ranked by position with 65-bit
// prefix sums pick the same predecessor as scanning N(cur). Returns false
// (the caller scans) when more than kBT candidates turn up or no interval
// holds r (every candidate sigma wrapped to 0).
template <class Store>
__device__ bool level_pick(Ctx& C, Store& S, uint32_t beg, uint32_t end, uint32_t lo, uint32_t hi, bool want_t,
                           uint32_t want_dist, unsigned long long r, uint32_t& cur, uint32_t& cmeta,
                           unsigned long long& csig) {
    Shared& sh = *C.sh;
    if (C.tid == 0) sh.dag_cnt = 0;
    __syncthreads();
    uint32_t probes = 0;
    // cur's search tree (hub_index.cuh), when it has one
    uint32_t tree = kNone;
    if constexpr (Store::kTrees)
        if (sh.hub_ref != nullptr && hub_has_tree(end - beg)) tree = __ldg(sh.hub_ref + cur);
#if ADSB_KARY
    if (hi - lo <= 2 * (kBT / 32)) {
        // short list: one warp per entry, 32-ary search (each round one
        // coalesced-ish probe per lane narrows the range 32x: ~4 L2 round trips
        // for a 10^5-entry hub instead of ~17 dependent ones)
        for (uint32_t j = lo + C.warp; j < hi; j += kBT / 32) {
            const uint32_t q = S.qv[want_t ? S.tpos(j) : j];
            uint32_t m;
            const uint32_t sl = S.find(q, m);
            if (sl == kNone || m_is_t(m) != want_t || m_dist(m) != want_dist || (want_t && !(m & kMetaDag)))
                continue;  // warp-uniform
            uint32_t l = beg, h = end;  // lower bound of q in [l, h)
            while (h - l > 32) {
                const uint32_t step = (h - l + 31) / 32;
                const uint32_t pos = l + C.lane * step;
                const bool below = pos < h && C.N(pos) < q;
                const uint32_t cnt = __popc(__ballot_sync(kFull, below));  // probes below q: a prefix
                probes += C.lane == 0 ? 32 : 0;
                // the lower bound lies in (probe cnt-1, probe cnt]: keep probe cnt
                const uint32_t nl = cnt == 0 ? l : l + (cnt - 1) * step + 1;
                const uint32_t nh = min(h, l + cnt * step + 1);
                l = nl;
                h = nh;
            }
            const uint32_t pos = l + C.lane;
            const uint32_t val = pos < h ? C.N(pos) : 0xFFFFFFFFu;
            const uint32_t cnt = __popc(__ballot_sync(kFull, pos < h && val < q));
            const bool hit = __any_sync(kFull, pos < h && val == q);
            probes += C.lane == 0 ? 32 : 0;
            if (hit && C.lane == 0) {
                const uint32_t k = atomicAdd(&sh.dag_cnt, 1u);
                if (k < kBT) {
                    sh.cbase[k] = l + cnt;
                    sh.cslot[k] = q;
                    sh.scan[k] = m;
                    sh.cval[k] = S.sigma(sl);
                }
            }
        }
    } else
#endif
    for (uint32_t j = lo + C.tid; j < hi; j += kBT) {
        const uint32_t q = S.qv[want_t ? S.tpos(j) : j];
        uint32_t m;
        const uint32_t sl = S.find(q, m);
        if (sl == kNone || m_is_t(m) != want_t || m_dist(m) != want_dist || (want_t && !(m & kMetaDag))) continue;
        uint32_t l = beg, h = end;
        if (Store::kTrees && tree != kNone) {
            l = tree_lower_bound(C, sh.hub_keys + tree, beg, end, q);
            probes += search_reads(end - beg, true);
        } else {
            while (l < h) {
                const uint32_t mid = (l + h) >> 1;
                ++probes;
                if (C.N(mid) < q) l = mid + 1;
                else h = mid;
            }
        }
        if (l < end && C.N(l) == q) {
            const uint32_t k = atomicAdd(&sh.dag_cnt, 1u);
            if (k < kBT) {
                sh.cbase[k] = l;
                sh.cslot[k] = q;
                sh.scan[k] = m;
                sh.cval[k] = S.sigma(sl);
            }
        }
    }
    const uint32_t wp = __reduce_add_sync(kFull, probes);
    if (C.lane == 0 && wp) sh.st_back[C.warp] += wp;
    __syncthreads();
    const uint32_t c = sh.dag_cnt;
    if (c == 0 || c > kBT) {
        __syncthreads();
        return false;
    }
    const bool mine = C.tid < c;
    const uint32_t my_pos = mine ? sh.cbase[C.tid] : 0u;
    const unsigned long long my_sig = mine ? sh.cval[C.tid] : 0ull;
    unsigned long long pre_lo = 0;
    uint32_t pre_hi = 0;
    if (mine)
        for (uint32_t j = 0; j < c; ++j)
            if (sh.cbase[j] < my_pos) add65(pre_lo, pre_hi, sh.cval[j], 0u);
    // candidate intervals [pre, pre + sigma) in scan order are disjoint: at most one holds r
    const bool hit = mine && pre_hi == 0 && pre_lo <= r && r - pre_lo < my_sig;
    if (C.tid == 0) sh.first = kNone;
    __syncthreads();
    if (hit) {
        sh.first = C.tid;
        sh.bch = sh.cslot[C.tid];
        sh.bchm = sh.scan[C.tid];
        sh.bchs = my_sig;
    }
    __syncthreads();
    const bool ok = sh.first != kNone;
    if (ok) {
        cur = sh.bch;
        cmeta = sh.bchm;
        csig = sh.bchs;
    }
    __syncthreads();
    return ok;
}

template <int kMode, class Store>
__device__ bool backtrack(Ctx& C, Store& S, const SamplerParams& p, SplitMix64& rng, uint32_t t, Meet mt,
                          uint32_t frame_local) {
    Shared& sh = *C.sh;
    constexpr uint32_t kNW = kBT / 32;
    const uint32_t d = mt.a + mt.b + 1;
    if (C.tid == 0) sh.last_d = d;
    if (d < 2) return true;
    constexpr bool kDet = kMode == kModeDet;
    if (kDet && C.tid == 0) sh.ev_pos = atomicAdd(p.ev_cursor, static_cast<unsigned long long>(d - 1));
    uint32_t cur = t, cmeta = 0;
    const uint32_t tslot = S.find(t, cmeta);
    unsigned long long csig = S.sigma(tslot);
    __syncthreads();
    const uint64_t ev_pos = kDet ? sh.ev_pos : 0;
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
        const uint32_t beg = C.O(cur), end = C.O(cur + 1);
        bool found = false;
        if (end - beg <= kSmallStep) {
            // Low-degree step: warp 0 scans alone (warp-level 65-bit prefix),
            // one barrier publishes the choice; saves the block-wide rounds.
            if (C.warp == 0) {
                uint32_t ch = kNone, chm = 0, first = kNone, firstm = 0;
                unsigned long long chs = 0;
                for (uint32_t base = beg; base < end && ch == kNone; base += 32) {
                    const uint32_t i = base + C.lane;
                    uint32_t q = 0, m = 0;
                    unsigned long long val = 0;
                    bool cand = false;
                    if (i < end) {
                        q = C.N(i);
#if ADSB_SPEC_SIGMA
                        // global store: a vertex's sigma sits next to its meta word,
                        // so both loads go out together (one round trip per step less)
                        const unsigned long long sv = Store::kSlotIsVertex ? S.sigma(q) : 0ull;
#endif
                        const uint32_t sl = S.find(q, m);
                        cand = sl != kNone && m_is_t(m) == want_t && m_dist(m) == want_dist &&
                               (!want_t || (m & kMetaDag));
                        if (cand) {
#if ADSB_SPEC_SIGMA
                            val = Store::kSlotIsVertex ? sv : S.sigma(sl);
#else
                            val = S.sigma(sl);
#endif
#if ADSB_BT_PREFETCH
                            // one of the candidates is the next step's cur: its offsets
                            // line is in L1 when that step starts
                            asm volatile("prefetch.global.L1 [%0];" ::"l"(C.off + q));
#endif
                        }
                    }
                    if (C.lane == 0) sh.st_back[C.warp] += min(32u, end - base);
                    const uint32_t cb = __ballot_sync(kFull, cand);
                    if (first == kNone && cb) {
                        const int f0 = __ffs(cb) - 1;
                        first = __shfl_sync(kFull, q, f0);
                        firstm = __shfl_sync(kFull, m, f0);
                    }
                    // the reference's sequential `r -= sigma[p]` over this
                    // chunk's predecessors, in id (= lane) order
                    const int f = pick_candidate(cb, val, r);
                    if (f >= 0) {
                        ch = __shfl_sync(kFull, q, f);
                        chm = __shfl_sync(kFull, m, f);
                        chs = __shfl_sync(kFull, val, f);
                    }
                }
                if (ch == kNone && first != kNone) {  // degenerate sigma (see the block path)
                    ch = first;
                    chm = firstm;
                    chs = 0;
                    if (C.lane == 0) sh.st_degen += 1;
                }
                if (C.lane == 0) {
                    sh.first = ch;
                    sh.ch = ch;
                    sh.chm = chm;
                    sh.chs = chs;
                }
            }
            __syncthreads();
            found = sh.first != kNone;
            cur = sh.ch;
            cmeta = sh.chm;
            csig = sh.chs;
            __syncthreads();
            if (!found) return false;
        }
#if ADSB_LEVEL_PICK
        if (!found && end - beg > ADSB_LP_MIN_ROUNDS * kBT) {
            const uint32_t lo = want_t ? S.tlev[want_dist] : S.slev[want_dist];
            const uint32_t hi = want_t ? S.tlev[want_dist + 1] : S.slev[want_dist + 1];
            const uint32_t deg = end - beg;
            if (hi - lo <= 4 * kBT && 2ull * (hi - lo) * search_cost(deg, Store::kTrees && sh.hub_ref != nullptr) < deg)
                found = level_pick(C, S, beg, end, lo, hi, want_t, want_dist, r, cur, cmeta, csig);
        }
#endif
        // the next round's neighbour id is loaded one round ahead, so its
        // latency overlaps this round's barriers (hub steps take many rounds)
        uint32_t q_next = !found && beg + C.tid < end ? C.N(beg + C.tid) : 0u;
        for (uint32_t base = beg; !found && base < end; base += kBT) {
            const uint32_t i = base + C.tid;
            uint32_t q = q_next, m = 0;
            unsigned long long val = 0;
            if (i + kBT < end) q_next = C.N(i + kBT);
            if (i < end) {
                const uint32_t sl = S.find(q, m);
                if (sl != kNone && m_is_t(m) == want_t && m_dist(m) == want_dist && (!want_t || (m & kMetaDag))) {
                    val = S.sigma(sl);
#if ADSB_BT_PREFETCH
                    asm volatile("prefetch.global.L1 [%0];" ::"l"(C.off + q));
#endif
                }
            }
            if (C.tid == 0) sh.st_back[0] += min(static_cast<uint32_t>(kBT), end - base);
            // per-warp 65-bit candidate totals, then the warp whose range holds
            // r walks its candidates in lane (= id) order
            const uint32_t cb = __ballot_sync(kFull, val != 0);
            unsigned long long wlo = 0;
            uint32_t whi = 0;
            if (__popc(cb) <= 4) {
                for (uint32_t bits = cb; bits; bits &= bits - 1)
                    add65(wlo, whi, __shfl_sync(kFull, val, __ffs(bits) - 1), 0u);
            } else {
                wlo = val;
#pragma unroll
                for (int dd = 16; dd >= 1; dd >>= 1)
                    add65(wlo, whi, __shfl_xor_sync(kFull, wlo, dd), __shfl_xor_sync(kFull, whi, dd));
            }
            if (C.lane == 0) {
                sh.wlo[C.warp] = wlo;
                sh.whi[C.warp] = whi;
            }
            __syncthreads();
            unsigned long long pre_lo = 0, tot_lo = 0;
            uint32_t pre_hi = 0, tot_hi = 0;
            for (uint32_t w = 0; w < kNW; ++w) {
                if (w == C.warp) {
                    pre_lo = tot_lo;
                    pre_hi = tot_hi;
                }
                add65(tot_lo, tot_hi, sh.wlo[w], sh.whi[w]);
            }
            // r in [pre, pre + wtot) for exactly one warp when the round holds the choice
            unsigned long long end_lo = pre_lo;
            uint32_t end_hi = pre_hi;
            add65(end_lo, end_hi, wlo, whi);
            if (pre_hi == 0 && pre_lo <= r && (end_hi > 0 || r < end_lo)) {
                unsigned long long rr = r - pre_lo;
                const int f = pick_candidate(cb, val, rr);
                if (C.lane == static_cast<uint32_t>(f)) {
                    sh.bch = q;
                    sh.bchm = m;
                    sh.bchs = val;
                }
            }
            __syncthreads();
            if (tot_hi > 0 || r < tot_lo) {
                // written again only after a later round's first barrier (the
                // warp-0 path has its own copy), so no trailing barrier
                cur = sh.bch;
                cmeta = sh.bchm;
                csig = sh.bchs;
                found = true;
                break;
            }
            r -= tot_lo;  // tot_hi == 0 here: otherwise the round would hold the choice
        }
        if (!found) {
            // sigma(cur) and every predecessor sigma are 0 mod 2^64: reference UB
            // (oracle.c documents the rule) -> the first predecessor in id order
            for (uint32_t base = beg; base < end && !found; base += kBT) {
                const uint32_t i = base + C.tid;
                uint32_t q = 0, m = 0;
                bool cand = false;
                if (i < end) {
                    q = C.N(i);
                    const uint32_t sl = S.find(q, m);
                    cand = sl != kNone && m_is_t(m) == want_t && m_dist(m) == want_dist && (!want_t || (m & kMetaDag));
                }
                if (C.tid == 0) sh.first = kNone;
                __syncthreads();
                const uint32_t ball = __ballot_sync(kFull, cand);
                if (ball && C.lane == static_cast<uint32_t>(__ffs(ball) - 1)) atomicMin(&sh.first, C.tid);
                __syncthreads();
                if (C.tid == sh.first) {
                    sh.ch = q;
                    sh.chm = m;
                    sh.chs = 0;
                }
                __syncthreads();
                if (sh.first != kNone) {
                    cur = sh.ch;
                    cmeta = sh.chm;
                    csig = sh.chs;
                    found = true;
                }
                __syncthreads();
            }
            if (!found) return false;
            if (C.tid == 0) sh.st_degen += 1;
        }
        if (C.tid == 0) {
            if (kMode == kModeDet) {
                if (ev_pos + step < p.ev_cap)
                    p.events[ev_pos + step] = (static_cast<unsigned long long>(cur) << 32) | frame_local;
            } else if (kMode == kModeEpoch) {
                atomicAdd(p.counts + cur, 1u);
            } else {
                // fused: frame_local is the ring slot; record first touches for the fold
                ++sh.recorded;
                const size_t base = static_cast<size_t>(frame_local) * p.n;
                if (atomicAdd(p.ring_cnt + base + cur, 1u) == 0u)
                    p.ring_list[base + atomicAdd(p.ring_len + frame_local, 1u)] = cur;
            }
        }
        ds_cur = m_is_t(cmeta) ? d - m_dist(cmeta) : m_dist(cmeta);
    }
    return true;
}

// Whole sample with one store. Returns 0 ok, 1 overflow (redo with the global
// store), 2 inconsistent state.
template <int kMode, class Store>
__device__ int run_sample(Ctx& C, Store& S, const SamplerParams& p, SplitMix64& rng, uint32_t s, uint32_t t,
                          uint32_t frame_local, BfsState* io = nullptr) {
    Shared& sh = *C.sh;
    S.begin(C.tid);
    if (C.tid == 0) {
        sh.overflow = 0;
    }
    __syncthreads();
    ADSB_PHASE_MARK(t0);
    const Meet mt = bfs(C, S, s, t, io);
    if (mt.status == 3) return 3;  // table kept intact for migrate_to_global
    ADSB_PHASE_MARK(t1);
    ADSB_PHASE_ADD(0, t1 - t0);
    ADSB_PHASE_ADD(5, mt.a + mt.b + 1);
#ifdef ADSB_DEBUG_CHECKS
    if (mt.status == 0 && mt.a + mt.b == 0 && C.tid == 0) {
        bool adj = false;
        for (uint32_t j = C.O(s); j < C.O(s + 1); ++j) adj |= C.N(j) == t;
        ADSB_DCHECK(adj, "met at distance 1 but t is not a neighbour of s");
    }
#endif
    if (mt.status != 0) {
        S.end(C, *C.sh);
        return mt.status;
    }
    if constexpr (Store::kHasDagQueue && ADSB_PUSH_REBUILD) {
        if (C.low_degree) rebuild_push(C, S, mt.b);
        else rebuild(C, S, mt.b);
    } else {
        rebuild(C, S, mt.b);
    }
    ADSB_PHASE_MARK(t2);
    const int rc = backtrack<kMode>(C, S, p, rng, t, mt, frame_local) ? 0 : 2;  // block-uniform
    ADSB_PHASE_MARK(t3);
    S.end(C, sh);
    ADSB_PHASE_MARK(t4);
    ADSB_PHASE_ADD(1, t2 - t1);
    ADSB_PHASE_ADD(2, t3 - t2);
    ADSB_PHASE_ADD(3, t4 - t3);
    ADSB_PHASE_ADD(7, 1);
    return rc;
}

// One sample (s, t draw + traversal + backtrack) with the shared-memory store
// first and the global store as fallback. Returns 0 ok or an error code.
extern __shared__ unsigned long long adsb_dyn[];

// Store descriptors are rebuilt per sample from the launch parameters rather
// than kept live across the sample loop (register budget: 64 per thread).
template <bool kVec = false>
__device__ __forceinline__ SmemStoreT<kVec> make_smem_store(const SamplerParams& p, Shared& sh) {
    SmemStoreT<kVec> sm;
    const uint32_t H = p.hash_cap;
    sm.sig = adsb_dyn;                                     // H x u64
    sm.km = reinterpret_cast<uint32_t*>(adsb_dyn + H);     // H x u32
    sm.qcap = H / 2;
    sm.qv = sm.km + H;                                     // H/2 x u32
    uint32_t* tail = sm.qv + H / 2;
#if ADSB_SMEM_FILTER
    sm.fb = tail;                                          // kFbWords x u32
    tail += SmemStoreT<kVec>::kFbWords;
#endif
    sm.crange = kVec ? tail : nullptr;                     // 2 kBT x u32 (vector kernels)
    sm.tlev = sh.tlev_small;
    sm.slev = sh.slev_small;
    sm.cap = H;
    sm.limit = H / 2;
    sm.level_cap = kSmemLevels;
    sm.sh = &sh;
    return sm;
}

template <bool kGlobalOnly, bool kTrees = false>
__device__ __forceinline__ GlobalStoreT<ADSB_LOAD_BATCH, kGlobalOnly, kTrees> make_global_store(const SamplerParams& p,
                                                                                                uint32_t slot, uint32_t tag) {
    GlobalStoreT<ADSB_LOAD_BATCH, kGlobalOnly, kTrees> gs;
    gs.st = p.state + 2ull * p.slot_stride * slot;
    gs.qv = p.queue + static_cast<size_t>(p.slot_stride) * slot;
    gs.tlev = p.tlev + static_cast<size_t>(p.level_cap) * slot;
    gs.slev = p.tlev + static_cast<size_t>(p.level_cap) * (p.slots + slot);
    gs.dq = p.dagq + static_cast<size_t>(p.slot_stride) * slot;
    gs.clear = p.clear_layout != 0;
    gs.filt = nullptr;
    {
        // the vector kernels' row ranges sit behind the table and queue (make_smem_store)
        const uint32_t H = p.hash_cap;
        uint32_t* tail = reinterpret_cast<uint32_t*>(adsb_dyn + H) + H + H / 2;
#if ADSB_SMEM_FILTER
        tail += SmemStoreT<kTrees>::kFbWords;
#endif
        gs.crange = kTrees ? tail : nullptr;
    }
    gs.tag = tag;
    gs.qcap = p.n;
    gs.level_cap = p.level_cap;
    return gs;
}

// Borrow a free global-state region (thread 0; shared-memory kernels, whose
// grid can exceed the number of regions on huge graphs). Spins while every
// region is lent: holders finish their sample without waiting on anything.
__device__ uint32_t acquire_region(const SamplerParams& p) {
    const uint32_t words = (p.slots + 31) / 32;
    for (uint32_t round = 0;; ++round) {
        for (uint32_t w0 = 0; w0 < words; ++w0) {
            const uint32_t w = (blockIdx.x + w0) % words;
            uint32_t free_bits = ~*reinterpret_cast<volatile uint32_t*>(p.slot_busy + w);
            if (w == words - 1 && (p.slots & 31)) free_bits &= (1u << (p.slots & 31)) - 1u;
            while (free_bits) {
                const uint32_t j = __ffs(free_bits) - 1;
                const uint32_t bit = 1u << j;
                if (!(atomicOr(p.slot_busy + w, bit) & bit)) {
                    __threadfence();
                    return w * 32 + j;
                }
                free_bits &= ~bit;
            }
        }
        __nanosleep(256);
    }
}

__device__ void release_region(const SamplerParams& p, uint32_t region, uint32_t tag) {
    p.slot_tag[region] = tag;
    // release: the tag is visible before the region is free (no L1 invalidation)
    asm volatile("red.release.gpu.global.and.b32 [%0], %1;" ::"l"(p.slot_busy + region / 32),
                 "r"(~(1u << (region & 31)))
                 : "memory");
}

// A sample whose shared-memory table filled up at a claim pass continues on a
// global region instead of being redone: the completed levels (s-side dist
// <= a, t-side dist <= b: vertex, side, dist, DAG flag, sigma), both queue
// ends and the level boundaries are copied; the partial claims of the failed
// level are dropped (its claim pass reruns on the region). Then the table is
// cleared for the membership filter. Results are unchanged: the region holds
// exactly the state the global store would have built.
template <bool kVec, class GS>
__device__ void migrate_to_global(Ctx& C, const SamplerParams& p, GS& gs, const BfsState& st) {
    Shared& sh = *C.sh;
    auto sm = make_smem_store<kVec>(p, sh);
    const unsigned long long hi_word = gs.clear ? GS::kPresent : static_cast<unsigned long long>(gs.tag) << 32;
    for (uint32_t h = C.tid; h < sm.cap; h += kBT) {
        const uint32_t w = sm.km[h];
        if (w == 0u) continue;
        const uint32_t meta = SmemStoreT<kVec>::decode(w);
        const bool keep = m_is_t(meta) ? m_dist(meta) <= st.b : m_dist(meta) <= st.a;
        if (!keep) continue;
        const uint32_t v = (w >> 8) - 1u;
        __stcg(gs.st + 2ull * v, hi_word | meta);
        __stcg(gs.st + 2ull * v + 1, sm.sig[h]);
    }
    for (uint32_t i = C.tid; i < st.s_hi; i += kBT) __stcg(gs.qv + i, sm.qv[i]);
    for (uint32_t j = C.tid; j < st.t_hi; j += kBT) __stcg(gs.qv + gs.tpos(j), sm.qv[sm.tpos(j)]);
    for (uint32_t k = C.tid; k <= st.b + 1 && k < kSmemLevels; k += kBT) gs.tlev[k] = sh.tlev_small[k];
    for (uint32_t k = C.tid; k <= st.a + 1 && k < kSmemLevels; k += kBT) gs.slev[k] = sh.slev_small[k];
    __threadfence_block();
    __syncthreads();
    sm.clear_all(C.tid);
    __syncthreads();
}

// gtag: the global-only kernel's generation tag for its own region (block-uniform).
template <int kMode, bool kGlobalOnly, bool kVec>
__device__ void one_sample(Ctx& C, const SamplerParams& p, SplitMix64& rng, uint32_t frame_local, uint32_t& gtag) {
    const uint32_t s = static_cast<uint32_t>(rng.next_below(p.n));
    uint32_t t = static_cast<uint32_t>(rng.next_below(p.n - 1));
    if (t >= s) ++t;
    if (C.tid == 0) C.sh->last_d = 0xFFFF;
    if (__ldg(p.label + s) != __ldg(p.label + t)) return;  // disconnected pair: empty sample
    ADSB_PHASE_MARK(os0);
    int rc = 1;
    BfsState mig{};
    mig.used = 0;
    if constexpr (!kGlobalOnly) {
        if (p.use_smem) {
            auto sm = make_smem_store<kVec>(p, *C.sh);
            // with the membership filter available, a table overflow at a claim
            // pass migrates the sample (rc 3) instead of redoing it from scratch
            const bool can_migrate = ADSB_MIGRATE && ADSB_FALLBACK_FILTER &&
                                     p.hash_cap * 12u >= (1u << GlobalStoreT<ADSB_LOAD_BATCH>::kFiltLog) / 8u;
            rc = run_sample<kMode>(C, sm, p, rng, s, t, frame_local, can_migrate ? &mig : nullptr);
        }
    }
    const bool fell_back = rc == 1 || rc == 3;
    (void)fell_back;
    if (rc == 1 || rc == 3) {
        uint32_t region = blockIdx.x, tag;
        if constexpr (kGlobalOnly) {
            tag = ++gtag;
        } else {
            Shared& sh = *C.sh;
            if (C.tid == 0) {
                sh.n_fallbacks += 1;
                sh.g_region = acquire_region(p);
                sh.g_tag = __ldcg(p.slot_tag + sh.g_region) + 1u;
            }
            __syncthreads();
            region = sh.g_region;
            tag = sh.g_tag;
        }
        if (tag == 0) {
            // u32 generation tags persist across calls; after 2^32 samples on a
            // region the tag wraps to 0, the value zeroed words carry: clear the
            // region's state once and restart at 1 (block-uniform branch)
            unsigned long long* st = p.state + 2ull * p.slot_stride * region;
            for (size_t i = C.tid; i < 2ull * p.slot_stride; i += kBT) __stcg(st + i, 0ull);
            __threadfence_block();
            __syncthreads();
            tag = 1;
            if constexpr (kGlobalOnly) gtag = 1;
        }
        auto gs = make_global_store<kGlobalOnly, kVec>(p, region, tag);
        if constexpr (!kGlobalOnly) {
            if (rc == 3) migrate_to_global<kVec>(C, p, gs, mig);
        }
#if ADSB_FALLBACK_FILTER
        // the table is empty here (the overflowed attempt cleared it, or the
        // migration did) and covers the filter: 2^18 bits = 32 KB <= hash_cap * 12 B
        if constexpr (!kGlobalOnly)
            if (p.hash_cap * 12u >= (1u << GlobalStoreT<ADSB_LOAD_BATCH>::kFiltLog) / 8u) {
                gs.filt = reinterpret_cast<uint32_t*>(adsb_dyn);
                if (rc == 3) {
                    // the filter holds exactly the migrated (claimed) vertices
                    for (uint32_t i = C.tid; i < mig.s_hi + mig.t_hi; i += kBT) {
                        const uint32_t q = i < mig.s_hi ? i : gs.tpos(i - mig.s_hi);
                        gs.fset(__ldcg(gs.qv + q));
                    }
                    __syncthreads();
                }
            }
#endif
        if (rc == 3) mig.used = ~0u;  // resume at the claim pass
        rc = run_sample<kMode>(C, gs, p, rng, s, t, frame_local, rc == 3 ? &mig : nullptr);
        if constexpr (!kGlobalOnly) {
            __syncthreads();  // every thread is done with the region
            if (C.tid == 0) release_region(p, region, tag);
#if ADSB_FALLBACK_FILTER
            if (gs.filt) {
                make_smem_store(p, *C.sh).clear_all(C.tid);  // the next sample needs an empty table
                __syncthreads();
            }
#endif
        }
    }
    if (rc != 0 && C.tid == 0) C.sh->n_errors += 1;
    ADSB_PHASE_MARK(os1);
    ADSB_PHASE_ADD(fell_back ? 14 : 15, os1 - os0);
}

__device__ __forceinline__ unsigned long long vload(const unsigned long long* a) {
    return *reinterpret_cast<const volatile unsigned long long*>(a);
}

// Fused epoch pipeline: fold finished epochs strictly in order (the reference's
// cumulative check, engine.hpp:267-341, at epoch granularity) and evaluate the
// stopping rule on the device. At most one block folds at a time (lock); a
// block that finishes an epoch while another folds leaves it to that block,
// which re-checks for completed successors after releasing the lock.
__device__ void fold_chain(Ctx& C, const SamplerParams& p) {
    Shared& sh = *C.sh;
    unsigned long long* ctl = p.ctl;
    const unsigned long long kNoEpoch = ~0ull;
    for (;;) {
        // The fence orders this block's completion (the release add on Done[k])
        // before its lock attempt: with the lock holder's exch + fence + re-read
        // of Done, one of the two always sees the other (store buffering).
        if (C.tid == 0) {
            __threadfence();
            sh.flag = atomicCAS(ctl + kCtlLock, 0ull, 1ull) == 0ull ? 1u : 0u;
        }
        __syncthreads();
        const bool got = sh.flag != 0;
        __syncthreads();
        if (!got) return;
        for (;;) {
            if (C.tid == 0) {
                __threadfence();
                const unsigned long long f = vload(ctl + kCtlFolded);
                const uint32_t k = static_cast<uint32_t>(f % p.ring_k);
                const bool go = vload(ctl + kCtlStop) == kNoEpoch && f < p.max_epochs &&
                                vload(ctl + kCtlDone + k) == p.epoch_b;
                sh.fold_epoch = go ? f : kNoEpoch;
                sh.fold_len = go ? *reinterpret_cast<volatile uint32_t*>(p.ring_len + k) : 0u;
                sh.fold_max = 0;
                __threadfence();
            }
            __syncthreads();
            const unsigned long long f = sh.fold_epoch;
            const uint32_t len = sh.fold_len;
            if (f == kNoEpoch) {
                __syncthreads();
                break;
            }
            const uint32_t k = static_cast<uint32_t>(f % p.ring_k);
            uint32_t* cnt = p.ring_cnt + static_cast<size_t>(k) * p.n;
            const uint32_t* list = p.ring_list + static_cast<size_t>(k) * p.n;
            uint32_t local = 0, consumed = 0;
            for (uint32_t j = C.tid; j < len; j += kBT) {
                const uint32_t v = __ldcg(list + j);
                const uint32_t c = atomicExch(cnt + v, 0u);
                consumed += c;
                const uint32_t tot = __ldcg(p.total + v) + c;
                __stcg(p.total + v, tot);
                local = max(local, tot);
            }
            if (local) atomicMax(&sh.fold_max, local);
            if (p.audit && consumed) atomicAdd(p.audit + p.max_epochs * p.epoch_b + f, consumed);
            // Every thread's total[] stores must reach L2 before thread 0
            // publishes the fold (a fence orders only its own thread's
            // accesses): otherwise the next lock holder can read a stale total
            // and overwrite it, losing this epoch's counts.
            __threadfence();
            __syncthreads();
            if (C.tid == 0) {
                const unsigned long long m = max(vload(ctl + kCtlMax), static_cast<unsigned long long>(sh.fold_max));
                ctl[kCtlMax] = m;
                const bool pass = rule_passes(m, (f + 1) * p.epoch_b, p.rule);
                p.ring_len[k] = 0;
                ctl[kCtlDone + k] = 0;
                if (pass) {
                    ctl[kCtlStop] = f;
                } else if (f + 1 >= p.max_epochs) {
                    ctl[kCtlCapped] = 1;
                    ctl[kCtlStop] = f;
                }
                __threadfence();
                atomicExch(ctl + kCtlFolded, f + 1);  // publishes the reset ring slot
                __threadfence();
            }
            __syncthreads();
        }
        if (C.tid == 0) {
            __threadfence();
            atomicExch(ctl + kCtlLock, 0ull);
            __threadfence();
            const unsigned long long f = vload(ctl + kCtlFolded);
            sh.flag = vload(ctl + kCtlStop) == kNoEpoch && f < p.max_epochs &&
                      vload(ctl + kCtlDone + f % p.ring_k) == p.epoch_b ? 1u : 0u;
        }
        __syncthreads();
        const bool again = sh.flag != 0;
        __syncthreads();
        if (!again) return;
    }
}

// kVec: the shared-memory store's flattened adjacency reads are 16-byte
// vectors (chosen for graphs whose CSR misses L2, where bytes in flight per
// load matter; scalar reads win on L2-resident CSRs).
template <int kMode, bool kGlobalOnly, bool kVec = false>
__global__ void __launch_bounds__(kBT, kGlobalOnly ? ADSB_GLOBAL_MINB * 256 / kBT : ADSB_MINB_PER_256 * 256 / kBT)
    sampler_cta_kernel(SamplerParams p) {
    __shared__ Shared sh;
    Ctx C;
    C.off = p.off;
    C.nbrs = p.nbrs;
    C.csr_hint = p.csr_hint;
#if ADSB_POL_HOIST
    C.pol = csr_policy(p.csr_hint);
#endif
    C.tid = threadIdx.x;
    C.hub_factor = p.hub_factor;
    C.lane = threadIdx.x & 31;
    C.warp = threadIdx.x >> 5;
    C.sh = &sh;
    C.n = p.n;
    C.low_degree = p.max_degree <= 32;
    const uint32_t slot = blockIdx.x;
    uint32_t gtag = kGlobalOnly ? p.slot_tag[slot] : 0u;  // shared-memory kernels borrow regions instead

    if constexpr (!kGlobalOnly) make_smem_store(p, sh).clear_all(C.tid);
    __syncthreads();
    ADSB_PHASE_MARK(k0);
    // The published ticket is double-buffered by loop parity: one barrier per
    // sample (slot `par` is rewritten two iterations later, after every thread
    // passed the next barrier). Tickets are not fetched ahead: a block holding
    // a second ticket through a long sample delays the tail (measured on C4).
    if (C.tid == 0) {
        sh.recorded = 0;
        sh.st_verts = sh.st_degen = 0;
        sh.n_samples = sh.n_fallbacks = sh.n_errors = 0;
        sh.last_d = 0;
        sh.pending = 0;
        sh.done_old = 0;
        sh.spare_tick = ~0ull;
        sh.hub_ref = p.hub_ref;
        sh.hub_keys = p.hub_keys;
    }
    if (C.tid < kBT / 32) sh.st_edges[C.tid] = sh.st_rebuild[C.tid] = sh.st_back[C.tid] = 0;
    __syncthreads();
    if (kMode != kModeFused) {
        for (uint32_t it = 0;; ++it) {
            const uint32_t par = it & 1;
            if (C.tid == 0) sh.tick[par] = atomicAdd(p.ticket, 1ull);
            __syncthreads();
            const unsigned long long item = sh.tick[par];
            if (item >= p.num_items) break;
            const uint64_t local = item * p.world + p.rank;
            SplitMix64 rng(reseed(p.seed, p.first + local));
            for (uint64_t i = 0; i < p.spf; ++i) {
                if (C.tid == 0) sh.n_samples += 1;
                one_sample<kMode, kGlobalOnly, kVec>(C, p, rng, static_cast<uint32_t>(local), gtag);
            }
        }
    } else {
        // Sample i belongs to epoch i / B and ring slot (i / B) % K. A block may
        // start epoch e only once epoch e - K has been folded (its slot is free);
        // every earlier epoch's samples are already held by running blocks, so
        // the wait always ends (one persistent grid, all blocks resident).
        // A sample's completion (Done counter) is issued after it and read at
        // the top of the next iteration: a block that completed an epoch folds
        // it before it may wait on a ring slot (its ticket is taken afterwards).
        for (uint32_t it = 0;; ++it) {
            const uint32_t par = it & 1;
            if (C.tid == 0) {
                const bool completed = sh.pending && sh.done_old + 1 == p.epoch_b;
                sh.pending = 0;
                unsigned long long i = ~0ull;
                if (!completed) {
                    // the ticket and both control words are fetched together
                    // (three round trips in flight, not one after another)
#if ADSB_TICKET_PAIR
                    // two consecutive tickets per fetch: every other sample
                    // skips the global atomic (a held spare above the stop is
                    // dropped; its epoch is never folded)
                    if (sh.spare_tick != ~0ull) {
                        i = sh.spare_tick;
                        sh.spare_tick = ~0ull;
                    } else {
                        i = atomicAdd(p.ctl + kCtlTicket, 2ull);
                        sh.spare_tick = i + 1;
                    }
#else
                    i = atomicAdd(p.ctl + kCtlTicket, 1ull);
#endif
                    unsigned long long stop_v = vload(p.ctl + kCtlStop), fold_v = vload(p.ctl + kCtlFolded);
                    const unsigned long long e = i / p.epoch_b;
                    for (;;) {
                        if (e > stop_v || e >= p.max_epochs) {
                            i = ~0ull;
                            break;
                        }
                        if (e < fold_v + p.ring_k) break;
                        __nanosleep(200);
                        stop_v = vload(p.ctl + kCtlStop);
                        fold_v = vload(p.ctl + kCtlFolded);
                    }
                }
                sh.tick[par] = i;
                sh.tflag[par] = completed ? 1u : 0u;
            }
            __syncthreads();
            const unsigned long long item = sh.tick[par];
            if (sh.tflag[par]) {
                fold_chain(C, p);
                continue;
            }
            if (item == ~0ull) break;
            const uint32_t k = static_cast<uint32_t>((item / p.epoch_b) % p.ring_k);
            SplitMix64 rng(reseed(p.seed, item));
            if (C.tid == 0) sh.n_samples += 1;
            const uint32_t rec0 = sh.recorded;
            one_sample<kMode, kGlobalOnly, kVec>(C, p, rng, k, gtag);
            if (C.tid == 0) {
                if (p.audit && item < p.max_epochs * p.epoch_b)
                    p.audit[item] = (sh.recorded - rec0) | (sh.last_d << 16);
                // release: this sample's counts and list entries become visible
                // before its completion does. A release atomic, not
                // __threadfence(): the full fence also invalidates the SM's L1
                // (CCTL.IVALL) after every sample, losing adjacency reuse.
                unsigned long long old;
                asm volatile("atom.add.release.gpu.global.u64 %0, [%1], %2;"
                             : "=l"(old)
                             : "l"(p.ctl + kCtlDone + k), "l"(1ull)
                             : "memory");
                sh.done_old = old;
                sh.pending = 1;
            }
        }
    }
    ADSB_PHASE_MARK(k1);
    ADSB_PHASE_ADD(4, k1 - k0);
    __syncthreads();  // low-degree expansions add edge counts from every warp
    if (C.tid == 0) {
        unsigned long long e = 0, r = 0, b = 0;
        for (uint32_t w = 0; w < kBT / 32; ++w) {
            e += sh.st_edges[w];
            r += sh.st_rebuild[w];
            b += sh.st_back[w];
        }
        atomicAdd(p.stats + kStatEdges, e + r + b);
        atomicAdd(p.stats + kStatRebuildEdges, r);
        atomicAdd(p.stats + kStatBacktrackEdges, b);
        atomicAdd(p.stats + kStatVertices, sh.st_verts);
    }
    if (C.tid == 0) {
        if (kGlobalOnly) p.slot_tag[slot] = gtag;
        atomicAdd(p.stats + kStatSamples, sh.n_samples);
        atomicAdd(p.stats + kStatFallbacks, sh.n_fallbacks);
        if (sh.n_errors) atomicAdd(p.stats + kStatErrors, sh.n_errors);
        if (sh.st_degen) atomicAdd(p.stats + kStatDegenerate, sh.st_degen);
    }
}
