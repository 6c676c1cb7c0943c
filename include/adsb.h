/*
 * adsb.h — C ABI of the B200-native KADABRA adaptive-sampling engine
 * (libadsb.so, built from paper_1903_09422_b200/csrc/).
 *
 * This is the drop-in boundary for the reference's hot path. Plain pointers and
 * sizes only; no torch or CUDA types. Every entry point returns an adsb_status
 * and, on failure, leaves a message in the calling thread's adsb_last_error().
 * Status codes map 1:1 onto the reference's exception types:
 *   ADSB_ERR_INVALID_ARGUMENT  std::invalid_argument (kadabra.hpp:310, :32-33, :43-46,
 *                              engine.hpp:97-105, graph.hpp:43-44)
 *   ADSB_ERR_DOMAIN            std::domain_error     (kadabra.hpp:69-75, :135)
 *   ADSB_ERR_PARSE             adsamp::ParseError    (graph.hpp:85-87)
 *   ADSB_ERR_LOGIC             std::logic_error      (engine.hpp:471-472, :632-633)
 *   ADSB_ERR_RUNTIME/CUDA/NCCL std::runtime_error    (file I/O, device and NCCL failures)
 * Reference paths are relative to /root/reference/proj/include/adsamp/.
 *
 * Output buffers are caller-allocated. The library owns device memory and
 * streams. One in-flight call per graph handle. There is no CPU fallback: the
 * compute entry points fail with ADSB_ERR_CUDA when no CUDA device is usable.
 */
#ifndef ADSB_H
#define ADSB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ADSB_ABI_VERSION 2

typedef enum {
    ADSB_OK = 0,
    ADSB_ERR_INVALID_ARGUMENT = 1,
    ADSB_ERR_DOMAIN = 2,
    ADSB_ERR_PARSE = 3,
    ADSB_ERR_LOGIC = 4,
    ADSB_ERR_RUNTIME = 5,
    ADSB_ERR_CUDA = 6,
    ADSB_ERR_NCCL = 7
} adsb_status;

/* engine.hpp:63 enum class Variant. On the GPU, `indexed` (and `sequential`,
 * which run_sequential keys as one stream, engine.hpp:238 — not bit-comparable)
 * run the deterministic frame pipeline. `barrier`, `local` and `shared` run
 * cumulative epochs (the stop rule on the running total after every epoch):
 *   shared, local  epochs of epoch_samples (default 1024) samples; sample i
 *                  drawn from stream_rng(seed, i). One GPU: one persistent
 *                  kernel folds epochs in order. Several GPUs: sample indices
 *                  are sharded, each rank's per-sample increments are
 *                  all-gathered and every rank folds them in index order, so
 *                  tau and the counts equal the one-GPU run's at any GPU count;
 *   barrier        rounds of check_interval samples (run_barrier's N,
 *                  engine.hpp:267-341) unless epoch_samples is set; several
 *                  GPUs split each round and all-reduce the n-length count
 *                  vector (NCCL) before every check. */
typedef enum {
    ADSB_VARIANT_SEQUENTIAL = 0,
    ADSB_VARIANT_BARRIER = 1,
    ADSB_VARIANT_LOCAL = 2,
    ADSB_VARIANT_SHARED = 3,
    ADSB_VARIANT_INDEXED = 4
} adsb_variant;

typedef enum { ADSB_REASON_EPS_CONVERGED = 0, ADSB_REASON_OMEGA_REACHED = 1, ADSB_REASON_CAPPED = 2 } adsb_reason;

typedef struct adsb_graph adsb_graph; /* graph.hpp:29-76 Graph (+ ParsedGraph::original_ids) */
typedef struct adsb_comm adsb_comm;   /* one rank per GPU: NCCL or host-callback transport */

typedef enum { ADSB_REDUCE_SUM = 0, ADSB_REDUCE_MAX = 1, ADSB_REDUCE_MIN = 2 } adsb_reduce_op;

/* Host transport for adsb_comm_init_host: collectives over HOST memory supplied
 * by the caller (e.g. torch.distributed with gloo), called from the thread
 * that called adsb_estimate_bc, in the same order on every rank. Each returns
 * 0 on success. */
typedef struct {
    /* in place: buf[i] = op over ranks of buf[i] */
    int (*allreduce_u64)(void *user, uint64_t *buf, size_t count, int op /* adsb_reduce_op */);
    int (*allreduce_u32_sum)(void *user, uint32_t *buf, size_t count);
    /* recv[r * count + i] = rank r's send[i] */
    int (*allgather_u64)(void *user, const uint64_t *send, uint64_t *recv, size_t count);
} adsb_host_collectives;

/* engine.hpp:85-96 EngineConfig, plus the GPU pipeline knobs. */
typedef struct {
    uint32_t struct_size;        /* sizeof(adsb_config) */
    int32_t variant;             /* adsb_variant; default ADSB_VARIANT_INDEXED */
    uint32_t threads;            /* T: nominal thread count; only used for stop_epoch = P/T+1 (engine.hpp:562) */
    uint32_t frame_groups;       /* F: validated (1 <= F <= T for shared), otherwise unused on GPU */
    uint64_t check_interval;     /* N (engine.hpp:89); validated */
    double latency_exponent;     /* xi (engine.hpp:90); validated */
    uint64_t samples_per_frame;  /* spf (engine.hpp:91): deterministic frame size */
    uint64_t epoch_samples;      /* non-det: samples per epoch across all ranks (0 = auto) */
    uint64_t base_seed;          /* engine.hpp:95 */
    uint64_t max_cycles;         /* 0 = until the stopping rule; else stop after this many checks */
    int32_t device;              /* CUDA ordinal; -1 = current device */
    uint32_t flags;              /* reserved, must be 0 */
    adsb_comm *comm;             /* NULL = single GPU */
    /* engine.hpp:92-94 (indexed). bounded_memory != 0 caps the frames sampled
     * ahead of the ordered cutoff at (reservation_block + 1) per sampler team
     * (run_indexed's reserve_indices block, engine.hpp:137-144): less event
     * memory, more batches; results are identical. queue_high_water sets
     * adsb_stats.queue_high_water_exceeded. */
    uint32_t bounded_memory;
    uint32_t reservation_block;  /* a >= 1 */
    uint64_t queue_high_water;
} adsb_config;

/* kadabra.hpp:295-304 BcResult + engine.hpp:163-171 RunResult scalars. */
typedef struct {
    uint64_t tau;                /* RunResult::num */
    uint64_t check_cycles;       /* RunResult::check_cycles */
    uint64_t stop_epoch;         /* RunResult::stop_epoch (nominal T) */
    uint64_t total_samples;      /* samples drawn, incl. unconsumed ones */
    uint64_t omega;
    uint64_t diameter_bound;
    int32_t reason;              /* adsb_reason */
    uint32_t num_components;
    double preprocess_seconds;
    double ads_seconds;
    uint64_t edges_scanned;      /* adjacency entries read by the executed (bidirectional) sampler */
    uint64_t vertices_expanded;  /* frontier vertices expanded (one offsets pair each) */
    uint64_t kernel_launches;    /* adsb kernels launched during the ADS phase */
    double sampler_ms;           /* device time of the sampler kernels (CUDA events) */
    uint64_t rebuild_edges;      /* of edges_scanned: t-side DAG sigma rebuild */
    uint64_t backtrack_edges;    /* of edges_scanned: predecessor scans of the backtrack */
    uint64_t store_fallbacks;    /* samples redone with global-memory state (shared-memory table overflow) */
    uint64_t degenerate_steps;   /* backtrack steps whose sigma and every predecessor sigma were 0 mod 2^64
                                    (undefined in the reference) */
    /* engine.hpp:156-161 QueueStats, per sampler team: frames sampled ahead of
     * the in-order consumption point (deterministic batches / epoch ring) */
    uint64_t queue_max_depth;
    double queue_mean_depth;
    uint64_t queue_allocated;    /* frame slots the pipeline allocated */
    uint32_t queue_high_water_exceeded;
    uint32_t world;              /* ranks that took part */
} adsb_stats;

void adsb_config_init(adsb_config *cfg); /* reference defaults (engine.hpp:85-96) */
const char *adsb_last_error(void);
int adsb_abi_version(void);

/* ---- graph (graph.hpp) ---------------------------------------------------- */
/* parse_edge_list (graph.hpp:93-131): first-appearance remap, '%'/'#' comments */
adsb_status adsb_graph_parse_text(const char *text, uint64_t len, adsb_graph **out);
adsb_status adsb_graph_parse_file(const char *path, adsb_graph **out);
/* the same semantics on already tokenised (id, id) records, 2*m entries */
adsb_status adsb_graph_from_pairs(const uint64_t *pairs, uint64_t m, adsb_graph **out);
/* Graph::from_edges (graph.hpp:35-58), 2*m dense endpoints */
adsb_status adsb_graph_from_edges(uint32_t n, const uint32_t *edges, uint64_t m, adsb_graph **out);
/* an existing CSR (offsets n+1, neighbours offsets[n]); must satisfy the Graph invariants */
adsb_status adsb_graph_from_csr(uint32_t n, const uint64_t *offsets, const uint32_t *neighbors,
                                adsb_graph **out);
void adsb_graph_destroy(adsb_graph *g);
/* Binary CSR cache: the graph exactly as ingested (dense ids, ascending
 * adjacency, original ids), written and read with parallel I/O and a
 * checksum; a damaged or truncated file fails with ADSB_ERR_PARSE. */
adsb_status adsb_graph_save(const adsb_graph *g, const char *path);
adsb_status adsb_graph_load(const char *path, adsb_graph **out);
adsb_status adsb_graph_info(const adsb_graph *g, uint32_t *n, uint64_t *nnz);
adsb_status adsb_graph_copy_csr(const adsb_graph *g, uint64_t *offsets, uint32_t *neighbors);
adsb_status adsb_graph_copy_original_ids(const adsb_graph *g, uint64_t *out);
/* serialize_edge_list (graph.hpp:140-144) into a caller buffer; *len in/out */
adsb_status adsb_graph_serialize(const adsb_graph *g, char *buf, uint64_t *len);

/* ---- preprocessing on the device (graph.hpp:153-214) ----------------------- */
adsb_status adsb_connected_components(const adsb_graph *g, int device, uint32_t *labels,
                                      uint32_t *num_components);
adsb_status adsb_eccentricity(const adsb_graph *g, int device, uint32_t source, uint64_t *out);
adsb_status adsb_diameter_upper_bound(const adsb_graph *g, int device, uint64_t *out);

/* ---- scalar rules (host; kadabra.hpp:30-91, engine.hpp:110-116, :137-144) --- */
adsb_status adsb_compute_omega(uint64_t diameter_bound, double eps, double delta, double c,
                               uint64_t *out);
adsb_status adsb_f_bound(double b, double delta_l, uint64_t omega, uint64_t tau, double *out);
adsb_status adsb_g_bound(double b, double delta_u, uint64_t omega, uint64_t tau, double *out);
adsb_status adsb_check_budget(uint64_t check_interval, uint32_t threads, double xi, uint64_t *out);
adsb_status adsb_reserve_indices(uint64_t claim, uint32_t threads, uint32_t a, uint64_t *out /* a+1 */);
/* stopping rule kadabra_check (kadabra.hpp:133-151) on host counts, uniform deltas */
adsb_status adsb_kadabra_check(const uint64_t *data, uint64_t n, uint64_t num, uint64_t omega,
                               double eps, double delta, int *stop);

/* ---- the drop-in: kadabra::estimate_bc (kadabra.hpp:308-348) ---------------- */
adsb_status adsb_estimate_bc(const adsb_graph *g, double epsilon, double delta,
                             const adsb_config *cfg, double *scores /* n, nullable */,
                             uint64_t *counts /* n, nullable */, adsb_stats *stats /* nullable */);

/* ---- sampler-level parity hook --------------------------------------------- */
/* Increments of frames [first, first+count), each = spf samples drawn from
 * stream_rng(seed, p) (engine.hpp:595-610, kadabra.hpp:250-258). frame_offsets
 * has count+1 entries; incs receives at most cap ids (t->s order per sample). */
adsb_status adsb_sample_frames(const adsb_graph *g, int device, uint64_t seed, uint64_t spf,
                               uint64_t first, uint64_t count, uint64_t *frame_offsets,
                               uint32_t *incs, uint64_t cap);

/* ---- validation: exact BC on the device (Brandes, f64) ---------------------- */
/* Exact betweenness of every vertex, normalised by n(n-1) like estimate_bc's
 * scores: the check the reference makes against ApspOracle / Brandes
 * (tests/test_util.hpp:164-206, tests/acceptance.cpp:60-101), on the GPU so
 * that it reaches graphs of C2's size. device_ms (nullable) receives the
 * kernel time. */
adsb_status adsb_exact_bc(const adsb_graph *g, int device, double *bc /* n */, double *device_ms);
/* ---- multi-GPU (one process per GPU, NCCL over NVLink) ---------------------- */
adsb_status adsb_comm_unique_id(uint8_t id[128]);
adsb_status adsb_comm_init(int nranks, int rank, const uint8_t id[128], int device, adsb_comm **out);
/* the same ranks over caller-supplied host collectives (see adsb_host_collectives);
 * ops is copied, user is passed back to every call */
adsb_status adsb_comm_init_host(int nranks, int rank, int device, const adsb_host_collectives *ops, void *user,
                                adsb_comm **out);
void adsb_comm_destroy(adsb_comm *comm);

/* ---- synthetic inputs (BASELINE.json configs) ---------------- */
/* Each returns 2*m original ids in edge-list order, largest connected component
 * only when lcc != 0; free with adsb_free. */
adsb_status adsb_gen_gnm(uint32_t n, uint64_t m, uint64_t seed, int lcc, uint64_t **pairs, uint64_t *count);
adsb_status adsb_gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c,
                          uint64_t seed, int lcc, uint64_t **pairs, uint64_t *count);
adsb_status adsb_gen_ba(uint32_t n, uint32_t m_per, uint64_t seed, uint64_t **pairs, uint64_t *count);
adsb_status adsb_gen_grid(uint32_t width, uint32_t height, double p_drop, uint64_t seed, int lcc,
                          uint64_t **pairs, uint64_t *count);
adsb_status adsb_write_edge_list(const char *path, const uint64_t *pairs, uint64_t m);
void adsb_free(void *p);

#ifdef __cplusplus
}
#endif
#endif
