/*
 * gen.c — the benchmark graphs for the CPU side of the measurement.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h). bench.py's reference arm must not
 * load the product library (libadsb.so), so the seeded synthetic stand-ins for
 * BASELINE.json's configs are generated here a second time, independently of
 * csrc/graph_host.cpp, and tests/test_oracle.py::test_generators_match_product
 * checks that both produce the identical edge sequence. The output for the
 * reference is its own public ingestion input: dense ids in first-appearance
 * order (graph.hpp:98-123's interning), which Graph::from_edges
 * (graph.hpp:35-58) turns into the same CSR as parse_edge_list would.
 *
 * Procedures:
 *   gnm   — tests/acceptance.cpp:34-46: distinct unordered pairs drawn with
 *           next_below(n) until m are collected, emitted sorted (u < v);
 *   rmat  — edge i draws `scale` quadrant choices from stream reseed(seed, i),
 *           each a 53-bit uniform, MSB first; self-loops dropped, duplicates kept;
 *   ba    — K_{m+1}, then each new vertex picks m distinct targets from the
 *           endpoint list (degree-proportional), emitted in pick order;
 *   grid  — row-major lattice, right then down edge per vertex, each dropped
 *           when next() < p * 2^64;
 *   lcc   — union-find (root = component minimum), the largest component,
 *           lowest root on ties; edges kept in generation order.
 */
#define _GNU_SOURCE
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle.h"

typedef struct {
    uint64_t *p;
    uint64_t len, cap; /* in u64 words */
} vec64;

static void v_push2(vec64 *v, uint64_t a, uint64_t b) {
    if (v->len + 2 > v->cap) {
        v->cap = v->cap ? v->cap * 2 : 1024;
        v->p = realloc(v->p, v->cap * sizeof(uint64_t));
    }
    v->p[v->len++] = a;
    v->p[v->len++] = b;
}

static int cmp_pair(const void *x, const void *y) {
    const uint64_t *a = x, *b = y;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
    return 0;
}

static vec64 gen_gnm(uint32_t n, uint64_t m, uint64_t seed) {
    vec64 out = {0};
    if (n < 2 || m > (uint64_t)n * (n - 1) / 2) return out;
    /* open-addressing set of (u << 32 | v) */
    uint64_t cap = 16;
    while (cap < 4 * m + 16) cap <<= 1;
    uint64_t *set = malloc(cap * sizeof(uint64_t));
    memset(set, 0xFF, cap * sizeof(uint64_t));
    uint64_t rng = seed, have = 0;
    while (have < m) {
        uint32_t u = (uint32_t)or_next_below(&rng, n);
        uint32_t v = (uint32_t)or_next_below(&rng, n);
        if (u == v) continue;
        if (u > v) {
            const uint32_t t = u;
            u = v;
            v = t;
        }
        const uint64_t key = ((uint64_t)u << 32) | v;
        uint64_t h = or_mix64(key) & (cap - 1);
        while (set[h] != UINT64_MAX && set[h] != key) h = (h + 1) & (cap - 1);
        if (set[h] == UINT64_MAX) {
            set[h] = key;
            v_push2(&out, u, v);
            ++have;
        }
    }
    free(set);
    qsort(out.p, out.len / 2, 2 * sizeof(uint64_t), cmp_pair);
    return out;
}

typedef struct {
    uint64_t lo, hi, seed;
    uint32_t scale;
    double a, ab, abc;
    uint64_t *raw;
    uint8_t *loop;
} rmat_job;

static void *rmat_worker(void *arg) {
    const rmat_job *j = arg;
    for (uint64_t i = j->lo; i < j->hi; ++i) {
        uint64_t rng = or_reseed(j->seed, i);
        uint64_t u = 0, v = 0;
        for (uint32_t bit = 0; bit < j->scale; ++bit) {
            const double r = (double)(or_next(&rng) >> 11) * 0x1.0p-53;
            const uint64_t bu = r >= j->ab ? 1 : 0;
            const uint64_t bv = ((r >= j->a && r < j->ab) || r >= j->abc) ? 1 : 0;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        j->raw[2 * i] = u;
        j->raw[2 * i + 1] = v;
        j->loop[i] = u == v;
    }
    return NULL;
}

static vec64 gen_rmat(uint32_t scale, uint32_t edge_factor, double a, double b, double c, uint64_t seed) {
    vec64 out = {0};
    if (scale < 1 || scale > 31) return out;
    const uint64_t m = (uint64_t)edge_factor << scale;
    uint64_t *raw = malloc(2 * m * sizeof(uint64_t));
    uint8_t *loop = malloc(m);
    enum { W = 16 };
    pthread_t tid[W];
    rmat_job jobs[W];
    for (int t = 0; t < W; ++t) {
        jobs[t] = (rmat_job){m * t / W, m * (t + 1) / W, seed, scale, a, a + b, a + b + c, raw, loop};
        pthread_create(&tid[t], NULL, rmat_worker, &jobs[t]);
    }
    for (int t = 0; t < W; ++t) pthread_join(tid[t], NULL);
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; ++i)
        if (!loop[i]) {
            raw[2 * k] = raw[2 * i];
            raw[2 * k + 1] = raw[2 * i + 1];
            ++k;
        }
    free(loop);
    out.p = raw;
    out.len = 2 * k;
    out.cap = 2 * m;
    return out;
}

static vec64 gen_ba(uint32_t n, uint32_t mp, uint64_t seed) {
    vec64 out = {0};
    if (mp < 1 || n <= mp) return out;
    const uint64_t total = (uint64_t)mp * (mp + 1) / 2 + (uint64_t)(n - mp - 1) * mp;
    out.cap = 2 * total;
    out.p = malloc(out.cap * sizeof(uint64_t));
    uint32_t *ends = malloc(2 * total * sizeof(uint32_t));
    uint64_t ne = 0;
    uint64_t rng = seed;
    for (uint32_t i = 0; i <= mp; ++i)
        for (uint32_t j = i + 1; j <= mp; ++j) {
            v_push2(&out, i, j);
            ends[ne++] = i;
            ends[ne++] = j;
        }
    uint32_t *picked = malloc(mp * sizeof(uint32_t));
    for (uint32_t v = mp + 1; v < n; ++v) {
        uint32_t k = 0;
        while (k < mp) {
            const uint32_t t = ends[or_next_below(&rng, ne)];
            int dup = 0;
            for (uint32_t j = 0; j < k; ++j) dup |= picked[j] == t;
            if (!dup) picked[k++] = t;
        }
        for (uint32_t j = 0; j < mp; ++j) {
            v_push2(&out, v, picked[j]);
            ends[ne++] = v;
            ends[ne++] = picked[j];
        }
    }
    free(picked);
    free(ends);
    return out;
}

static vec64 gen_grid(uint32_t w, uint32_t h, double p, uint64_t seed) {
    vec64 out = {0};
    if (w < 1 || h < 1 || !(p >= 0.0 && p < 1.0)) return out;
    const uint64_t thr = (uint64_t)(p * 18446744073709551616.0);
    uint64_t rng = seed;
    out.cap = 4ull * w * h + 2;
    out.p = malloc(out.cap * sizeof(uint64_t));
    for (uint32_t r = 0; r < h; ++r)
        for (uint32_t c = 0; c < w; ++c) {
            const uint64_t u = (uint64_t)r * w + c;
            if (c + 1 < w && or_next(&rng) >= thr) v_push2(&out, u, u + 1);
            if (r + 1 < h && or_next(&rng) >= thr) v_push2(&out, u, u + w);
        }
    return out;
}

static uint32_t uf_find(uint32_t *parent, uint32_t x) {
    while (parent[x] != x) x = parent[x] = parent[parent[x]];
    return x;
}

static void keep_lcc(vec64 *v) {
    const uint64_t m = v->len / 2;
    uint64_t max_id = 0;
    for (uint64_t i = 0; i < v->len; ++i)
        if (v->p[i] > max_id) max_id = v->p[i];
    uint32_t *parent = malloc((max_id + 1) * sizeof(uint32_t));
    uint8_t *present = calloc(max_id + 1, 1);
    uint32_t *size = calloc(max_id + 1, sizeof(uint32_t));
    for (uint64_t x = 0; x <= max_id; ++x) parent[x] = (uint32_t)x;
    for (uint64_t i = 0; i < m; ++i) {
        const uint32_t a = (uint32_t)v->p[2 * i], b = (uint32_t)v->p[2 * i + 1];
        if (a == b) continue;
        present[a] = present[b] = 1;
        const uint32_t ra = uf_find(parent, a), rb = uf_find(parent, b);
        if (ra != rb) parent[ra > rb ? ra : rb] = ra < rb ? ra : rb;
    }
    for (uint64_t x = 0; x <= max_id; ++x)
        if (present[x]) size[uf_find(parent, (uint32_t)x)]++;
    uint32_t best = 0;
    for (uint64_t x = 0; x <= max_id; ++x)
        if (size[x] > size[best]) best = (uint32_t)x;
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; ++i) {
        const uint32_t a = (uint32_t)v->p[2 * i], b = (uint32_t)v->p[2 * i + 1];
        if (a == b || uf_find(parent, a) != best) continue;
        v->p[2 * k] = a;
        v->p[2 * k + 1] = b;
        ++k;
    }
    v->len = 2 * k;
    free(parent);
    free(present);
    free(size);
}

/* kind: 0 gnm(n, m, seed), 1 rmat(scale, ef, a, b, c, seed), 2 ba(n, m, seed),
 * 3 grid(w, h, p, seed); lcc != 0 keeps the largest component (gnm, rmat, grid).
 * Returns the pairs (malloc'ed, 2 * *m_out words; free with or_free). */
uint64_t *or_gen_pairs(int kind, const double *params, int lcc, uint64_t *m_out) {
    vec64 v = {0};
    switch (kind) {
        case 0: v = gen_gnm((uint32_t)params[0], (uint64_t)params[1], (uint64_t)params[2]); break;
        case 1:
            v = gen_rmat((uint32_t)params[0], (uint32_t)params[1], params[2], params[3], params[4],
                         (uint64_t)params[5]);
            break;
        case 2: v = gen_ba((uint32_t)params[0], (uint32_t)params[1], (uint64_t)params[2]); break;
        case 3: v = gen_grid((uint32_t)params[0], (uint32_t)params[1], params[2], (uint64_t)params[3]); break;
        default: break;
    }
    if (lcc && kind != 2 && v.len) keep_lcc(&v);
    *m_out = v.len / 2;
    return v.p;
}

void or_free(void *p) { free(p); }

/* Dense ids in first-appearance order (graph.hpp:98-123 interning) written as
 * u32 n, u64 m, then m (u32, u32) pairs: Graph::from_edges' input. */
int or_write_dense_edges(const char *path, const uint64_t *pairs, uint64_t m) {
    uint64_t max_id = 0;
    for (uint64_t i = 0; i < 2 * m; ++i)
        if (pairs[i] > max_id) max_id = pairs[i];
    if (max_id > 0xFFFFFFFFull) return OR_EINVAL;
    uint32_t *remap = malloc((max_id + 1) * sizeof(uint32_t));
    memset(remap, 0xFF, (max_id + 1) * sizeof(uint32_t));
    uint32_t *dense = malloc(2 * m * sizeof(uint32_t));
    uint32_t n = 0;
    for (uint64_t i = 0; i < 2 * m; ++i) {
        uint32_t *r = &remap[pairs[i]];
        if (*r == UINT32_MAX) *r = n++;
        dense[i] = *r;
    }
    free(remap);
    FILE *f = fopen(path, "wb");
    if (!f) {
        free(dense);
        return OR_EINVAL;
    }
    int ok = fwrite(&n, sizeof n, 1, f) == 1 && fwrite(&m, sizeof m, 1, f) == 1 &&
             fwrite(dense, sizeof(uint32_t), 2 * m, f) == 2 * m;
    ok = (fclose(f) == 0) && ok;
    free(dense);
    return ok ? OR_OK : OR_EINVAL;
}
