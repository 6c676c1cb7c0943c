/*
 * oracle.c — CPU restatement of the reference KADABRA sampling path.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h). Plain C11 + unsigned __int128,
 * compiled with -ffp-contract=off so the FP64 stopping rule is evaluated in
 * the reference's expression order with no FMA contraction, exactly like the
 * reference's x86-64 -O3 build (proj/CMakeLists.txt:6-8, no -march).
 *
 * Every function cites the reference line it restates; paths are relative to
 * /root/reference/proj/include/adsamp/.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <ctype.h>
#include <math.h>
#include <pthread.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define SET_ERR(...)                                   \
    do {                                               \
        if (err && errlen) snprintf(err, errlen, __VA_ARGS__); \
    } while (0)

/* ------------------------------------------------------------------------ */
/* rng.hpp:12-19 mix64, :27-30 next, :33-44 next_below, :53-55 reseed        */
/* ------------------------------------------------------------------------ */
uint64_t or_mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

uint64_t or_next(uint64_t *state) {
    *state += 0x9E3779B97F4A7C15ull;
    return or_mix64(*state);
}

uint64_t or_next_below(uint64_t *state, uint64_t bound) {
    unsigned __int128 m = (unsigned __int128)or_next(state) * bound;
    uint64_t lo = (uint64_t)m;
    if (lo < bound) {
        const uint64_t threshold = (0 - bound) % bound;
        while (lo < threshold) {
            m = (unsigned __int128)or_next(state) * bound;
            lo = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

uint64_t or_reseed(uint64_t base_seed, uint64_t index) {
    return or_mix64(base_seed ^ (index * 0x9E3779B97F4A7C15ull));
}

/* ------------------------------------------------------------------------ */
/* graph.hpp:35-58 Graph::from_edges: drop self-loops, symmetrise, sort,     */
/* unique -> CSR with ascending adjacency                                    */
/* ------------------------------------------------------------------------ */
static void radix_sort_u64(uint64_t *a, uint64_t *tmp, uint64_t len) {
    for (int pass = 0; pass < 4; ++pass) {
        const int shift = pass * 16;
        uint64_t *cnt = calloc(65537, sizeof(uint64_t));
        for (uint64_t i = 0; i < len; ++i) cnt[((a[i] >> shift) & 0xFFFF) + 1]++;
        for (int b = 0; b < 65536; ++b) cnt[b + 1] += cnt[b];
        for (uint64_t i = 0; i < len; ++i) tmp[cnt[(a[i] >> shift) & 0xFFFF]++] = a[i];
        memcpy(a, tmp, len * sizeof(uint64_t));
        free(cnt);
    }
}

static int build_csr(uint32_t n, const uint32_t *edges, uint64_t m, or_graph *g, char *err,
                     size_t errlen) {
    uint64_t *dir = malloc((2 * m + 1) * sizeof(uint64_t));
    uint64_t *tmp = malloc((2 * m + 1) * sizeof(uint64_t));
    if (!dir || !tmp) {
        free(dir);
        free(tmp);
        SET_ERR("out of memory");
        return OR_ENOMEM;
    }
    uint64_t k = 0;
    for (uint64_t i = 0; i < m; ++i) {
        const uint32_t u = edges[2 * i], v = edges[2 * i + 1];
        if (u == v) continue;
        if (u >= n || v >= n) {
            free(dir);
            free(tmp);
            SET_ERR("edge endpoint out of range");
            return OR_EINVAL;
        }
        dir[k++] = ((uint64_t)u << 32) | v;
        dir[k++] = ((uint64_t)v << 32) | u;
    }
    radix_sort_u64(dir, tmp, k);
    uint64_t w = 0;
    for (uint64_t i = 0; i < k; ++i)
        if (i == 0 || dir[i] != dir[i - 1]) dir[w++] = dir[i];
    free(tmp);
    g->n = n;
    g->nnz = w;
    g->offsets = calloc((size_t)n + 1, sizeof(uint64_t));
    g->nbrs = malloc((w + 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < w; ++i) {
        g->offsets[(dir[i] >> 32) + 1]++;
        g->nbrs[i] = (uint32_t)dir[i];
    }
    for (uint32_t u = 0; u < n; ++u) g->offsets[u + 1] += g->offsets[u];
    free(dir);
    return OR_OK;
}

int or_graph_from_edges(uint32_t n, const uint32_t *edges, uint64_t m, or_graph *g, char *err,
                        size_t errlen) {
    memset(g, 0, sizeof(*g));
    return build_csr(n, edges, m, g, err, errlen);
}

void or_graph_free(or_graph *g) {
    free(g->offsets);
    free(g->nbrs);
    free(g->original_ids);
    memset(g, 0, sizeof(*g));
}

/* First-appearance interning, graph.hpp:98-104 (unordered_map try_emplace). */
typedef struct {
    uint64_t *keys;
    uint32_t *vals;
    uint8_t *used;
    uint64_t cap, size;
    uint64_t *ids;  /* dense -> original */
    uint64_t ids_cap;
} intern_map;

static uint64_t hash_u64(uint64_t x) { return or_mix64(x + 0x9E3779B97F4A7C15ull); }

static void im_init(intern_map *im) {
    memset(im, 0, sizeof(*im));
    im->cap = 1024;
    im->keys = malloc(im->cap * sizeof(uint64_t));
    im->vals = malloc(im->cap * sizeof(uint32_t));
    im->used = calloc(im->cap, 1);
    im->ids_cap = 1024;
    im->ids = malloc(im->ids_cap * sizeof(uint64_t));
}

static void im_free(intern_map *im) {
    free(im->keys);
    free(im->vals);
    free(im->used);
    free(im->ids);
}

static uint32_t im_intern(intern_map *im, uint64_t key) {
    if (2 * (im->size + 1) > im->cap) {
        uint64_t ncap = im->cap * 2;
        uint64_t *nk = malloc(ncap * sizeof(uint64_t));
        uint32_t *nv = malloc(ncap * sizeof(uint32_t));
        uint8_t *nu = calloc(ncap, 1);
        for (uint64_t i = 0; i < im->cap; ++i) {
            if (!im->used[i]) continue;
            uint64_t h = hash_u64(im->keys[i]) & (ncap - 1);
            while (nu[h]) h = (h + 1) & (ncap - 1);
            nu[h] = 1;
            nk[h] = im->keys[i];
            nv[h] = im->vals[i];
        }
        free(im->keys);
        free(im->vals);
        free(im->used);
        im->keys = nk;
        im->vals = nv;
        im->used = nu;
        im->cap = ncap;
    }
    uint64_t h = hash_u64(key) & (im->cap - 1);
    while (im->used[h]) {
        if (im->keys[h] == key) return im->vals[h];
        h = (h + 1) & (im->cap - 1);
    }
    im->used[h] = 1;
    im->keys[h] = key;
    im->vals[h] = (uint32_t)im->size;
    if (im->size == im->ids_cap) {
        im->ids_cap *= 2;
        im->ids = realloc(im->ids, im->ids_cap * sizeof(uint64_t));
    }
    im->ids[im->size] = key;
    return (uint32_t)im->size++;
}

static int finish_parsed(intern_map *im, uint32_t *edges, uint64_t m, or_graph *g, char *err,
                         size_t errlen) {
    if (im->size == 0) {
        SET_ERR("no vertices found in edge list");
        return OR_EPARSE;
    }
    int rc = build_csr((uint32_t)im->size, edges, m, g, err, errlen);
    if (rc) return rc;
    g->original_ids = malloc(im->size * sizeof(uint64_t));
    memcpy(g->original_ids, im->ids, im->size * sizeof(uint64_t));
    return OR_OK;
}

int or_graph_from_pairs(const uint64_t *pairs, uint64_t m, or_graph *g, char *err, size_t errlen) {
    memset(g, 0, sizeof(*g));
    intern_map im;
    im_init(&im);
    uint32_t *edges = malloc((2 * m + 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < m; ++i) {
        if (pairs[2 * i] > 0xFFFFFFFFull || pairs[2 * i + 1] > 0xFFFFFFFFull) {
            SET_ERR("pair %llu: vertex id exceeds 2^32-1", (unsigned long long)(i + 1));
            free(edges);
            im_free(&im);
            return OR_EPARSE;
        }
        edges[2 * i] = im_intern(&im, pairs[2 * i]);
        edges[2 * i + 1] = im_intern(&im, pairs[2 * i + 1]);
    }
    int rc = finish_parsed(&im, edges, m, g, err, errlen);
    free(edges);
    im_free(&im);
    return rc;
}

/* std::istream >> uint64_t as libstdc++ num_get does it: skip isspace, optional
 * sign, at least one decimal digit, overflow -> failure, '-' negates mod 2^64. */
static int is_space(char c) {
    return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

static int get_u64(const char **pp, const char *e, uint64_t *out) {
    const char *p = *pp;
    while (p < e && is_space(*p)) ++p;
    int neg = 0;
    if (p < e && (*p == '+' || *p == '-')) {
        neg = *p == '-';
        ++p;
    }
    if (p == e || !(*p >= '0' && *p <= '9')) {
        *pp = p;
        return 0;
    }
    uint64_t v = 0;
    int overflow = 0;
    while (p < e && *p >= '0' && *p <= '9') {
        const uint64_t d = (uint64_t)(*p - '0');
        if (v > (UINT64_MAX - d) / 10) overflow = 1;
        v = v * 10 + d;
        ++p;
    }
    *pp = p;
    if (overflow) return 0;
    *out = neg ? (uint64_t)(0 - v) : v;
    return 1;
}

/* graph.hpp:93-131 parse_edge_list */
int or_parse_edge_list_text(const char *text, size_t len, or_graph *g, char *err, size_t errlen) {
    memset(g, 0, sizeof(*g));
    intern_map im;
    im_init(&im);
    uint64_t ecap = 1024, m = 0;
    uint32_t *edges = malloc(ecap * 2 * sizeof(uint32_t));
    const char *p = text, *end = text + len;
    uint64_t line_no = 0;
    int rc = OR_OK;
    while (p < end) {
        const char *nl = memchr(p, '\n', (size_t)(end - p));
        const char *le = nl ? nl : end;
        ++line_no;
        const char *q = p;
        while (q < le && (*q == ' ' || *q == '\t' || *q == '\r')) ++q;
        if (q == le || *q == '%' || *q == '#') {
            p = nl ? nl + 1 : end;
            continue;
        }
        const char *c = p;
        uint64_t a = 0, b = 0;
        if (!get_u64(&c, le, &a) || !get_u64(&c, le, &b)) {
            SET_ERR("line %llu: expected two vertex ids", (unsigned long long)line_no);
            rc = OR_EPARSE;
            break;
        }
        while (c < le && is_space(*c)) ++c;
        if (c < le) {
            const char *te = c;
            while (te < le && !is_space(*te)) ++te;
            SET_ERR("line %llu: trailing token '%.*s'", (unsigned long long)line_no, (int)(te - c), c);
            rc = OR_EPARSE;
            break;
        }
        if (a > 0xFFFFFFFFull || b > 0xFFFFFFFFull) {
            SET_ERR("line %llu: vertex id exceeds 2^32-1", (unsigned long long)line_no);
            rc = OR_EPARSE;
            break;
        }
        if (m == ecap) {
            ecap *= 2;
            edges = realloc(edges, ecap * 2 * sizeof(uint32_t));
        }
        edges[2 * m] = im_intern(&im, a);
        edges[2 * m + 1] = im_intern(&im, b);
        ++m;
        p = nl ? nl + 1 : end;
    }
    if (rc == OR_OK) rc = finish_parsed(&im, edges, m, g, err, errlen);
    free(edges);
    im_free(&im);
    return rc;
}

int or_parse_edge_list_file(const char *path, or_graph *g, char *err, size_t errlen) {
    FILE *f = fopen(path, "rb");
    if (!f) {
        SET_ERR("cannot open graph file '%s'", path);
        return OR_EINVAL;
    }
    fseek(f, 0, SEEK_END);
    long sz = ftell(f);
    fseek(f, 0, SEEK_SET);
    char *buf = malloc((size_t)sz + 1);
    size_t got = fread(buf, 1, (size_t)sz, f);
    fclose(f);
    int rc = or_parse_edge_list_text(buf, got, g, err, errlen);
    free(buf);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* graph.hpp:153-175 connected_components (stack DFS, labels in id order)    */
/* ------------------------------------------------------------------------ */
uint32_t or_connected_components(const or_graph *g, uint32_t *label) {
    const uint32_t n = g->n;
    for (uint32_t v = 0; v < n; ++v) label[v] = n;
    uint32_t *stack = malloc(((size_t)n + 1) * sizeof(uint32_t));
    uint32_t comps = 0;
    for (uint32_t s = 0; s < n; ++s) {
        if (label[s] != n) continue;
        const uint32_t c = comps++;
        label[s] = c;
        uint64_t top = 0;
        stack[top++] = s;
        while (top) {
            const uint32_t u = stack[--top];
            for (uint64_t e = g->offsets[u]; e < g->offsets[u + 1]; ++e) {
                const uint32_t v = g->nbrs[e];
                if (label[v] == n) {
                    label[v] = c;
                    stack[top++] = v;
                }
            }
        }
    }
    free(stack);
    return comps;
}

/* graph.hpp:178-197 eccentricity */
uint64_t or_eccentricity(const or_graph *g, uint32_t source) {
    uint32_t *dist = malloc(((size_t)g->n + 1) * sizeof(uint32_t));
    uint32_t *q = malloc(((size_t)g->n + 1) * sizeof(uint32_t));
    for (uint32_t v = 0; v < g->n; ++v) dist[v] = UINT32_MAX;
    uint64_t head = 0, tail = 0, ecc = 0;
    dist[source] = 0;
    q[tail++] = source;
    while (head < tail) {
        const uint32_t u = q[head++];
        for (uint64_t e = g->offsets[u]; e < g->offsets[u + 1]; ++e) {
            const uint32_t v = g->nbrs[e];
            if (dist[v] == UINT32_MAX) {
                dist[v] = dist[u] + 1;
                ecc = dist[v];
                q[tail++] = v;
            }
        }
    }
    free(dist);
    free(q);
    return ecc;
}

/* graph.hpp:202-214 diameter_upper_bound: max over components of
 * 2*ecc(max-degree vertex, lowest id on ties) */
uint64_t or_diameter_upper_bound(const or_graph *g) {
    const uint32_t n = g->n;
    uint32_t *label = malloc(((size_t)n + 1) * sizeof(uint32_t));
    const uint32_t comps = or_connected_components(g, label);
    uint32_t *start = malloc(((size_t)comps + 1) * sizeof(uint32_t));
    for (uint32_t c = 0; c < comps; ++c) start[c] = n;
    for (uint32_t u = 0; u < n; ++u) {
        uint32_t *s = &start[label[u]];
        if (*s == n || (g->offsets[u + 1] - g->offsets[u]) > (g->offsets[*s + 1] - g->offsets[*s]))
            *s = u;
    }
    uint64_t bound = 0;
    for (uint32_t c = 0; c < comps; ++c) {
        const uint64_t b = 2 * or_eccentricity(g, start[c]);
        if (b > bound) bound = b;
    }
    free(label);
    free(start);
    return bound;
}

/* ------------------------------------------------------------------------ */
/* kadabra.hpp:41-53 compute_omega                                           */
/* ------------------------------------------------------------------------ */
int or_compute_omega(uint64_t diameter_bound, double eps, double delta, double c, uint64_t *omega) {
    if (!(eps > 0.0 && eps < 1.0)) return OR_EINVAL;
    if (!(delta > 0.0 && delta < 1.0)) return OR_EINVAL;
    const uint64_t vd = diameter_bound + 1;
    const uint64_t arg = vd > 4 ? vd - 2 : 2;
    const double log2_floor = (double)(63 - __builtin_clzll(arg));
    const double value = (c / (eps * eps)) * (log2_floor + 1.0 + log(1.0 / delta));
    *omega = (uint64_t)ceil(value);
    return OR_OK;
}

/* kadabra.hpp:59-67 f_kernel / g_kernel (expression order preserved) */
static double f_kernel(double b, double log_inv, double omega, double tau) {
    const double t = 1.0 / 3.0 - omega / tau;
    return (log_inv / tau) * (t + sqrt(t * t + 2.0 * b * omega / log_inv));
}

static double g_kernel(double b, double log_inv, double omega, double tau) {
    const double t = 1.0 / 3.0 + omega / tau;
    return (log_inv / tau) * (t + sqrt(t * t + 2.0 * b * omega / log_inv));
}

/* kadabra.hpp:69-91 f_bound / g_bound with the domain checks */
static int bound_domain(double b, double delta_v, uint64_t tau) {
    if (tau < 1) return OR_EDOMAIN;
    if (!(delta_v > 0.0 && delta_v < 1.0)) return OR_EDOMAIN;
    if (!(b >= 0.0 && b <= 1.0)) return OR_EDOMAIN;
    return OR_OK;
}

int or_f_bound(double b, double delta_v, uint64_t omega, uint64_t tau, double *out) {
    int rc = bound_domain(b, delta_v, tau);
    if (rc) return rc;
    *out = f_kernel(b, log(1.0 / delta_v), (double)omega, (double)tau);
    return OR_OK;
}

int or_g_bound(double b, double delta_v, uint64_t omega, uint64_t tau, double *out) {
    int rc = bound_domain(b, delta_v, tau);
    if (rc) return rc;
    *out = g_kernel(b, log(1.0 / delta_v), (double)omega, (double)tau);
    return OR_OK;
}

/* kadabra.hpp:133-144 kadabra_converged, uniform deltas (kadabra.hpp:30-36) */
static int converged(const uint64_t *data, uint64_t n, uint64_t num, uint64_t omega, double eps,
                     double log_inv) {
    const double omega_d = (double)omega, tau_d = (double)num;
    for (uint64_t v = 0; v < n; ++v) {
        const double b = (double)data[v] / tau_d;
        if (f_kernel(b, log_inv, omega_d, tau_d) > eps) return 0;
        if (g_kernel(b, log_inv, omega_d, tau_d) > eps) return 0;
    }
    return 1;
}

/* kadabra.hpp:148-151 kadabra_check */
int or_kadabra_check(const uint64_t *data, uint64_t n, uint64_t num, uint64_t omega, double eps,
                     double delta_v, int *stop) {
    if (num >= omega) {
        *stop = 1;
        return OR_OK;
    }
    if (num < 1) return OR_EDOMAIN;
    *stop = converged(data, n, num, omega, eps, log(1.0 / delta_v));
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* kadabra.hpp:157-258 PathScratch + sample_path_between + sample_path       */
/* (a u32 generation stamp replaces the 7-bit stamp; equivalent per          */
/*  test_kadabra.cpp:358-380)                                                */
/* ------------------------------------------------------------------------ */
typedef struct {
    uint32_t n;
    uint32_t gen;
    uint32_t *stamp;
    uint32_t *dist;
    uint64_t *sigma;
    uint32_t *queue;
    uint64_t edges_scanned;
    uint64_t vertices_expanded;
    uint64_t degenerate_steps;
} scratch_t;

void *or_scratch_new(uint32_t n) {
    scratch_t *s = calloc(1, sizeof(scratch_t));
    s->n = n;
    s->stamp = calloc((size_t)n + 1, sizeof(uint32_t));
    s->dist = calloc((size_t)n + 1, sizeof(uint32_t));
    s->sigma = calloc((size_t)n + 1, sizeof(uint64_t));
    s->queue = calloc((size_t)n + 1, sizeof(uint32_t));
    return s;
}

void or_scratch_free(void *p) {
    scratch_t *s = p;
    if (!s) return;
    free(s->stamp);
    free(s->dist);
    free(s->sigma);
    free(s->queue);
    free(s);
}

static uint32_t sample_between(const or_graph *g, scratch_t *sc, uint64_t *rng, uint32_t s,
                               uint32_t t, uint32_t *out) {
    if (++sc->gen == 0) {
        memset(sc->stamp, 0, (size_t)sc->n * sizeof(uint32_t));
        sc->gen = 1;
    }
    const uint32_t gen = sc->gen;
    uint32_t *dist = sc->dist, *queue = sc->queue, *stamp = sc->stamp;
    uint64_t *sigma = sc->sigma;
    uint64_t head = 0, tail = 0;
    stamp[s] = gen;
    dist[s] = 0;
    sigma[s] = 1;
    queue[tail++] = s;
    uint32_t t_dist = UINT32_MAX;
    /* kadabra.hpp:208-222 */
    for (; head < tail; ++head) {
        const uint32_t u = queue[head];
        if (dist[u] >= t_dist) break;
        sc->vertices_expanded++;
        sc->edges_scanned += g->offsets[u + 1] - g->offsets[u];
        for (uint64_t e = g->offsets[u]; e < g->offsets[u + 1]; ++e) {
            const uint32_t v = g->nbrs[e];
            if (stamp[v] != gen) {
                stamp[v] = gen;
                dist[v] = dist[u] + 1;
                sigma[v] = sigma[u];
                queue[tail++] = v;
                if (v == t) t_dist = dist[v];
            } else if (dist[v] == dist[u] + 1) {
                sigma[v] += sigma[u];
            }
        }
    }
    if (stamp[t] != gen) return 0;
    /* kadabra.hpp:227-242 sigma-weighted backtrack, ascending neighbours */
    uint32_t cur = t, len = 0;
    while (dist[cur] > 1) {
        uint64_t r = or_next_below(rng, sigma[cur]);
        uint32_t chosen = UINT32_MAX, first_pred = UINT32_MAX;
        for (uint64_t e = g->offsets[cur]; e < g->offsets[cur + 1]; ++e) {
            const uint32_t p = g->nbrs[e];
            sc->edges_scanned++;
            if (stamp[p] == gen && dist[p] + 1 == dist[cur]) {
                if (first_pred == UINT32_MAX) first_pred = p;
                if (r < sigma[p]) {
                    chosen = p;
                    break;
                }
                r -= sigma[p];
            }
        }
        if (chosen == UINT32_MAX) {
            /* Reached only when sigma[cur] and every predecessor's sigma are
             * 0 mod 2^64 (r = next_below(0) = 0). The reference then indexes
             * dist[] with UINT32_MAX (kadabra.hpp:230-241; it segfaults on C4,
             * frame 247 of seed 42). Defined here, and identically on the GPU:
             * take the first predecessor in ascending id order. */
            chosen = first_pred;
            sc->degenerate_steps++;
        }
        cur = chosen;
        out[len++] = cur;
    }
    return len;
}

uint32_t or_sample_path(const or_graph *g, const uint32_t *label, uint64_t *rng, uint32_t *out,
                        void *scratch) {
    const uint32_t n = g->n;
    const uint32_t s = (uint32_t)or_next_below(rng, n);
    uint32_t t = (uint32_t)or_next_below(rng, n - 1);
    if (t >= s) ++t;
    if (label[s] != label[t]) return 0;
    return sample_between(g, (scratch_t *)scratch, rng, s, t, out);
}

uint64_t or_sample_frame(const or_graph *g, const uint32_t *label, uint64_t seed, uint64_t position,
                         uint64_t spf, uint32_t *out, uint64_t cap, void *scratch) {
    uint64_t rng = or_reseed(seed, position);
    uint64_t len = 0;
    uint32_t *buf = malloc(((size_t)g->n + 1) * sizeof(uint32_t));
    for (uint64_t i = 0; i < spf; ++i) {
        const uint32_t k = or_sample_path(g, label, &rng, buf, scratch);
        for (uint32_t j = 0; j < k; ++j) {
            if (len < cap) out[len] = buf[j];
            ++len;
        }
    }
    free(buf);
    return len;
}

/* ------------------------------------------------------------------------ */
/* kadabra.hpp:308-348 estimate_bc with                                      */
/*   INDEXED: engine.hpp:490-643 run_indexed — frame p = spf samples from    */
/*            stream_rng(seed, p); fold in position order; check after each  */
/*            frame; tau = (P+1)*spf; stop_epoch = P/T + 1 (engine.hpp:562)  */
/*   EPOCH:   cumulative epoch semantics (run_barrier's cumulative check,    */
/*            engine.hpp:272,315): sample i keyed by stream_rng(seed, i),    */
/*            check every epoch_samples samples on the running total.        */
/* ------------------------------------------------------------------------ */
int or_estimate_bc(const or_graph *g, double eps, double delta, const or_config *cfg,
                   uint64_t *counts, double *scores, or_result *res, char *err, size_t errlen) {
    memset(res, 0, sizeof(*res));
    const uint32_t n = g->n;
    if (n == 0) {
        SET_ERR("graph has no vertices");
        return OR_EINVAL;
    }
    if (cfg->samples_per_frame < 1 || cfg->nominal_threads < 1) {
        SET_ERR("samples per frame must be >= 1");
        return OR_EINVAL;
    }
    if (cfg->mode == OR_MODE_EPOCH && cfg->epoch_samples < 1) {
        SET_ERR("epoch samples must be >= 1");
        return OR_EINVAL;
    }
    if (n == 1) { /* kadabra.hpp:314-317 */
        if (counts) counts[0] = 0;
        if (scores) scores[0] = 0.0;
        res->reason = OR_REASON_EPS;
        return OR_OK;
    }
    uint32_t *label = malloc((size_t)n * sizeof(uint32_t));
    or_connected_components(g, label);
    const uint64_t dub = or_diameter_upper_bound(g);
    uint64_t omega = 0;
    if (or_compute_omega(dub, eps, delta, cfg->c, &omega)) {
        SET_ERR("epsilon and delta must lie in (0,1)");
        free(label);
        return OR_EINVAL;
    }
    const double delta_v = delta / (2.0 * (double)n); /* kadabra.hpp:34 */
    const double log_inv = log(1.0 / delta_v);        /* kadabra.hpp:123 */

    uint64_t *data = calloc(n, sizeof(uint64_t));
    uint32_t *inc = malloc(((size_t)n + 1) * sizeof(uint32_t));
    scratch_t *sc = or_scratch_new(n);
    uint64_t num = 0, cycles = 0, stop_epoch = 0;
    int reason_capped = 0;
    const int epoch_mode = cfg->mode == OR_MODE_EPOCH;
    const uint64_t per_cycle = epoch_mode ? cfg->epoch_samples : 1;
    const uint64_t spf = epoch_mode ? 1 : cfg->samples_per_frame;
    uint64_t position = 0;
    for (;;) {
        for (uint64_t f = 0; f < per_cycle; ++f, ++position) {
            uint64_t rng = or_reseed(cfg->seed, position);
            for (uint64_t i = 0; i < spf; ++i) {
                const uint32_t k = or_sample_path(g, label, &rng, inc, sc);
                for (uint32_t j = 0; j < k; ++j) data[inc[j]]++;
                ++num;
            }
        }
        ++cycles;
        int stop = 0;
        or_kadabra_check(data, n, num, omega, eps, delta_v, &stop);
        if (stop) {
            stop_epoch = epoch_mode ? cycles : (cycles - 1) / cfg->nominal_threads + 1;
            break;
        }
        if (cfg->max_frames && cycles >= cfg->max_frames) {
            reason_capped = 1;
            stop_epoch = epoch_mode ? cycles : (cycles - 1) / cfg->nominal_threads + 1;
            break;
        }
    }
    res->tau = num;
    res->check_cycles = cycles;
    res->stop_epoch = stop_epoch;
    res->omega = omega;
    res->diameter_bound = dub;
    res->total_samples = num;
    res->edges_scanned = sc->edges_scanned;
    res->vertices_expanded = sc->vertices_expanded;
    res->degenerate_steps = sc->degenerate_steps;
    /* kadabra.hpp:339-343 */
    res->reason = OR_REASON_OMEGA;
    if (num >= 1 && converged(data, n, num, omega, eps, log_inv)) res->reason = OR_REASON_EPS;
    if (reason_capped) res->reason = OR_REASON_CAPPED;
    for (uint32_t v = 0; v < n; ++v) {
        if (counts) counts[v] = data[v];
        if (scores) scores[v] = num == 0 ? 0.0 : (double)data[v] / (double)num;
    }
    or_scratch_free(sc);
    free(inc);
    free(data);
    free(label);
    return OR_OK;
}

/* ------------------------------------------------------------------------ */
/* Exact normalized betweenness, the ApspOracle quantity                     */
/* (tests/test_util.hpp:186-205), computed with Brandes' accumulation.       */
/* ------------------------------------------------------------------------ */
typedef struct {
    const or_graph *g;
    double *bc;
    uint32_t begin, step;
} brandes_job;

static void *brandes_worker(void *arg) {
    brandes_job *job = arg;
    const or_graph *g = job->g;
    const uint32_t n = g->n;
    int32_t *dist = malloc((size_t)n * sizeof(int32_t));
    double *sigma = malloc((size_t)n * sizeof(double));
    double *dep = malloc((size_t)n * sizeof(double));
    uint32_t *order = malloc((size_t)n * sizeof(uint32_t));
    for (uint32_t s = job->begin; s < n; s += job->step) {
        for (uint32_t v = 0; v < n; ++v) {
            dist[v] = -1;
            sigma[v] = 0.0;
            dep[v] = 0.0;
        }
        uint64_t head = 0, tail = 0;
        dist[s] = 0;
        sigma[s] = 1.0;
        order[tail++] = s;
        while (head < tail) {
            const uint32_t u = order[head++];
            for (uint64_t e = g->offsets[u]; e < g->offsets[u + 1]; ++e) {
                const uint32_t v = g->nbrs[e];
                if (dist[v] < 0) {
                    dist[v] = dist[u] + 1;
                    order[tail++] = v;
                }
                if (dist[v] == dist[u] + 1) sigma[v] += sigma[u];
            }
        }
        for (uint64_t i = tail; i-- > 0;) {
            const uint32_t w = order[i];
            for (uint64_t e = g->offsets[w]; e < g->offsets[w + 1]; ++e) {
                const uint32_t v = g->nbrs[e];
                if (dist[v] == dist[w] - 1) dep[v] += sigma[v] / sigma[w] * (1.0 + dep[w]);
            }
            if (w != s) job->bc[w] += dep[w];
        }
    }
    free(dist);
    free(sigma);
    free(dep);
    free(order);
    return NULL;
}

void or_brandes(const or_graph *g, double *bc, int threads) {
    const uint32_t n = g->n;
    if (threads < 1) threads = 1;
    brandes_job *jobs = calloc((size_t)threads, sizeof(brandes_job));
    pthread_t *tids = calloc((size_t)threads, sizeof(pthread_t));
    for (int i = 0; i < threads; ++i) {
        jobs[i].g = g;
        jobs[i].bc = calloc(n ? n : 1, sizeof(double));
        jobs[i].begin = (uint32_t)i;
        jobs[i].step = (uint32_t)threads;
        pthread_create(&tids[i], NULL, brandes_worker, &jobs[i]);
    }
    for (uint32_t v = 0; v < n; ++v) bc[v] = 0.0;
    for (int i = 0; i < threads; ++i) {
        pthread_join(tids[i], NULL);
        for (uint32_t v = 0; v < n; ++v) bc[v] += jobs[i].bc[v];
        free(jobs[i].bc);
    }
    const double pairs = (double)n * (double)(n > 0 ? n - 1 : 0);
    if (pairs > 0)
        for (uint32_t v = 0; v < n; ++v) bc[v] /= pairs;
    free(jobs);
    free(tids);
}

/* ------------------------------------------------------------------------ */
/* or_estimate_bc_threads: or_estimate_bc's semantics (run_indexed,          */
/* engine.hpp:490-643, or the cumulative epochs) computed by T threads the   */
/* way run_indexed itself parallelises: frames are sampled independently     */
/* (each from its own stream_rng(seed, p), engine.hpp:595-610) and folded    */
/* strictly in position order by one thread, which evaluates kadabra_check   */
/* after every cycle (engine.hpp:544-565). Results are identical to          */
/* or_estimate_bc at any T. The check first evaluates f/g at the largest     */
/* count: if that vertex fails, kadabra_converged (kadabra.hpp:133-144) is   */
/* false exactly (it scans that vertex too); otherwise the full scan runs.   */
/* ------------------------------------------------------------------------ */
typedef struct {
    const or_graph *g;
    const uint32_t *label;
    uint64_t seed, spf, first, count;
    uint32_t **buf;      /* per frame: increments (malloc'ed) */
    uint64_t *len;       /* per frame */
    uint64_t next;       /* work counter (atomic) */
    scratch_t *sc;       /* per worker */
    uint32_t *tmp;       /* per worker, n + 1 */
} frames_job;

typedef struct {
    frames_job *job;
    int id;
} frames_worker_arg;

static void *frames_worker(void *argp) {
    frames_worker_arg *a = argp;
    frames_job *j = a->job;
    scratch_t *sc = &j->sc[a->id];
    uint32_t *tmp = j->tmp + (size_t)a->id * ((size_t)j->g->n + 1);
    for (;;) {
        const uint64_t i = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
        if (i >= j->count) break;
        uint64_t rng = or_reseed(j->seed, j->first + i);
        uint64_t cap = 64, len = 0;
        uint32_t *out = malloc(cap * sizeof(uint32_t));
        for (uint64_t k = 0; k < j->spf; ++k) {
            const uint32_t m = or_sample_path(j->g, j->label, &rng, tmp, sc);
            if (len + m > cap) {
                while (len + m > cap) cap *= 2;
                out = realloc(out, cap * sizeof(uint32_t));
            }
            memcpy(out + len, tmp, (size_t)m * sizeof(uint32_t));
            len += m;
        }
        j->buf[i] = out;
        j->len[i] = len;
    }
    return NULL;
}

int or_estimate_bc_threads(const or_graph *g, double eps, double delta, const or_config *cfg, int threads,
                           uint64_t *counts, double *scores, or_result *res, char *err, size_t errlen) {
    if (threads <= 1 || g->n <= 1) return or_estimate_bc(g, eps, delta, cfg, counts, scores, res, err, errlen);
    memset(res, 0, sizeof(*res));
    const uint32_t n = g->n;
    if (cfg->samples_per_frame < 1 || cfg->nominal_threads < 1) {
        SET_ERR("samples per frame must be >= 1");
        return OR_EINVAL;
    }
    if (cfg->mode == OR_MODE_EPOCH && cfg->epoch_samples < 1) {
        SET_ERR("epoch samples must be >= 1");
        return OR_EINVAL;
    }
    uint32_t *label = malloc((size_t)n * sizeof(uint32_t));
    or_connected_components(g, label);
    const uint64_t dub = or_diameter_upper_bound(g);
    uint64_t omega = 0;
    if (or_compute_omega(dub, eps, delta, cfg->c, &omega)) {
        SET_ERR("epsilon and delta must lie in (0,1)");
        free(label);
        return OR_EINVAL;
    }
    const double delta_v = delta / (2.0 * (double)n); /* kadabra.hpp:34 */
    const double log_inv = log(1.0 / delta_v);        /* kadabra.hpp:123 */
    const int epoch_mode = cfg->mode == OR_MODE_EPOCH;
    const uint64_t per_cycle = epoch_mode ? cfg->epoch_samples : 1; /* frames per check */
    const uint64_t spf = epoch_mode ? 1 : cfg->samples_per_frame;

    uint64_t *data = calloc(n, sizeof(uint64_t));
    scratch_t *sc = calloc((size_t)threads, sizeof(scratch_t));
    for (int t = 0; t < threads; ++t) {
        scratch_t *s = or_scratch_new(n);
        sc[t] = *s;
        free(s);
    }
    uint32_t *tmp = malloc((size_t)threads * ((size_t)n + 1) * sizeof(uint32_t));
    /* ~64 samples per worker per batch; frames past the stop are discarded */
    const uint64_t batch = (uint64_t)threads * (spf >= 64 ? 1 : 64 / spf);
    uint32_t **buf = calloc(batch, sizeof(uint32_t *));
    uint64_t *lens = calloc(batch, sizeof(uint64_t));
    pthread_t *tids = calloc((size_t)threads, sizeof(pthread_t));
    frames_worker_arg *args = calloc((size_t)threads, sizeof(frames_worker_arg));

    uint64_t num = 0, cycles = 0, stop_epoch = 0, position = 0, max_count = 0, in_cycle = 0;
    int reason_capped = 0, done = 0;
    while (!done) {
        frames_job job = {g, label, cfg->seed, spf, position, batch, buf, lens, 0, sc, tmp};
        for (int t = 0; t < threads; ++t) {
            args[t].job = &job;
            args[t].id = t;
            pthread_create(&tids[t], NULL, frames_worker, &args[t]);
        }
        for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
        for (uint64_t i = 0; i < batch; ++i) {
            if (!done) {
                for (uint64_t k = 0; k < lens[i]; ++k) {
                    const uint64_t c = ++data[buf[i][k]];
                    if (c > max_count) max_count = c;
                }
                num += spf;
                if (++in_cycle == per_cycle) {
                    in_cycle = 0;
                    ++cycles;
                    /* kadabra.hpp:148-151 */
                    int stop = num >= omega;
                    if (!stop) {
                        const double b = (double)max_count / (double)num;
                        if (f_kernel(b, log_inv, (double)omega, (double)num) <= eps &&
                            g_kernel(b, log_inv, (double)omega, (double)num) <= eps)
                            stop = converged(data, n, num, omega, eps, log_inv);
                    }
                    if (stop || (cfg->max_frames && cycles >= cfg->max_frames)) {
                        reason_capped = !stop;
                        stop_epoch = epoch_mode ? cycles : (cycles - 1) / cfg->nominal_threads + 1;
                        done = 1;
                    }
                }
            }
            free(buf[i]);
            buf[i] = NULL;
        }
        position += batch;
    }
    res->tau = num;
    res->check_cycles = cycles;
    res->stop_epoch = stop_epoch;
    res->omega = omega;
    res->diameter_bound = dub;
    res->total_samples = num;
    for (int t = 0; t < threads; ++t) {
        res->edges_scanned += sc[t].edges_scanned;
        res->vertices_expanded += sc[t].vertices_expanded;
        res->degenerate_steps += sc[t].degenerate_steps;
    }
    res->reason = OR_REASON_OMEGA;
    if (num >= 1 && converged(data, n, num, omega, eps, log_inv)) res->reason = OR_REASON_EPS;
    if (reason_capped) res->reason = OR_REASON_CAPPED;
    for (uint32_t v = 0; v < n; ++v) {
        if (counts) counts[v] = data[v];
        if (scores) scores[v] = num == 0 ? 0.0 : (double)data[v] / (double)num;
    }
    for (int t = 0; t < threads; ++t) {
        free(sc[t].stamp);
        free(sc[t].dist);
        free(sc[t].sigma);
        free(sc[t].queue);
    }
    free(sc);
    free(tmp);
    free(buf);
    free(lens);
    free(tids);
    free(args);
    free(data);
    free(label);
    return OR_OK;
}

/* Frames [first, first+count) by `threads` workers (or_sample_frame per frame,
 * engine.hpp:595-610 keying). lens[i] = increments of frame i; ids receives the
 * concatenation (up to cap). Returns the total number of increments. */
uint64_t or_sample_frames_threads(const or_graph *g, const uint32_t *label, uint64_t seed, uint64_t spf,
                                  uint64_t first, uint64_t count, int threads, uint64_t *lens, uint32_t *ids,
                                  uint64_t cap) {
    if (threads < 1) threads = 1;
    scratch_t *sc = calloc((size_t)threads, sizeof(scratch_t));
    for (int t = 0; t < threads; ++t) {
        scratch_t *s = or_scratch_new(g->n);
        sc[t] = *s;
        free(s);
    }
    uint32_t *tmp = malloc((size_t)threads * ((size_t)g->n + 1) * sizeof(uint32_t));
    uint32_t **buf = calloc(count ? count : 1, sizeof(uint32_t *));
    frames_job job = {g, label, seed, spf, first, count, buf, lens, 0, sc, tmp};
    pthread_t *tids = calloc((size_t)threads, sizeof(pthread_t));
    frames_worker_arg *args = calloc((size_t)threads, sizeof(frames_worker_arg));
    for (int t = 0; t < threads; ++t) {
        args[t].job = &job;
        args[t].id = t;
        pthread_create(&tids[t], NULL, frames_worker, &args[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tids[t], NULL);
    uint64_t total = 0;
    for (uint64_t i = 0; i < count; ++i) {
        for (uint64_t k = 0; k < lens[i]; ++k, ++total)
            if (total < cap) ids[total] = buf[i][k];
        free(buf[i]);
    }
    for (int t = 0; t < threads; ++t) {
        free(sc[t].stamp);
        free(sc[t].dist);
        free(sc[t].sigma);
        free(sc[t].queue);
    }
    free(sc);
    free(tmp);
    free(buf);
    free(tids);
    free(args);
    return total;
}
