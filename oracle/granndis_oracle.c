/*
 * granndis_oracle.c -- CPU restatement of the GraNNDis reference hot path.
 * TEST INFRASTRUCTURE ONLY (see granndis_oracle.h).  Citations are
 * /root/reference/proj file:line.
 */
#include "granndis_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define GAMMA 0x9e3779b97f4a7c15ULL

/* rng.hpp:11-16 */
uint64_t gro_mix64(uint64_t x) {
    x += GAMMA;
    x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
    x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
    return x ^ (x >> 31);
}

/* rng.hpp:20-24: three mix64 rounds over (seed, k1, k2) */
void gro_rng_init(gro_rng* r, uint64_t seed, uint64_t k1, uint64_t k2) {
    uint64_t s = gro_mix64(seed);
    s = gro_mix64(s ^ (k1 + GAMMA));
    s = gro_mix64(s ^ (k2 + 0xc2b2ae3d27d4eb4fULL));
    r->state = s;
}

/* rng.hpp:26-32: SplitMix64 step */
uint64_t gro_next_u64(gro_rng* r) {
    r->state += GAMMA;
    uint64_t z = r->state;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:35-37 */
double gro_next_double(gro_rng* r) { return (double)(gro_next_u64(r) >> 11) * 0x1.0p-53; }

/* rng.hpp:41-44: Lemire multiply-shift */
uint64_t gro_next_below(gro_rng* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)gro_next_u64(r) * n) >> 64);
}

/* rng.hpp:46-48 */
static double uniform(gro_rng* r, double lo, double hi) { return lo + (hi - lo) * gro_next_double(r); }

/* rng.hpp:55-61: backward Fisher-Yates */
void gro_shuffle_u32(uint32_t* items, uint64_t count, gro_rng* r) {
    for (uint64_t i = count; i > 1; --i) {
        uint64_t j = gro_next_below(r, i);
        uint32_t t = items[i - 1];
        items[i - 1] = items[j];
        items[j] = t;
    }
}

/* ------------------------------------------------------------------------- */
/* graph.cpp:86-94 geometric_skip */
static uint64_t geometric_skip(gro_rng* r, double p, double log1mp) {
    if (p >= 1.0) return 0;
    double u = gro_next_double(r);
    if (u <= 0.0) u = 0x1.0p-53;
    double skip = floor(log(u) / log1mp);
    if (skip < 0.0) skip = 0.0;
    if (skip > 1e18) skip = 1e18;
    return (uint64_t)skip;
}

/* graph.cpp:99-111 sample_range; emits via callback-free two-mode walker */
typedef struct {
    uint64_t* deg;        /* count mode: deg[u+1]++, deg[v+1]++ */
    uint64_t* cursor;     /* fill mode */
    uint32_t* cols;
} asm_state;

static void emit_pair(asm_state* s, uint32_t u, uint32_t v) {
    if (s->cols) {
        s->cols[s->cursor[u]++] = v;
        s->cols[s->cursor[v]++] = u;
    } else {
        s->deg[u + 1]++;
        s->deg[v + 1]++;
    }
}

static void sample_range(uint64_t seed, uint32_t u, uint32_t start, uint32_t limit, double p,
                         uint64_t tag, asm_state* s) {
    if (p <= 0.0 || start >= limit) return;
    gro_rng r;
    gro_rng_init(&r, seed, u, tag);
    double log1mp = (p < 1.0) ? log1p(-p) : 0.0;
    uint64_t v = start;
    v += geometric_skip(&r, p, log1mp);
    while (v < limit) {
        emit_pair(s, u, (uint32_t)v);
        v += 1 + geometric_skip(&r, p, log1mp);
    }
}

/* graph.cpp:137-154 gen_random_graph scan (u ascending; u<v pairs) */
static void random_scan(uint32_t n, double avg_degree, uint64_t seed, asm_state* s) {
    if (n <= 1 || avg_degree == 0.0) return;
    double p = avg_degree / (double)(n - 1);
    if (p > 1.0) p = 1.0;
    for (uint32_t u = 0; u + 1 < n; ++u) sample_range(seed, u, u + 1, n, p, 0, s);
}

/* graph.cpp:116-132 assemble_undirected, pass 1 */
uint64_t gro_gen_random_graph_count(uint32_t n, double avg_degree, uint64_t seed,
                                    uint64_t* ro) {
    memset(ro, 0, sizeof(uint64_t) * ((size_t)n + 1));
    asm_state s = {ro, NULL, NULL};
    random_scan(n, avg_degree, seed, &s);
    for (uint32_t i = 0; i < n; ++i) ro[i + 1] += ro[i];
    return ro[n];
}

/* pass 2: slices come out sorted (lower endpoints ascending, then own highers) */
void gro_gen_random_graph_fill(uint32_t n, double avg_degree, uint64_t seed, const uint64_t* ro,
                               uint32_t* cols) {
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    memcpy(cursor, ro, sizeof(uint64_t) * ((size_t)n + 1));
    asm_state s = {NULL, cursor, cols};
    random_scan(n, avg_degree, seed, &s);
    free(cursor);
}

/* graph.cpp:156-185 planted partition */
static uint32_t planted_block_of(uint32_t v, uint32_t n, uint32_t parts) {
    return (uint32_t)((((uint64_t)v + 1) * parts - 1) / n);
}
static uint32_t block_end(uint32_t b, uint32_t n, uint32_t parts) {
    return (uint32_t)(((uint64_t)b + 1) * n / parts);
}
static void planted_scan(uint32_t n, uint32_t parts, double p_in, double p_out, uint64_t seed,
                         asm_state* s) {
    for (uint32_t u = 0; u + 1 < n; ++u) {
        uint32_t be = block_end(planted_block_of(u, n, parts), n, parts);
        sample_range(seed, u, u + 1, be, p_in, 1, s);
        sample_range(seed, u, be, n, p_out, 2, s);
    }
}
uint64_t gro_gen_planted_count(uint32_t n, uint32_t parts, double p_in, double p_out,
                               uint64_t seed, uint64_t* ro) {
    memset(ro, 0, sizeof(uint64_t) * ((size_t)n + 1));
    asm_state s = {ro, NULL, NULL};
    planted_scan(n, parts, p_in, p_out, seed, &s);
    for (uint32_t i = 0; i < n; ++i) ro[i + 1] += ro[i];
    return ro[n];
}
void gro_gen_planted_fill(uint32_t n, uint32_t parts, double p_in, double p_out, uint64_t seed,
                          const uint64_t* ro, uint32_t* cols) {
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    memcpy(cursor, ro, sizeof(uint64_t) * ((size_t)n + 1));
    asm_state s = {NULL, cursor, cols};
    planted_scan(n, parts, p_in, p_out, seed, &s);
    free(cursor);
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return (x > y) - (x < y);
}

/* graph.cpp:25-67 Graph::from_edges (undirected): drop self loops, sort+dedup slices */
uint64_t gro_from_edges(const uint32_t* edges, uint64_t m, uint32_t n, uint64_t* ro,
                        uint32_t* cols) {
    uint64_t* off = (uint64_t*)calloc((size_t)n + 1, sizeof(uint64_t));
    for (uint64_t e = 0; e < m; ++e) {
        uint32_t u = edges[2 * e], v = edges[2 * e + 1];
        if (u == v) continue;
        off[u + 1]++;
        off[v + 1]++;
    }
    for (uint32_t i = 0; i < n; ++i) off[i + 1] += off[i];
    uint64_t* cursor = (uint64_t*)malloc(sizeof(uint64_t) * ((size_t)n + 1));
    memcpy(cursor, off, sizeof(uint64_t) * ((size_t)n + 1));
    for (uint64_t e = 0; e < m; ++e) {
        uint32_t u = edges[2 * e], v = edges[2 * e + 1];
        if (u == v) continue;
        cols[cursor[u]++] = v;
        cols[cursor[v]++] = u;
    }
    uint64_t write = 0;
    ro[0] = 0;
    for (uint32_t v = 0; v < n; ++v) {
        uint64_t b = off[v], e = off[v + 1];
        qsort(cols + b, (size_t)(e - b), sizeof(uint32_t), cmp_u32);
        for (uint64_t i = b; i < e; ++i) {
            if (i > b && cols[i] == cols[i - 1]) continue;
            cols[write++] = cols[i];
        }
        ro[v + 1] = write;
    }
    free(off);
    free(cursor);
    return write;
}

/* partition.cpp:51-61 */
void gro_partition_random(uint32_t n, uint32_t parts, uint64_t seed, uint32_t* assignment) {
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)n);
    for (uint32_t i = 0; i < n; ++i) perm[i] = i;
    gro_rng r;
    gro_rng_init(&r, seed, 0x7061727469ULL, 0);
    gro_shuffle_u32(perm, n, &r);
    for (uint32_t i = 0; i < n; ++i) assignment[perm[i]] = i % parts;
    free(perm);
}

/* ------------------------------------------------------------------------- */
/* reference_gnn.cpp:11-16 */
void gro_make_features(uint32_t n, uint32_t dim, uint64_t seed, double* out) {
    gro_rng r;
    gro_rng_init(&r, seed, 0x66656174ULL, 0);
    uint64_t total = (uint64_t)n * dim;
    for (uint64_t i = 0; i < total; ++i) out[i] = uniform(&r, -0.5, 0.5);
}

/* Rows ids[0..count) of make_features' matrix (reference_gnn.cpp:11-16) without
 * generating the others: row v's values are draws v*dim .. v*dim+dim-1 of the one
 * stream, and SplitMix64 draw i is reached by adding (i+1)*gamma to the keyed state
 * (the stream is a counter).  For feature matrices too large for host memory
 * (papers shape: 111 M x 128). */
void gro_feature_rows(const uint32_t* ids, uint64_t count, uint32_t dim, uint64_t seed,
                      double* out, int nthreads) {
    gro_rng r0;
    gro_rng_init(&r0, seed, 0x66656174ULL, 0);
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (uint64_t i = 0; i < count; ++i) {
        gro_rng r;
        r.state = r0.state + (uint64_t)ids[i] * dim * GAMMA;
        for (uint32_t c = 0; c < dim; ++c) out[i * dim + c] = uniform(&r, -0.5, 0.5);
    }
}

/* reference_gnn.cpp:18-32: layer 0 is hidden x feature_dim, the rest hidden x hidden */
void gro_make_layer_weights(uint32_t layers, uint32_t F, uint32_t H, uint64_t seed,
                            double* out) {
    gro_rng r;
    gro_rng_init(&r, seed, 0x77656967ULL, 0);
    uint64_t total = 0;
    for (uint32_t l = 0; l < layers; ++l) total += (uint64_t)H * (l == 0 ? F : H);
    for (uint64_t i = 0; i < total; ++i) out[i] = uniform(&r, -0.5, 0.5);
}

/* reference_gnn.cpp:53-60 apply_layer: out = relu(W agg) */
static void apply_layer(const double* w, uint32_t rows, uint32_t cols, const double* agg,
                        double* out) {
    for (uint32_t r = 0; r < rows; ++r) {
        double acc = 0.0;
        const double* wr = w + (size_t)r * cols;
        for (uint32_t c = 0; c < cols; ++c) acc += wr[c] * agg[c];
        out[r] = acc > 0.0 ? acc : 0.0;
    }
}

/* reference_gnn.cpp:64-89 forward_full: self first, then neighbors ascending */
void gro_forward_full(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                      uint32_t F, const double* w, uint32_t H, uint32_t layers, double* out,
                      int nthreads) {
    if (layers == 0) {
        memcpy(out, x, sizeof(double) * (size_t)n * F);
        return;
    }
    uint32_t maxw = F > H ? F : H;
    double* prev = (double*)malloc(sizeof(double) * (size_t)n * maxw);
    double* next = (double*)malloc(sizeof(double) * (size_t)n * maxw);
    memcpy(prev, x, sizeof(double) * (size_t)n * F);
    uint32_t width = F;
    const double* wl = w;
    for (uint32_t l = 0; l < layers; ++l) {
#pragma omp parallel num_threads(nthreads > 0 ? nthreads : 1)
        {
            double* agg = (double*)malloc(sizeof(double) * width);
#pragma omp for schedule(static)
            for (int64_t vv = 0; vv < (int64_t)n; ++vv) {
                uint32_t v = (uint32_t)vv;
                memcpy(agg, prev + (size_t)v * width, sizeof(double) * width);
                for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
                    const double* nb = prev + (size_t)ci[e] * width;
                    for (uint32_t c = 0; c < width; ++c) agg[c] += nb[c];
                }
                apply_layer(wl, H, width, agg, next + (size_t)v * H);
            }
            free(agg);
        }
        wl += (size_t)H * width;
        width = H;
        double* t = prev;
        prev = next;
        next = t;
    }
    memcpy(out, prev, sizeof(double) * (size_t)n * H);
    free(prev);
    free(next);
}

/* reference_gnn.cpp:91-147 forward_server_local with hop masking */
void gro_forward_server_local(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                              const double* x, uint32_t F, const double* w, uint32_t H,
                              uint32_t layers, const uint32_t* hop, double* out) {
    int64_t* local_of = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
    uint32_t local_n = 0;
    for (uint32_t v = 0; v < n; ++v) local_of[v] = (hop[v] == GRO_UNSEEN) ? -1 : (int64_t)local_n++;
    uint32_t* all = (uint32_t*)malloc(sizeof(uint32_t) * (local_n ? local_n : 1));
    uint32_t* lhop = (uint32_t*)malloc(sizeof(uint32_t) * (local_n ? local_n : 1));
    for (uint32_t v = 0; v < n; ++v)
        if (local_of[v] >= 0) {
            all[local_of[v]] = v;
            lhop[local_of[v]] = hop[v];
        }
    uint32_t maxw = F > H ? F : H;
    double* prev = (double*)calloc((size_t)local_n * maxw + 1, sizeof(double));
    double* next = (double*)calloc((size_t)local_n * maxw + 1, sizeof(double));
    for (uint32_t i = 0; i < local_n; ++i)
        memcpy(prev + (size_t)i * F, x + (size_t)all[i] * F, sizeof(double) * F);
    double* agg = (double*)malloc(sizeof(double) * maxw);
    uint32_t width = F;
    const double* wl = w;
    for (uint32_t l = 1; l <= layers; ++l) {
        uint32_t need = layers - l;
        memset(next, 0, sizeof(double) * (size_t)local_n * H);
        for (uint32_t i = 0; i < local_n; ++i) {
            if (lhop[i] > need) continue;
            memcpy(agg, prev + (size_t)i * width, sizeof(double) * width);
            uint32_t g = all[i];
            for (uint64_t e = ro[g]; e < ro[g + 1]; ++e) {
                int64_t j = local_of[ci[e]];
                if (j < 0 || lhop[j] > need + 1) continue;
                const double* nb = prev + (size_t)j * width;
                for (uint32_t c = 0; c < width; ++c) agg[c] += nb[c];
            }
            apply_layer(wl, H, width, agg, next + (size_t)i * H);
        }
        wl += (size_t)H * width;
        width = H;
        double* t = prev;
        prev = next;
        next = t;
    }
    uint32_t r = 0;
    for (uint32_t i = 0; i < local_n; ++i)
        if (lhop[i] == 0) {
            memcpy(out + (size_t)r * width, prev + (size_t)i * width, sizeof(double) * width);
            ++r;
        }
    free(local_of);
    free(all);
    free(lhop);
    free(prev);
    free(next);
    free(agg);
}

/* ------------------------------------------------------------------------- */
/* extract.cpp:49-58 count_induced_edges over inner + halo */
static uint64_t induced_edges(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                              const uint32_t* hop) {
    uint64_t count = 0;
    for (uint32_t v = 0; v < n; ++v) {
        if (hop[v] == GRO_UNSEEN) continue;
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e)
            if (hop[ci[e]] != GRO_UNSEEN) ++count;
    }
    return count;
}

/* extract.cpp:87-113 multi-source BFS from the inner set (ascending), depth <= layers */
uint64_t gro_extract_full(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                          const uint32_t* assignment, uint32_t server, uint32_t layers,
                          uint32_t* hop) {
    uint32_t* queue = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint64_t head = 0, tail = 0;
    for (uint32_t v = 0; v < n; ++v) {
        hop[v] = GRO_UNSEEN;
        if (assignment[v] == server) {
            hop[v] = 0;
            queue[tail++] = v;
        }
    }
    while (head < tail) {
        uint32_t v = queue[head++];
        if (hop[v] == layers) continue;
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
            uint32_t u = ci[e];
            if (hop[u] != GRO_UNSEEN) continue;
            hop[u] = hop[v] + 1;
            queue[tail++] = u;
        }
    }
    free(queue);
    return induced_edges(n, ro, ci, hop);
}

/* extract.cpp:120-131 sampled_prefix: first k of the (seed, v, "samp") shuffle of
 * the candidate list; candidates are written to buf, returns the exposed count */
static uint64_t sampled_prefix(const uint64_t* ro, const uint32_t* ci, const uint8_t* excluded,
                               const uint8_t* allowed, uint32_t v, uint32_t fanout,
                               uint64_t seed, uint32_t* buf) {
    uint64_t c = 0;
    for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
        uint32_t u = ci[e];
        if (excluded[u]) continue;
        if (allowed && !allowed[u]) continue;
        buf[c++] = u;
    }
    if (fanout == GRO_UNLIMITED_FANOUT || c <= fanout) return c;
    gro_rng r;
    gro_rng_init(&r, seed, v, 0x73616d70ULL);
    gro_shuffle_u32(buf, c, &r);
    return fanout;
}

/* Shared hop loop of extract.cpp:158-178 and batch_plan.cpp:49-66.
 * excluded = inner/target mask, allowed = universe (nullable), mark[] holds the
 * hop label (0 for excluded, GRO_UNSEEN otherwise) and is updated in place. */
static void sampled_growth(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                           const uint8_t* excluded, const uint8_t* allowed, uint32_t max_hop,
                           uint32_t fanout, uint64_t seed, uint32_t* mark) {
    uint32_t maxdeg = 0;
    for (uint32_t v = 0; v < n; ++v)
        if (ro[v + 1] - ro[v] > maxdeg) maxdeg = (uint32_t)(ro[v + 1] - ro[v]);
    uint32_t* buf = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)maxdeg + 1));
    uint32_t* frontier = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint32_t* added = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint64_t nf = 0;
    /* hop-1 frontier: excluded vertices (ascending) with >= 1 candidate neighbor */
    for (uint32_t v = 0; v < n; ++v) {
        if (!excluded[v]) continue;
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
            uint32_t u = ci[e];
            if (!excluded[u] && (!allowed || allowed[u])) {
                frontier[nf++] = v;
                break;
            }
        }
    }
    for (uint32_t h = 1; h <= max_hop && nf > 0; ++h) {
        uint64_t na = 0;
        for (uint64_t i = 0; i < nf; ++i) {
            uint32_t v = frontier[i];
            uint64_t k = sampled_prefix(ro, ci, excluded, allowed, v, fanout, seed, buf);
            for (uint64_t t = 0; t < k; ++t) {
                uint32_t u = buf[t];
                if (mark[u] != GRO_UNSEEN) continue;
                mark[u] = h;
                added[na++] = u;
            }
        }
        qsort(added, (size_t)na, sizeof(uint32_t), cmp_u32);
        uint32_t* t = frontier;
        frontier = added;
        added = t;
        nf = na;
    }
    free(buf);
    free(frontier);
    free(added);
}

/* extract.cpp:135-182 extract_sampled */
uint64_t gro_extract_sampled(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                             const uint32_t* assignment, uint32_t server, uint32_t max_hop,
                             uint32_t fanout, uint64_t seed, uint32_t* hop) {
    uint8_t* inner = (uint8_t*)malloc((size_t)n + 1);
    for (uint32_t v = 0; v < n; ++v) {
        inner[v] = assignment[v] == server;
        hop[v] = inner[v] ? 0 : GRO_UNSEEN;
    }
    sampled_growth(n, ro, ci, inner, NULL, max_hop, fanout, seed, hop);
    free(inner);
    return induced_edges(n, ro, ci, hop);
}

/* batch_plan.cpp:28-70 batch_closure */
uint64_t gro_batch_closure(uint32_t n, const uint64_t* ro, const uint32_t* ci,
                           const uint8_t* universe, const uint32_t* targets, uint64_t nt,
                           uint32_t max_hop, uint32_t fanout, uint64_t seed,
                           uint8_t* in_closure) {
    uint8_t* in_targets = (uint8_t*)calloc((size_t)n + 1, 1);
    uint32_t* mark = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    for (uint64_t i = 0; i < nt; ++i) in_targets[targets[i]] = 1;
    for (uint32_t v = 0; v < n; ++v) mark[v] = in_targets[v] ? 0 : GRO_UNSEEN;
    sampled_growth(n, ro, ci, in_targets, universe, max_hop, fanout, seed, mark);
    uint64_t size = 0;
    for (uint32_t v = 0; v < n; ++v) {
        in_closure[v] = mark[v] != GRO_UNSEEN;
        size += in_closure[v];
    }
    free(in_targets);
    free(mark);
    return size;
}

/* batch_plan.cpp:75-101 peel_mfg */
void gro_peel_mfg(uint32_t n, const uint64_t* ro, const uint32_t* ci, const uint8_t* in_batch,
                  const uint32_t* targets, uint64_t nt, uint32_t layers, uint64_t* counts) {
    uint8_t* in_set = (uint8_t*)calloc((size_t)n + 1, 1);
    uint32_t* frontier = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint32_t* added = (uint32_t*)malloc(sizeof(uint32_t) * ((size_t)n + 1));
    uint64_t nf = nt, total = nt;
    for (uint64_t i = 0; i < nt; ++i) {
        in_set[targets[i]] = 1;
        frontier[i] = targets[i];
    }
    counts[layers] = nt;
    for (uint32_t back = 1; back <= layers; ++back) {
        uint64_t na = 0;
        for (uint64_t i = 0; i < nf; ++i) {
            uint32_t v = frontier[i];
            for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
                uint32_t u = ci[e];
                if (!in_batch[u] || in_set[u]) continue;
                in_set[u] = 1;
                added[na++] = u;
            }
        }
        total += na;
        counts[layers - back] = total;
        uint32_t* t = frontier;
        frontier = added;
        added = t;
        nf = na;
    }
    free(in_set);
    free(frontier);
    free(added);
}

/* sim.cpp:81-102 split_batch: inner -> home GPU, halo ascending -> least loaded */
void gro_split_batch(const uint32_t* bv, uint64_t nb, const uint32_t* sp, const uint32_t* gp,
                     uint32_t server, uint32_t gpus, uint32_t* share_of) {
    uint64_t* size = (uint64_t*)calloc(gpus, sizeof(uint64_t));
    for (uint64_t i = 0; i < nb; ++i)
        if (sp[bv[i]] == server) {
            share_of[i] = gp[bv[i]] - server * gpus;
            size[share_of[i]]++;
        }
    for (uint64_t i = 0; i < nb; ++i) {
        if (sp[bv[i]] == server) continue;
        uint32_t best = 0;
        for (uint32_t w = 1; w < gpus; ++w)
            if (size[w] < size[best]) best = w;
        share_of[i] = best;
        size[best]++;
    }
    free(size);
}

/* ========================================================================= */
/* Training extension (UNPINNED).  Model per layer l (0-based), H^0 = X:      */
/*   SUM : P = W (H_v + sum_u H_u)                     (reference_gnn.cpp:64-89) */
/*   GCN : P = W s_v (s_v H_v + sum_u s_u H_u), s = (deg+1)^-1/2               */
/*   SAGE: P = Ws H_v + Wn (1/deg) sum_u H_u   (0 when deg = 0)                */
/*   H^{l+1} = relu(P) for l < L-1 (and for the last layer iff relu_last).     */
/* ========================================================================= */

uint64_t gro_weight_count(const gro_model* m) {
    uint64_t t = 0;
    for (uint32_t l = 0; l < m->layers; ++l)
        t += (uint64_t)m->dims[l + 1] * m->dims[l] * (m->kind == GRO_SAGE ? 2 : 1);
    return t;
}

static int nthr(int t) { return t > 0 ? t : 1; }

/* agg[v] for v < rows: SUM: H_v + sum; GCN: s_v(s_v H_v + sum s_u H_u); SAGE: mean */
static void aggregate(int kind, uint32_t rows, const uint64_t* ro, const uint32_t* ci,
                      const double* h, uint32_t w, const double* s, double* agg, int nt) {
#pragma omp parallel for schedule(static) num_threads(nthr(nt))
    for (int64_t vv = 0; vv < (int64_t)rows; ++vv) {
        uint32_t v = (uint32_t)vv;
        double* a = agg + (size_t)v * w;
        const double* hv = h + (size_t)v * w;
        if (kind == GRO_SUM) {
            for (uint32_t c = 0; c < w; ++c) a[c] = hv[c];
        } else if (kind == GRO_GCN) {
            for (uint32_t c = 0; c < w; ++c) a[c] = s[v] * hv[c];
        } else {
            for (uint32_t c = 0; c < w; ++c) a[c] = 0.0;
        }
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
            const double* hu = h + (size_t)ci[e] * w;
            if (kind == GRO_GCN) {
                double su = s[ci[e]];
                for (uint32_t c = 0; c < w; ++c) a[c] += su * hu[c];
            } else {
                for (uint32_t c = 0; c < w; ++c) a[c] += hu[c];
            }
        }
        uint64_t deg = ro[v + 1] - ro[v];
        if (kind == GRO_GCN) {
            for (uint32_t c = 0; c < w; ++c) a[c] *= s[v];
        } else if (kind == GRO_SAGE) {
            double inv = deg ? 1.0 / (double)deg : 0.0;
            for (uint32_t c = 0; c < w; ++c) a[c] *= inv;
        }
    }
}

/* Transposed aggregation (all three operators are symmetric up to the SAGE mean):
 * SUM/GCN: out = Agg^T g = Agg g; SAGE: out_v = sum_{u in N(v)} g_u / deg_u */
static void aggregate_t(int kind, uint32_t rows, const uint64_t* ro, const uint32_t* ci,
                        const double* g, uint32_t w, const double* s, double* out, int nt) {
    if (kind != GRO_SAGE) {
        aggregate(kind, rows, ro, ci, g, w, s, out, nt);
        return;
    }
#pragma omp parallel for schedule(static) num_threads(nthr(nt))
    for (int64_t vv = 0; vv < (int64_t)rows; ++vv) {
        uint32_t v = (uint32_t)vv;
        double* o = out + (size_t)v * w;
        for (uint32_t c = 0; c < w; ++c) o[c] = 0.0;
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) {
            uint32_t u = ci[e];
            double inv = 1.0 / (double)(ro[u + 1] - ro[u]);
            const double* gu = g + (size_t)u * w;
            for (uint32_t c = 0; c < w; ++c) o[c] += gu[c] * inv;
        }
    }
}

/* out[v] (+)= W a_v for v < rows; W is (o x i) row-major */
static void rows_times_wt(uint32_t rows, const double* a, uint32_t i, const double* W,
                          uint32_t o, double* out, int accumulate, int nt) {
#pragma omp parallel for schedule(static) num_threads(nthr(nt))
    for (int64_t vv = 0; vv < (int64_t)rows; ++vv) {
        const double* av = a + (size_t)vv * i;
        double* ov = out + (size_t)vv * o;
        for (uint32_t r = 0; r < o; ++r) {
            const double* wr = W + (size_t)r * i;
            double acc = 0.0;
            for (uint32_t c = 0; c < i; ++c) acc += wr[c] * av[c];
            ov[r] = accumulate ? ov[r] + acc : acc;
        }
    }
}

/* out[v] (+)= g_v W for v < rows; W is (o x i), g is rows x o, out rows x i */
static void rows_times_w(uint32_t rows, const double* g, uint32_t o, const double* W, uint32_t i,
                         double* out, int accumulate, int nt) {
#pragma omp parallel for schedule(static) num_threads(nthr(nt))
    for (int64_t vv = 0; vv < (int64_t)rows; ++vv) {
        const double* gv = g + (size_t)vv * o;
        double* ov = out + (size_t)vv * i;
        if (!accumulate)
            for (uint32_t c = 0; c < i; ++c) ov[c] = 0.0;
        for (uint32_t r = 0; r < o; ++r) {
            const double* wr = W + (size_t)r * i;
            double gr = gv[r];
            for (uint32_t c = 0; c < i; ++c) ov[c] += gr * wr[c];
        }
    }
}

/* dW (o x i) = sum_v g_v^T a_v over v < rows (per-thread partials, fixed order) */
static void outer_sum(uint32_t rows, const double* g, uint32_t o, const double* a, uint32_t i,
                      double* dW, int nt) {
    int T = nthr(nt);
    double* part = (double*)calloc((size_t)T * o * i, sizeof(double));
#pragma omp parallel num_threads(T)
    {
        int t = 0;
#ifdef _OPENMP
        t = omp_get_thread_num();
#endif
        double* p = part + (size_t)t * o * i;
#pragma omp for schedule(static)
        for (int64_t vv = 0; vv < (int64_t)rows; ++vv) {
            const double* gv = g + (size_t)vv * o;
            const double* av = a + (size_t)vv * i;
            for (uint32_t r = 0; r < o; ++r) {
                double gr = gv[r];
                if (gr == 0.0) continue;
                double* pr = p + (size_t)r * i;
                for (uint32_t c = 0; c < i; ++c) pr[c] += gr * av[c];
            }
        }
    }
    memset(dW, 0, sizeof(double) * (size_t)o * i);
    for (int t = 0; t < T; ++t)
        for (size_t k = 0; k < (size_t)o * i; ++k) dW[k] += part[(size_t)t * o * i + k];
    free(part);
}

static double* gcn_scale(uint32_t n, const uint64_t* ro) {
    double* s = (double*)malloc(sizeof(double) * ((size_t)n + 1));
    for (uint32_t v = 0; v < n; ++v) s[v] = 1.0 / sqrt((double)(ro[v + 1] - ro[v]) + 1.0);
    return s;
}

/* forward over rows < rows; keeps H^l (acts[l]) and the aggregated inputs */
typedef struct {
    double** H;   /* H[0] = x (borrowed), H[l] n x dims[l] */
    double** A;   /* aggregated input per layer (n x dims[l]) */
    double* s;
} fwd_state;

static void forward_impl(uint32_t n, uint32_t rows, const uint64_t* ro, const uint32_t* ci,
                         const double* x, const gro_model* m, const double* w, fwd_state* st,
                         int nt, const uint32_t* layer_rows) {
    uint32_t L = m->layers;
    st->H = (double**)calloc(L + 1, sizeof(double*));
    st->A = (double**)calloc(L, sizeof(double*));
    st->s = m->kind == GRO_GCN ? gcn_scale(n, ro) : NULL;
    st->H[0] = (double*)x;
    const double* wl = w;
    for (uint32_t l = 0; l < L; ++l) {
        uint32_t di = m->dims[l], dout = m->dims[l + 1];
        st->A[l] = (double*)calloc((size_t)n * di, sizeof(double));
        st->H[l + 1] = (double*)calloc((size_t)n * dout, sizeof(double));
        /* hop masking (reference_gnn.cpp:119-137): layer l produces rows < layer_rows[l];
         * rows never produced stay zero and contribute nothing when gathered */
        if (layer_rows) rows = layer_rows[l];
        aggregate(m->kind, rows, ro, ci, st->H[l], di, st->s, st->A[l], nt);
        if (m->kind == GRO_SAGE) {
            rows_times_wt(rows, st->H[l], di, wl, dout, st->H[l + 1], 0, nt);
            rows_times_wt(rows, st->A[l], di, wl + (size_t)dout * di, dout, st->H[l + 1], 1, nt);
            wl += 2 * (size_t)dout * di;
        } else {
            rows_times_wt(rows, st->A[l], di, wl, dout, st->H[l + 1], 0, nt);
            wl += (size_t)dout * di;
        }
        int relu = (l + 1 < L) || m->relu_last;
        if (relu) {
            double* h = st->H[l + 1];
            for (size_t k = 0; k < (size_t)rows * dout; ++k) h[k] = h[k] > 0.0 ? h[k] : 0.0;
        }
    }
}

static void free_state(const gro_model* m, fwd_state* st) {
    for (uint32_t l = 0; l < m->layers; ++l) {
        free(st->A[l]);
        free(st->H[l + 1]);
    }
    free(st->A);
    free(st->H);
    free(st->s);
}

void gro_model_forward(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                       const gro_model* m, const double* w, double* acts, int nthreads) {
    fwd_state st;
    forward_impl(n, n, ro, ci, x, m, w, &st, nthreads, NULL);
    size_t off = 0;
    for (uint32_t l = 1; l <= m->layers; ++l) {
        size_t sz = (size_t)n * m->dims[l];
        if (acts) memcpy(acts + off, st.H[l], sizeof(double) * sz);
        off += sz;
    }
    free_state(m, &st);
}

static double train_impl(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                         const int32_t* labels, uint32_t C, const gro_model* m, double* w,
                         double lr, double* grads, double* acts, double* dacts, uint32_t row_limit,
                         uint32_t loss_rows, double loss_count, int nthreads,
                         const uint32_t* layer_rows) {
    uint32_t L = m->layers;
    uint32_t rows = row_limit < n ? row_limit : n;
    if (loss_rows > rows) loss_rows = rows;
    fwd_state st;
    forward_impl(n, rows, ro, ci, x, m, w, &st, nthreads, layer_rows);

    /* softmax cross-entropy over rows < loss_rows, normalised by loss_count */
    double* dH = (double*)calloc((size_t)n * C, sizeof(double));
    double loss = 0.0;
    const double* logits = st.H[L];
    for (uint32_t v = 0; v < loss_rows; ++v) {
        const double* z = logits + (size_t)v * C;
        double mx = z[0];
        for (uint32_t c = 1; c < C; ++c) mx = z[c] > mx ? z[c] : mx;
        double sum = 0.0;
        for (uint32_t c = 0; c < C; ++c) sum += exp(z[c] - mx);
        double lse = mx + log(sum);
        loss += lse - z[labels[v]];
        for (uint32_t c = 0; c < C; ++c)
            dH[(size_t)v * C + c] = (exp(z[c] - lse) - (c == (uint32_t)labels[v] ? 1.0 : 0.0)) / loss_count;
    }
    loss /= loss_count;

    uint64_t wc = gro_weight_count(m);
    double* dW = (double*)calloc(wc, sizeof(double));
    /* weight block offsets */
    uint64_t* woff = (uint64_t*)calloc(L + 1, sizeof(uint64_t));
    for (uint32_t l = 0; l < L; ++l)
        woff[l + 1] = woff[l] + (uint64_t)m->dims[l + 1] * m->dims[l] * (m->kind == GRO_SAGE ? 2 : 1);

    size_t dacts_off_total = 0;
    for (uint32_t l = 1; l <= L; ++l) dacts_off_total += (size_t)n * m->dims[l];

    for (int64_t l = (int64_t)L - 1; l >= 0; --l) {
        uint32_t di = m->dims[l], dout = m->dims[l + 1];
        if (dacts) {
            size_t off = 0;
            for (uint32_t k = 1; k <= (uint32_t)l; ++k) off += (size_t)n * m->dims[k];
            memcpy(dacts + off, dH, sizeof(double) * (size_t)n * dout);
        }
        /* dP = dH * relu'(P) */
        int relu = (l + 1 < (int64_t)L) || m->relu_last;
        if (relu) {
            const double* h = st.H[l + 1];
            for (size_t k = 0; k < (size_t)rows * dout; ++k)
                if (!(h[k] > 0.0)) dH[k] = 0.0;
        }
        double* dP = dH;
        const double* wl = w + woff[l];
        double* dwl = dW + woff[l];
        double* dX = (l > 0) ? (double*)calloc((size_t)n * di, sizeof(double)) : NULL;
        if (m->kind == GRO_SAGE) {
            outer_sum(rows, dP, dout, st.H[l], di, dwl, nthreads);
            outer_sum(rows, dP, dout, st.A[l], di, dwl + (size_t)dout * di, nthreads);
            if (dX) {
                double* g = (double*)calloc((size_t)n * di, sizeof(double));
                rows_times_w(rows, dP, dout, wl + (size_t)dout * di, di, g, 0, nthreads);
                aggregate_t(GRO_SAGE, rows, ro, ci, g, di, NULL, dX, nthreads);
                rows_times_w(rows, dP, dout, wl, di, dX, 1, nthreads);
                free(g);
            }
        } else {
            outer_sum(rows, dP, dout, st.A[l], di, dwl, nthreads);
            if (dX) {
                double* g = (double*)calloc((size_t)n * di, sizeof(double));
                rows_times_w(rows, dP, dout, wl, di, g, 0, nthreads);
                aggregate_t(m->kind, rows, ro, ci, g, di, st.s, dX, nthreads);
                free(g);
            }
        }
        free(dH);
        dH = dX;
    }
    (void)dacts_off_total;
    if (grads) memcpy(grads, dW, sizeof(double) * wc);
    if (lr != 0.0)
        for (uint64_t k = 0; k < wc; ++k) w[k] -= lr * dW[k];
    if (acts) {
        size_t off = 0;
        for (uint32_t l = 1; l <= L; ++l) {
            memcpy(acts + off, st.H[l], sizeof(double) * (size_t)n * m->dims[l]);
            off += (size_t)n * m->dims[l];
        }
    }
    free(dW);
    free(woff);
    free(dH);
    free_state(m, &st);
    return loss;
}

double gro_train_epoch(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                       const int32_t* labels, uint32_t C, const gro_model* m, double* w,
                       double lr, double* grads, double* acts, double* dacts, uint32_t row_limit,
                       int nthreads) {
    uint32_t rows = row_limit < n ? row_limit : n;
    return train_impl(n, ro, ci, x, labels, C, m, w, lr, grads, acts, dacts, row_limit, rows,
                      (double)rows, nthreads, NULL);
}

double gro_train_epoch_masked(uint32_t n, const uint64_t* ro, const uint32_t* ci, const double* x,
                              const int32_t* labels, uint32_t C, const gro_model* m, double* w,
                              double lr, double* grads, uint32_t loss_rows, double loss_count,
                              const uint32_t* layer_rows, int nthreads) {
    return train_impl(n, ro, ci, x, labels, C, m, w, lr, grads, NULL, NULL, n, loss_rows, loss_count,
                      nthreads, layer_rows);
}
