/* oracle/solar_oracle.c — TEST INFRASTRUCTURE ONLY (see solar_oracle.h).
 *
 * Plain-C restatement of the reference planner path, written from the
 * reference's documented behaviour and code (cited per function). Dense
 * arrays over the id space replace the reference's hash containers; the
 * eviction choice (max valid (next_use, id)) does not depend on container
 * internals (buffer.cpp:19-35), so results are identical.
 */
#include "solar_oracle.h"

#include <stdlib.h>
#include <string.h>

#define GAMMA UINT64_C(0x9E3779B97F4A7C15)

/* ---------------------------------------------------------------- PRNG --- */
/* prng.hpp:18-23 */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * UINT64_C(0xBF58476D1CE4E5B9);
    z = (z ^ (z >> 27)) * UINT64_C(0x94D049BB133111EB);
    return z ^ (z >> 31);
}
uint64_t or_splitmix_next(uint64_t* s) { *s += GAMMA; return mix64(*s); }
/* prng.hpp:28 (modulo-biased on purpose) */
static inline uint64_t next_below(uint64_t* s, uint64_t bound) { return or_splitmix_next(s) % bound; }
/* prng.hpp:31-33 */
static inline double next_double(uint64_t* s) {
    return (double)(or_splitmix_next(s) >> 11) * (1.0 / 9007199254740992.0);
}
/* prng.hpp:45-53 */
static void fy_u32(uint32_t* a, uint64_t n, uint64_t* s) {
    for (uint64_t i = n; i > 1; --i) {
        uint64_t j = next_below(s, i);
        uint32_t t = a[i - 1]; a[i - 1] = a[j]; a[j] = t;
    }
}

/* --------------------------------------------------------------- trace --- */
/* trace.cpp:12-16 */
uint64_t or_steps_per_epoch(uint64_t D, uint32_t N, uint64_t b, int drop_last) {
    uint64_t B = (uint64_t)N * b;
    if (B == 0) return 0;
    return drop_last ? D / B : (D + B - 1) / B;
}
/* trace.cpp:18-24 */
static int validate_trace(uint64_t D, uint32_t E, uint32_t N, uint64_t b) {
    if (N == 0 || b == 0 || E == 0) return 2;
    if (D < (uint64_t)N * b) return 2;
    return 0;
}
static uint64_t keep_len(uint64_t D, uint32_t N, uint64_t b, int drop_last) {
    return drop_last ? or_steps_per_epoch(D, N, b, 1) * (uint64_t)N * b : D;
}
/* trace.cpp:26-43 */
int or_generate_trace(uint64_t D, uint32_t E, uint32_t N, uint64_t b, uint64_t seed,
                      int drop_last, uint32_t* out) {
    int rc = validate_trace(D, E, N, b);
    if (rc) return rc;
    uint64_t keep = keep_len(D, N, b, drop_last);
    uint32_t* ids = (uint32_t*)malloc(D * sizeof(uint32_t));
    for (uint32_t e = 0; e < E; ++e) {
        uint64_t s = seed ^ (GAMMA * ((uint64_t)e + 1));
        for (uint64_t i = 0; i < D; ++i) ids[i] = (uint32_t)i;
        fy_u32(ids, D, &s);
        memcpy(out + (uint64_t)e * keep, ids, keep * sizeof(uint32_t));
    }
    free(ids);
    return 0;
}

/* --------------------------------------------------------- reuse graph --- */
/* reuse_graph.cpp:14-29: distinct ids from the front/back until `want`. */
static uint64_t distinct_window(const uint32_t* seq, uint64_t n, uint64_t want, int first,
                                uint32_t* stamp, uint32_t tag, uint32_t* out) {
    uint64_t got = 0;
    if (want == 0) return 0;
    for (uint64_t i = 0; i < n; ++i) {
        uint32_t id = first ? seq[i] : seq[n - 1 - i];
        if (stamp[id] != tag) { stamp[id] = tag; out[got++] = id; }
        if (got >= want) break;
    }
    return got;
}
/* reuse_graph.cpp:31-41: node k's concatenated slices (trace.cpp:45-57). */
static uint64_t node_sequence(const uint32_t* seq, uint64_t len, uint64_t steps, uint64_t B,
                              uint64_t b, uint32_t k, uint32_t* out) {
    uint64_t n = 0;
    for (uint64_t t = 0; t < steps; ++t) {
        uint64_t lo = t * B + (uint64_t)k * b, hi = lo + b;
        if (lo > len) lo = len;
        if (hi > len) hi = len;
        for (uint64_t i = lo; i < hi; ++i) out[n++] = seq[i];
    }
    return n;
}
/* reuse_graph.cpp:77-101 */
int or_build_reuse_graph(const uint32_t* ids, uint32_t E, uint64_t len, uint64_t D, uint32_t N,
                         uint64_t b, int drop_last, uint64_t buffer_size, int mode,
                         uint64_t* w) {
    if (buffer_size == 0) return 3;
    uint32_t W = mode == 0 ? 1 : N; /* windows per epoch */
    uint64_t steps = or_steps_per_epoch(D, N, b, drop_last), B = (uint64_t)N * b;
    uint64_t* foff = (uint64_t*)calloc((size_t)E * W + 1, sizeof(uint64_t));
    uint64_t* loff = (uint64_t*)calloc((size_t)E * W + 1, sizeof(uint64_t));
    uint32_t* fwin = (uint32_t*)malloc(((size_t)E * W * len + 1) * sizeof(uint32_t));
    uint32_t* lwin = (uint32_t*)malloc(((size_t)E * W * len + 1) * sizeof(uint32_t));
    uint32_t* stamp = (uint32_t*)calloc(D, sizeof(uint32_t));
    uint32_t* nseq = (uint32_t*)malloc((len + 1) * sizeof(uint32_t));
    uint8_t* mark = (uint8_t*)calloc(D, 1);
    uint32_t tag = 0;
    uint64_t fpos = 0, lpos = 0;
    for (uint32_t e = 0; e < E; ++e) {
        const uint32_t* seq = ids + (uint64_t)e * len;
        for (uint32_t k = 0; k < W; ++k) {
            const uint32_t* s = seq;
            uint64_t n = len, want = buffer_size * N;
            if (mode != 0) { n = node_sequence(seq, len, steps, B, b, k, nseq); s = nseq; want = buffer_size; }
            fpos += distinct_window(s, n, want, 1, stamp, ++tag, fwin + fpos);
            foff[(size_t)e * W + k + 1] = fpos;
            lpos += distinct_window(s, n, want, 0, stamp, ++tag, lwin + lpos);
            loff[(size_t)e * W + k + 1] = lpos;
        }
    }
    for (uint32_t u = 0; u < E; ++u) {
        for (uint32_t v = 0; v < E; ++v) {
            uint64_t acc = 0;
            if (u == v) { w[(size_t)u * E + v] = 0; continue; }
            for (uint32_t k = 0; k < W; ++k) {
                size_t lu = (size_t)u * W + k, fv = (size_t)v * W + k;
                for (uint64_t i = loff[lu]; i < loff[lu + 1]; ++i) mark[lwin[i]] = 1;
                for (uint64_t i = foff[fv]; i < foff[fv + 1]; ++i) acc += !mark[fwin[i]];
                for (uint64_t i = loff[lu]; i < loff[lu + 1]; ++i) mark[lwin[i]] = 0;
            }
            w[(size_t)u * E + v] = acc;
        }
    }
    free(foff); free(loff); free(fwin); free(lwin); free(stamp); free(nseq); free(mark);
    return 0;
}

/* --------------------------------------------------------- epoch order --- */
static uint64_t cost_of(const uint64_t* w, uint32_t E, const uint32_t* o) {
    uint64_t c = 0;
    for (uint32_t i = 0; i + 1 < E; ++i) c += w[(size_t)o[i] * E + o[i + 1]];
    return c;
}
/* epoch_order.cpp:32-52: lexicographic next_permutation, strict improvement. */
static int next_perm(uint32_t* a, uint32_t n) {
    if (n < 2) return 0;
    uint32_t i = n - 1;
    while (i > 0 && a[i - 1] >= a[i]) --i;
    if (i == 0) return 0;
    uint32_t j = n - 1;
    while (a[j] <= a[i - 1]) --j;
    uint32_t t = a[i - 1]; a[i - 1] = a[j]; a[j] = t;
    for (uint32_t l = i, r = n - 1; l < r; ++l, --r) { t = a[l]; a[l] = a[r]; a[r] = t; }
    return 1;
}
int or_brute_force_order(const uint64_t* w, uint32_t E, uint32_t* order, uint64_t* cost) {
    if (E == 0) return 3;
    if (E > 10) return 4;
    uint32_t perm[10];
    for (uint32_t i = 0; i < E; ++i) perm[i] = order[i] = i;
    uint64_t best = cost_of(w, E, perm);
    while (next_perm(perm, E)) {
        uint64_t c = 0;
        for (uint32_t i = 0; i + 1 < E && c < best; ++i) c += w[(size_t)perm[i] * E + perm[i + 1]];
        if (c < best) { best = c; memcpy(order, perm, E * sizeof(uint32_t)); }
    }
    *cost = best;
    return 0;
}

typedef struct { uint32_t i, j; } swp;
typedef struct {
    uint32_t *pos, *inv, *best;
    swp* vel; size_t nvel, cap;
    uint64_t cost, best_cost;
    uint32_t stale;
} particle;

static void apply_swap(particle* p, uint32_t i, uint32_t j) {
    uint32_t t = p->pos[i]; p->pos[i] = p->pos[j]; p->pos[j] = t;
    p->inv[p->pos[i]] = i;
    p->inv[p->pos[j]] = j;
}
static void push_swap(swp** v, size_t* n, size_t* cap, uint32_t i, uint32_t j) {
    if (*n == *cap) { *cap = *cap ? *cap * 2 : 64; *v = (swp*)realloc(*v, *cap * sizeof(swp)); }
    (*v)[*n].i = i; (*v)[(*n)++].j = j;
}
/* epoch_order.cpp:77-87 */
static void pull_toward(particle* p, const uint32_t* target, uint32_t E, double prob, uint64_t* rng,
                        swp** out, size_t* n, size_t* cap) {
    for (uint32_t i = 0; i < E; ++i) {
        if (next_double(rng) >= prob) continue;
        uint32_t want = target[i];
        if (p->pos[i] == want) continue;
        uint32_t j = p->inv[want];
        apply_swap(p, i, j);
        push_swap(out, n, cap, i, j);
    }
}
/* epoch_order.cpp:93-117 */
static void descend(const uint64_t* w, uint32_t E, uint32_t* order, uint64_t* cost) {
    for (;;) {
        uint64_t best = *cost;
        uint32_t bi = 0, bj = 0;
        for (uint32_t i = 0; i + 1 < E; ++i)
            for (uint32_t j = i + 1; j < E; ++j) {
                uint32_t t = order[i]; order[i] = order[j]; order[j] = t;
                uint64_t c = cost_of(w, E, order);
                t = order[i]; order[i] = order[j]; order[j] = t;
                if (c < best) { best = c; bi = i; bj = j; }
            }
        if (best == *cost) return;
        uint32_t t = order[bi]; order[bi] = order[bj]; order[bj] = t;
        *cost = best;
    }
}
/* epoch_order.cpp:121-221 */
int or_pso_order(const uint64_t* w, uint32_t E, uint32_t swarm, uint32_t iters, double p_personal,
                 double p_global, double inertia, double kick, uint32_t stagnation,
                 uint32_t restart, uint64_t seed, uint32_t* order, uint64_t* cost,
                 uint64_t* hist, uint32_t* n_iters) {
    if (E == 0 || swarm == 0) return 3;
    if (inertia < 0.0 || inertia >= 1.0) return 3;
    if (kick < 0.0 || kick > 1.0) return 3;
    uint64_t rng = seed;
    const int polish = E <= 32;
    particle* sw = (particle*)calloc(swarm, sizeof(particle));
    for (uint32_t p = 0; p < swarm; ++p) {
        particle* q = &sw[p];
        q->pos = (uint32_t*)malloc(E * sizeof(uint32_t));
        q->inv = (uint32_t*)malloc(E * sizeof(uint32_t));
        q->best = (uint32_t*)malloc(E * sizeof(uint32_t));
        for (uint32_t i = 0; i < E; ++i) q->pos[i] = i;
        if (p != 0) fy_u32(q->pos, E, &rng);
        for (uint32_t i = 0; i < E; ++i) q->inv[q->pos[i]] = i;
        q->cost = cost_of(w, E, q->pos);
        if (polish) { descend(w, E, q->pos, &q->cost); for (uint32_t i = 0; i < E; ++i) q->inv[q->pos[i]] = i; }
        memcpy(q->best, q->pos, E * sizeof(uint32_t));
        q->best_cost = q->cost;
        q->stale = 0;
    }
    uint32_t* gbest = (uint32_t*)malloc(E * sizeof(uint32_t));
    uint32_t* gsnap = (uint32_t*)malloc(E * sizeof(uint32_t));
    memcpy(gbest, sw[0].pos, E * sizeof(uint32_t));
    uint64_t gcost = sw[0].cost;
    for (uint32_t p = 0; p < swarm; ++p)
        if (sw[p].cost < gcost) { gcost = sw[p].cost; memcpy(gbest, sw[p].pos, E * sizeof(uint32_t)); }

    swp* nv = NULL; size_t nn = 0, ncap = 0;
    uint32_t stagnant = 0, done = 0;
    for (uint32_t it = 0; it < iters; ++it) {
        memcpy(gsnap, gbest, E * sizeof(uint32_t));
        int improved = 0;
        for (uint32_t p = 0; p < swarm; ++p) {
            particle* q = &sw[p];
            if (restart > 0 && q->stale >= restart) {
                fy_u32(q->pos, E, &rng);
                for (uint32_t i = 0; i < E; ++i) q->inv[q->pos[i]] = i;
                q->nvel = 0;
                q->cost = cost_of(w, E, q->pos);
                if (polish) { descend(w, E, q->pos, &q->cost); for (uint32_t i = 0; i < E; ++i) q->inv[q->pos[i]] = i; }
                memcpy(q->best, q->pos, E * sizeof(uint32_t));
                q->best_cost = q->cost;
                q->stale = 0;
                continue;
            }
            nn = 0;
            for (size_t v = 0; v < q->nvel; ++v) {
                if (next_double(&rng) >= inertia) continue;
                apply_swap(q, q->vel[v].i, q->vel[v].j);
                push_swap(&nv, &nn, &ncap, q->vel[v].i, q->vel[v].j);
            }
            pull_toward(q, q->best, E, p_personal, &rng, &nv, &nn, &ncap);
            pull_toward(q, gsnap, E, p_global, &rng, &nv, &nn, &ncap);
            if (E > 1 && next_double(&rng) < kick) {
                uint32_t i = (uint32_t)next_below(&rng, E);
                uint32_t j = (uint32_t)next_below(&rng, E - 1);
                if (j >= i) ++j;
                apply_swap(q, i, j);
                push_swap(&nv, &nn, &ncap, i, j);
            }
            if (q->cap < nn) { q->cap = nn; q->vel = (swp*)realloc(q->vel, nn * sizeof(swp)); }
            if (nn) memcpy(q->vel, nv, nn * sizeof(swp));
            q->nvel = nn;
            q->cost = cost_of(w, E, q->pos);
            if (q->cost < q->best_cost) {
                if (polish) { descend(w, E, q->pos, &q->cost); for (uint32_t i = 0; i < E; ++i) q->inv[q->pos[i]] = i; }
                memcpy(q->best, q->pos, E * sizeof(uint32_t));
                q->best_cost = q->cost;
                q->stale = 0;
            } else {
                ++q->stale;
            }
        }
        for (uint32_t p = 0; p < swarm; ++p)
            if (sw[p].best_cost < gcost) {
                gcost = sw[p].best_cost;
                memcpy(gbest, sw[p].best, E * sizeof(uint32_t));
                improved = 1;
            }
        if (hist) hist[it] = gcost;
        ++done;
        stagnant = improved ? 0 : stagnant + 1;
        if (stagnant >= stagnation) break;
    }
    memcpy(order, gbest, E * sizeof(uint32_t));
    *cost = gcost;
    *n_iters = done;
    for (uint32_t p = 0; p < swarm; ++p) { free(sw[p].pos); free(sw[p].inv); free(sw[p].best); free(sw[p].vel); }
    free(sw); free(gbest); free(gsnap); free(nv);
    return 0;
}

/* ------------------------------------------------------------- buffers --- */
/* buffer.cpp:14-59 (clairvoyant, lazy max-heap on (next_use, id)) and
 * buffer.cpp:61-93 (LRU). Dense per-id state over [0, D). */
typedef struct {
    int policy;
    uint64_t cap, size;
    uint8_t* res;
    uint64_t* key;              /* clairvoyant */
    uint64_t* hk; uint32_t* hid; size_t hn, hcap;
    uint32_t *prev, *next, head, tail; /* lru; UINT32_MAX = none */
} obuf;

static void buf_init(obuf* b, int policy, uint64_t cap, uint64_t D) {
    memset(b, 0, sizeof *b);
    b->policy = policy; b->cap = cap;
    b->res = (uint8_t*)calloc(D ? D : 1, 1);
    if (policy == 0) b->key = (uint64_t*)malloc((D ? D : 1) * sizeof(uint64_t));
    else {
        b->prev = (uint32_t*)malloc((D ? D : 1) * sizeof(uint32_t));
        b->next = (uint32_t*)malloc((D ? D : 1) * sizeof(uint32_t));
        b->head = b->tail = UINT32_MAX;
    }
}
static void buf_free(obuf* b) { free(b->res); free(b->key); free(b->hk); free(b->hid); free(b->prev); free(b->next); }
static int heap_less(const obuf* b, size_t x, size_t y) {
    return b->hk[x] < b->hk[y] || (b->hk[x] == b->hk[y] && b->hid[x] < b->hid[y]);
}
static void heap_swap(obuf* b, size_t x, size_t y) {
    uint64_t k = b->hk[x]; b->hk[x] = b->hk[y]; b->hk[y] = k;
    uint32_t i = b->hid[x]; b->hid[x] = b->hid[y]; b->hid[y] = i;
}
static void heap_push(obuf* b, uint64_t k, uint32_t id) {
    if (b->hn == b->hcap) {
        b->hcap = b->hcap ? b->hcap * 2 : 1024;
        b->hk = (uint64_t*)realloc(b->hk, b->hcap * sizeof(uint64_t));
        b->hid = (uint32_t*)realloc(b->hid, b->hcap * sizeof(uint32_t));
    }
    size_t i = b->hn++;
    b->hk[i] = k; b->hid[i] = id;
    while (i > 0) { size_t p = (i - 1) / 2; if (!heap_less(b, p, i)) break; heap_swap(b, p, i); i = p; }
}
static void heap_pop(obuf* b) {
    b->hn--;
    if (b->hn == 0) return;
    b->hk[0] = b->hk[b->hn]; b->hid[0] = b->hid[b->hn];
    size_t i = 0;
    for (;;) {
        size_t l = 2 * i + 1, r = l + 1, m = i;
        if (l < b->hn && heap_less(b, m, l)) m = l;
        if (r < b->hn && heap_less(b, m, r)) m = r;
        if (m == i) break;
        heap_swap(b, i, m); i = m;
    }
}
static int cv_evict(obuf* b) {
    while (b->hn) {
        uint64_t k = b->hk[0]; uint32_t id = b->hid[0];
        heap_pop(b);
        if (!b->res[id] || b->key[id] != k) continue; /* stale entry */
        b->res[id] = 0; b->size--;
        return 0;
    }
    return 7;
}
static void lru_unlink(obuf* b, uint32_t id) {
    uint32_t p = b->prev[id], n = b->next[id];
    if (p != UINT32_MAX) b->next[p] = n; else b->head = n;
    if (n != UINT32_MAX) b->prev[n] = p; else b->tail = p;
}
static void lru_front(obuf* b, uint32_t id) {
    b->prev[id] = UINT32_MAX; b->next[id] = b->head;
    if (b->head != UINT32_MAX) b->prev[b->head] = id; else b->tail = id;
    b->head = id;
}
static int lru_touch(obuf* b, uint32_t id) {
    if (b->res[id]) { lru_unlink(b, id); lru_front(b, id); return 0; }
    b->res[id] = 1; b->size++;
    lru_front(b, id);
    if (b->size > b->cap) {
        uint32_t v = b->tail;
        lru_unlink(b, v);
        b->res[v] = 0; b->size--;
    }
    return 0;
}
/* returns 1 hit, 0 miss, <0 error */
static int buf_access(obuf* b, uint32_t id, uint64_t nu) {
    if (b->policy != 0) { int hit = b->res[id]; lru_touch(b, id); return hit; }
    if (b->res[id]) { b->key[id] = nu; heap_push(b, nu, id); return 1; }
    b->res[id] = 1; b->size++;
    b->key[id] = nu; heap_push(b, nu, id);
    if (b->size > b->cap && cv_evict(b)) return -7;
    return 0;
}
static int buf_insert_silent(obuf* b, uint32_t id, uint64_t nu) {
    if (b->policy != 0) return lru_touch(b, id);
    if (b->res[id]) return 0;
    b->res[id] = 1; b->size++;
    b->key[id] = nu; heap_push(b, nu, id);
    if (b->size > b->cap && cv_evict(b)) return 7;
    return 0;
}

/* ------------------------------------------------------- assign/balance --- */
typedef struct { uint32_t* v; uint64_t n; } olist;

/* locality.cpp:7-42 (slice=0) and :57-73 (slice=1). res[k] = node k's
 * residency byte map. */
static int assign_core(uint8_t* const* res, const uint32_t* batch, uint64_t len, uint32_t N,
                       uint64_t b, int slice, olist* lists, uint32_t* fetch_scratch) {
    for (uint32_t k = 0; k < N; ++k) lists[k].n = 0;
    if (slice) {
        for (uint64_t p = 0; p < len; ++p) {
            uint64_t k = p / b;
            if (k >= N) return 3;
            uint32_t id = batch[p];
            lists[k].v[lists[k].n++] = id | (res[k][id] ? OR_HIT_BIT : 0u);
        }
        return 0;
    }
    if (len > (uint64_t)N * b) return 3;
    uint64_t nf = 0;
    for (uint64_t j = 0; j < len; ++j) {
        uint32_t id = batch[j], chosen = N;
        for (uint32_t k = 0; k < N; ++k) {
            if (lists[k].n >= b) continue;
            if (!res[k][id]) continue;
            if (chosen == N || lists[k].n < lists[chosen].n) chosen = k;
        }
        if (chosen == N) fetch_scratch[nf++] = id;
        else lists[chosen].v[lists[chosen].n++] = id | OR_HIT_BIT;
    }
    uint32_t k = 0;
    for (uint64_t f = 0; f < nf; ++f) {
        while (k < N && lists[k].n >= b) ++k;
        if (k == N) return 7;
        lists[k].v[lists[k].n++] = fetch_scratch[f];
    }
    return 0;
}

/* balance.cpp:10-39 */
static int balance_core(olist* lists, uint32_t N, uint64_t* moves_out) {
    uint64_t* counts = (uint64_t*)calloc(N, sizeof(uint64_t));
    for (uint32_t k = 0; k < N; ++k)
        for (uint64_t i = 0; i < lists[k].n; ++i) counts[k] += !(lists[k].v[i] & OR_HIT_BIT);
    uint64_t moves = 0;
    for (;;) {
        uint32_t d = 0, r = 0;
        for (uint32_t k = 1; k < N; ++k) {
            if (counts[k] > counts[d]) d = k;
            if (counts[k] < counts[r]) r = k;
        }
        if (counts[d] - counts[r] <= 1) break;
        olist* from = &lists[d];
        uint64_t best = from->n;
        for (uint64_t i = 0; i < from->n; ++i) {
            if (from->v[i] & OR_HIT_BIT) continue;
            if (best == from->n || from->v[i] > from->v[best]) best = i;
        }
        if (best == from->n) { free(counts); return 7; }
        lists[r].v[lists[r].n++] = from->v[best];
        memmove(from->v + best, from->v + best + 1, (from->n - best - 1) * sizeof(uint32_t));
        from->n--;
        counts[d]--; counts[r]++; moves++;
    }
    free(counts);
    if (moves_out) *moves_out = moves;
    return 0;
}

static int cmp_u32(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}

int or_remap_step(const uint64_t* holders, const uint32_t* batch, uint64_t len, uint32_t N,
                  uint64_t b, int slice, uint32_t* out_items, uint32_t* node_off) {
    if (N == 0 || N > 64 || b == 0) return 3;
    uint32_t D = 0;
    for (uint64_t j = 0; j < len; ++j) if (batch[j] + 1 > D) D = batch[j] + 1;
    uint8_t** res = (uint8_t**)malloc(N * sizeof(uint8_t*));
    olist* lists = (olist*)malloc(N * sizeof(olist));
    uint32_t* scratch = (uint32_t*)malloc((len + 1) * sizeof(uint32_t));
    for (uint32_t k = 0; k < N; ++k) {
        res[k] = (uint8_t*)calloc(D + 1, 1);
        for (uint64_t j = 0; j < len; ++j) res[k][batch[j]] = (uint8_t)((holders[j] >> k) & 1);
        lists[k].v = (uint32_t*)malloc((len + 1) * sizeof(uint32_t));
    }
    int rc = assign_core(res, batch, len, N, b, slice, lists, scratch);
    if (!rc) {
        uint32_t off = 0;
        for (uint32_t k = 0; k < N; ++k) {
            node_off[k] = off;
            memcpy(out_items + off, lists[k].v, lists[k].n * sizeof(uint32_t));
            off += (uint32_t)lists[k].n;
        }
        node_off[N] = off;
    }
    for (uint32_t k = 0; k < N; ++k) { free(res[k]); free(lists[k].v); }
    free(res); free(lists); free(scratch);
    return rc;
}

int or_balance_step(uint32_t* items, uint32_t* node_off, uint32_t N, uint64_t* moves) {
    if (N == 0) return 3;
    uint64_t total = node_off[N];
    olist* lists = (olist*)malloc(N * sizeof(olist));
    for (uint32_t k = 0; k < N; ++k) {
        lists[k].n = node_off[k + 1] - node_off[k];
        lists[k].v = (uint32_t*)malloc((total + 1) * sizeof(uint32_t));
        memcpy(lists[k].v, items + node_off[k], lists[k].n * sizeof(uint32_t));
    }
    int rc = balance_core(lists, N, moves);
    uint32_t off = 0;
    for (uint32_t k = 0; k < N; ++k) {
        node_off[k] = off;
        memcpy(items + off, lists[k].v, lists[k].n * sizeof(uint32_t));
        off += (uint32_t)lists[k].n;
        free(lists[k].v);
    }
    node_off[N] = off;
    free(lists);
    return rc;
}

/* chunking.cpp:9-45: sorted-unique fetch ids merged into reads of span <=
 * threshold; returns the redundant (streamed but unrequested) ids ascending. */
static uint64_t redundant_of(const uint32_t* fetch, uint64_t n, uint64_t thr, uint32_t* tmp,
                             uint32_t** out, uint64_t* cap) {
    memcpy(tmp, fetch, n * sizeof(uint32_t));
    qsort(tmp, n, sizeof(uint32_t), cmp_u32);
    uint64_t u = 0;
    for (uint64_t i = 0; i < n; ++i) if (u == 0 || tmp[u - 1] != tmp[i]) tmp[u++] = tmp[i];
    uint64_t nr = 0, i = 0;
    while (i < u) {
        uint64_t start = tmp[i], j = i + 1;
        while (j < u && tmp[j] - start + 1 <= thr) ++j;
        if (j - i > 1) {
            uint64_t k = i;
            for (uint64_t id = start; id <= tmp[j - 1]; ++id) {
                while (k < j && tmp[k] < id) ++k;
                if (k < j && tmp[k] == id) continue;
                if (nr == *cap) { *cap = *cap ? *cap * 2 : 256; *out = (uint32_t*)realloc(*out, *cap * sizeof(uint32_t)); }
                (*out)[nr++] = (uint32_t)id;
            }
        }
        i = j;
    }
    return nr;
}

/* ---------------------------------------------------------------- plan --- */
static uint64_t digest_mix(uint64_t id) { return mix64(id + GAMMA); }

/* pipeline.cpp:32-120 */
int or_plan(const or_config* c, uint32_t* trace, uint64_t* graph, uint32_t* order, uint64_t* cost,
            uint64_t* hist, uint32_t* n_iters, uint32_t* items, uint32_t* node_off, uint32_t* fb,
            uint32_t* fa, uint64_t* residency) {
    const uint64_t D = c->dataset_size, b = c->local_batch, C = c->buffer_capacity;
    const uint32_t E = c->num_epochs, N = c->num_nodes;
    int rc = validate_trace(D, E, N, b);
    if (rc) return rc;
    if (C == 0) return 2;
    if (c->chunk_threshold == 0) return 2;
    const uint64_t B = (uint64_t)N * b, S = or_steps_per_epoch(D, N, b, c->drop_last);
    const uint64_t keep = keep_len(D, N, b, c->drop_last);
    if ((rc = or_generate_trace(D, E, N, b, c->seed, c->drop_last, trace))) return rc;
    if ((rc = or_build_reuse_graph(trace, E, keep, D, N, b, c->drop_last, C, c->graph_mode, graph))) return rc;
    if (c->optim_order) {
        rc = or_pso_order(graph, E, c->pso_swarm, c->pso_iters, c->pso_p_personal, c->pso_p_global,
                          c->pso_inertia, c->pso_kick, c->pso_stagnation, c->pso_restart, c->seed,
                          order, cost, hist, n_iters);
        if (rc) return rc;
    } else {
        for (uint32_t i = 0; i < E; ++i) order[i] = i;
        *cost = cost_of(graph, E, order);
        *n_iters = 0;
    }
    /* occurrence table (pipeline.cpp:54-60) as CSR over ids */
    const uint64_t T = (uint64_t)E * S;
    uint64_t* ocnt = (uint64_t*)calloc(D + 1, sizeof(uint64_t));
    for (uint64_t i = 0; i < (uint64_t)E * keep; ++i) ocnt[trace[i] + 1]++;
    for (uint64_t x = 0; x < D; ++x) ocnt[x + 1] += ocnt[x];
    uint64_t* occ = (uint64_t*)malloc(((uint64_t)E * keep + 1) * sizeof(uint64_t));
    uint64_t* fill = (uint64_t*)calloc(D, sizeof(uint64_t));
    uint64_t g = 0;
    for (uint32_t i = 0; i < E; ++i)
        for (uint64_t t = 0; t < S; ++t, ++g) {
            const uint32_t* seq = trace + (uint64_t)order[i] * keep;
            uint64_t lo = t * B, hi = lo + B;
            if (hi > keep) hi = keep;
            for (uint64_t p = lo; p < hi; ++p) { uint32_t x = seq[p]; occ[ocnt[x] + fill[x]++] = g; }
        }
    uint64_t* cursor = (uint64_t*)calloc(D, sizeof(uint64_t));
    obuf* bufs = (obuf*)malloc(N * sizeof(obuf));
    uint8_t** res = (uint8_t**)malloc(N * sizeof(uint8_t*));
    olist* lists = (olist*)malloc(N * sizeof(olist));
    for (uint32_t k = 0; k < N; ++k) {
        buf_init(&bufs[k], c->policy, C, D);
        res[k] = bufs[k].res;
        lists[k].v = (uint32_t*)malloc((B + 1) * sizeof(uint32_t));
    }
    uint32_t* scratch = (uint32_t*)malloc((B + 1) * sizeof(uint32_t));
    uint32_t* fetch = (uint32_t*)malloc((B + 1) * sizeof(uint32_t));
    uint32_t* red = NULL;
    uint32_t** reds = (uint32_t**)calloc(N, sizeof(uint32_t*));
    uint64_t* nreds = (uint64_t*)calloc(N, sizeof(uint64_t));
    uint64_t* redcaps = (uint64_t*)calloc(N, sizeof(uint64_t));
    const int redundant = c->insert_redundant && c->optim_chunk;
    uint64_t base = 0;
    g = 0;
    for (uint32_t i = 0; i < E && !rc; ++i) {
        const uint32_t* seq = trace + (uint64_t)order[i] * keep;
        for (uint64_t t = 0; t < S && !rc; ++t, ++g) {
            uint64_t lo = t * B, hi = lo + B;
            if (lo > keep) lo = keep;
            if (hi > keep) hi = keep;
            const uint32_t* batch = seq + lo;
            const uint64_t len = hi - lo;
            if ((rc = assign_core(res, batch, len, N, b, !c->optim_remap, lists, scratch))) break;
            for (uint32_t k = 0; k < N; ++k) {
                uint32_t f = 0;
                for (uint64_t q = 0; q < lists[k].n; ++q) f += !(lists[k].v[q] & OR_HIT_BIT);
                fb[g * N + k] = f;
            }
            if (c->optim_balance && (rc = balance_core(lists, N, NULL))) break;
            uint32_t off = 0;
            for (uint32_t k = 0; k < N; ++k) {
                uint32_t f = 0;
                for (uint64_t q = 0; q < lists[k].n; ++q) f += !(lists[k].v[q] & OR_HIT_BIT);
                fa[g * N + k] = f;
                node_off[g * (N + 1) + k] = off;
                memcpy(items + base + off, lists[k].v, lists[k].n * sizeof(uint32_t));
                off += (uint32_t)lists[k].n;
            }
            node_off[g * (N + 1) + N] = off;
            base += off;
            if (off != len) { rc = 7; break; }
            if (redundant) {
                for (uint32_t k = 0; k < N; ++k) {
                    uint64_t nf = 0;
                    for (uint64_t q = 0; q < lists[k].n; ++q)
                        if (!(lists[k].v[q] & OR_HIT_BIT)) fetch[nf++] = lists[k].v[q];
                    nreds[k] = redundant_of(fetch, nf, c->chunk_threshold, scratch, &reds[k], &redcaps[k]);
                }
            }
            /* advance residency (pipeline.cpp:90-102) */
            for (uint32_t k = 0; k < N && !rc; ++k)
                for (uint64_t q = 0; q < lists[k].n; ++q) {
                    uint32_t x = lists[k].v[q] & ~OR_HIT_BIT;
                    uint64_t cur = cursor[x], n = ocnt[x + 1] - ocnt[x];
                    if (cur >= n || occ[ocnt[x] + cur] != g) { rc = 7; break; }
                    uint64_t nu = cur + 1 < n ? occ[ocnt[x] + cur + 1] : OR_NEVER;
                    cursor[x]++;
                    if (buf_access(&bufs[k], x, nu) < 0) { rc = 7; break; }
                }
            if (redundant && !rc) /* pipeline.cpp:103-114 */
                for (uint32_t k = 0; k < N && !rc; ++k)
                    for (uint64_t q = 0; q < nreds[k]; ++q) {
                        uint32_t x = reds[k][q];
                        uint64_t cur = cursor[x], n = ocnt[x + 1] - ocnt[x];
                        uint64_t nu = cur < n ? occ[ocnt[x] + cur] : OR_NEVER;
                        if (buf_insert_silent(&bufs[k], x, nu)) { rc = 7; break; }
                    }
            if (residency)
                for (uint32_t k = 0; k < N; ++k) {
                    uint64_t sum = 0, xr = 0;
                    for (uint64_t x = 0; x < D; ++x)
                        if (bufs[k].res[x]) { uint64_t z = digest_mix(x); sum += z; xr ^= z; }
                    residency[(g * N + k) * 3 + 0] = bufs[k].size;
                    residency[(g * N + k) * 3 + 1] = sum;
                    residency[(g * N + k) * 3 + 2] = xr;
                }
        }
    }
    (void)T;
    for (uint32_t k = 0; k < N; ++k) { buf_free(&bufs[k]); free(lists[k].v); free(reds[k]); }
    free(bufs); free(res); free(lists); free(scratch); free(fetch); free(red); free(reds);
    free(nreds); free(redcaps); free(ocnt); free(occ); free(fill); free(cursor);
    return rc;
}

/* ------------------------------------------------------------ simulate --- */
/* buffer.cpp:183-247 with insert_redundant = false; next_use_chain
 * (buffer.cpp:103-112) on each node's flattened sequence. */
int or_simulate(const uint32_t* items, const uint32_t* node_off, uint64_t T, uint32_t N,
                uint64_t D, uint64_t C, int policy, uint32_t* hits, uint32_t* misses) {
    return or_simulate_ex(items, node_off, T, N, D, C, policy, NULL, NULL, NULL, hits, misses);
}

/* buffer.cpp:183-247 with insert_redundant (:224-238) when rstart != NULL:
 * after list (g, k), redundant_ids(reads, fetch_ids) (chunking.cpp:35-45;
 * a read with start < end is a Chunk, start == end a Single) are inserted
 * silently with next = the first position of the id on node k at or after
 * the node's cursor (std::lower_bound over its positions). Reads of list
 * (g, k) sit at the list's item offsets, rcount[g*N+k] of them. */
static int cmp_u32r(const void* a, const void* b) {
    uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
    return x < y ? -1 : x > y;
}
int or_simulate_ex(const uint32_t* items, const uint32_t* node_off, uint64_t T, uint32_t N,
                   uint64_t D, uint64_t C, int policy, const uint32_t* rstart, const uint32_t* rend,
                   const uint32_t* rcount, uint32_t* hits, uint32_t* misses) {
    if (C == 0) return 3;
    uint64_t* len = (uint64_t*)calloc(N, sizeof(uint64_t));
    uint64_t base = 0;
    for (uint64_t g = 0; g < T; ++g) {
        const uint32_t* off = node_off + g * (N + 1);
        for (uint32_t k = 0; k < N; ++k) len[k] += off[k + 1] - off[k];
    }
    uint32_t** seq = (uint32_t**)malloc(N * sizeof(uint32_t*));
    uint64_t** nxt = (uint64_t**)malloc(N * sizeof(uint64_t*));
    uint64_t* fillp = (uint64_t*)calloc(N, sizeof(uint64_t));
    for (uint32_t k = 0; k < N; ++k) {
        seq[k] = (uint32_t*)malloc((len[k] + 1) * sizeof(uint32_t));
        nxt[k] = (uint64_t*)malloc((len[k] + 1) * sizeof(uint64_t));
    }
    for (uint64_t g = 0; g < T; ++g) {
        const uint32_t* off = node_off + g * (N + 1);
        for (uint32_t k = 0; k < N; ++k)
            for (uint32_t i = off[k]; i < off[k + 1]; ++i) seq[k][fillp[k]++] = items[base + i] & ~OR_HIT_BIT;
        base += off[N];
    }
    uint64_t* last = (uint64_t*)malloc((D ? D : 1) * sizeof(uint64_t));
    for (uint32_t k = 0; k < N; ++k) {
        for (uint64_t x = 0; x < D; ++x) last[x] = OR_NEVER;
        for (uint64_t i = len[k]; i > 0; --i) {
            uint32_t x = seq[k][i - 1];
            nxt[k][i - 1] = last[x];
            last[x] = i - 1;
        }
    }
    /* positions of every id on every node (CSR by id), for the silent inserts */
    uint64_t** pstart = NULL;
    uint64_t** plist = NULL;
    if (rstart) {
        pstart = (uint64_t**)malloc(N * sizeof(uint64_t*));
        plist = (uint64_t**)malloc(N * sizeof(uint64_t*));
        for (uint32_t k = 0; k < N; ++k) {
            pstart[k] = (uint64_t*)calloc(D + 1, sizeof(uint64_t));
            plist[k] = (uint64_t*)malloc((len[k] + 1) * sizeof(uint64_t));
            for (uint64_t i = 0; i < len[k]; ++i) pstart[k][seq[k][i] + 1]++;
            for (uint64_t x = 0; x < D; ++x) pstart[k][x + 1] += pstart[k][x];
            uint64_t* f2 = (uint64_t*)calloc(D + 1, sizeof(uint64_t));
            for (uint64_t i = 0; i < len[k]; ++i) { uint32_t x = seq[k][i]; plist[k][pstart[k][x] + f2[x]++] = i; }
            free(f2);
        }
    }
    uint32_t* fetch = (uint32_t*)malloc(sizeof(uint32_t));
    uint64_t fcap = 1;
    int rc = 0;
    obuf* bufs = (obuf*)malloc(N * sizeof(obuf));
    for (uint32_t k = 0; k < N; ++k) { buf_init(&bufs[k], policy, C, D); fillp[k] = 0; }
    uint64_t gbase = 0;
    for (uint64_t g = 0; g < T && !rc; ++g) {
        const uint32_t* off = node_off + g * (N + 1);
        for (uint32_t k = 0; k < N; ++k) {
            uint32_t h = 0, m = 0;
            for (uint32_t i = off[k]; i < off[k + 1]; ++i) {
                uint64_t p = fillp[k]++;
                int r = buf_access(&bufs[k], seq[k][p], nxt[k][p]);
                if (r < 0) { rc = 7; break; }
                if (r) ++h; else ++m;
            }
            hits[g * N + k] = h;
            misses[g * N + k] = m;
            if (rstart && !rc) {
                const uint64_t lo = gbase + off[k], L = off[k + 1] - off[k];
                if (L > fcap) { fcap = L; fetch = (uint32_t*)realloc(fetch, fcap * sizeof(uint32_t)); }
                uint64_t nf = 0;
                for (uint64_t i = 0; i < L; ++i)
                    if (!(items[lo + i] & OR_HIT_BIT)) fetch[nf++] = items[lo + i];
                qsort(fetch, nf, sizeof(uint32_t), cmp_u32r);
                for (uint32_t r = 0; r < rcount[g * N + k]; ++r) {
                    const uint32_t st = rstart[lo + r], en = rend[lo + r];
                    if (st >= en) continue;
                    for (uint64_t id = st; id <= en; ++id) {
                        uint32_t key = (uint32_t)id;
                        if (bsearch(&key, fetch, nf, sizeof(uint32_t), cmp_u32r)) continue;
                        /* std::lower_bound(positions, cursor) */
                        uint64_t nx = OR_NEVER;
                        const uint64_t* pl = plist[k] + pstart[k][id];
                        uint64_t a0 = 0, a1 = pstart[k][id + 1] - pstart[k][id];
                        while (a0 < a1) { uint64_t mid = (a0 + a1) / 2; if (pl[mid] < fillp[k]) a0 = mid + 1; else a1 = mid; }
                        if (a0 < pstart[k][id + 1] - pstart[k][id]) nx = pl[a0];
                        if (buf_insert_silent(&bufs[k], key, nx)) { rc = 7; break; }
                    }
                    if (rc) break;
                }
            }
        }
        gbase += off[N];
    }
    for (uint32_t k = 0; k < N; ++k) {
        buf_free(&bufs[k]); free(seq[k]); free(nxt[k]);
        if (pstart) { free(pstart[k]); free(plist[k]); }
    }
    free(pstart); free(plist); free(fetch);
    free(bufs); free(seq); free(nxt); free(len); free(fillp); free(last);
    return rc;
}

int or_simulate_sequence(const uint32_t* seq, uint64_t n, uint64_t D, uint64_t C, int policy,
                         uint64_t* misses) {
    if (C == 0) return 3;
    uint64_t* nxt = (uint64_t*)malloc((n + 1) * sizeof(uint64_t));
    uint64_t* last = (uint64_t*)malloc((D ? D : 1) * sizeof(uint64_t));
    for (uint64_t x = 0; x < D; ++x) last[x] = OR_NEVER;
    for (uint64_t i = n; i > 0; --i) { nxt[i - 1] = last[seq[i - 1]]; last[seq[i - 1]] = i - 1; }
    obuf b;
    buf_init(&b, policy, C, D);
    uint64_t m = 0;
    int rc = 0;
    for (uint64_t i = 0; i < n; ++i) {
        int r = buf_access(&b, seq[i], policy == 0 ? nxt[i] : 0);
        if (r < 0) { rc = 7; break; }
        m += !r;
    }
    *misses = m;
    buf_free(&b); free(nxt); free(last);
    return rc;
}

/* ---------------------------------------------------------------- store --- */
/* store.cpp:70-80: one continuous splitmix64 byte stream (LE words). */
void or_store_payload(uint64_t fill_seed, uint64_t offset, uint64_t n, uint8_t* out) {
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t j = offset + i;
        uint64_t word = mix64(fill_seed + (j / 8 + 1) * GAMMA);
        out[i] = (uint8_t)(word >> (8 * (j % 8)));
    }
}

/* ------------------------------------------------------------ chunking --- */
/* chunking.cpp:9-33 (plan_chunks) and pipeline.cpp:21-28 (singles_plan) on
 * each (step, node) fetch list of a finished plan. Reads of list (g, k) are
 * written at that list's item offsets; counts/needed/redundant per (g, k). */
int or_plan_reads(const uint32_t* items, const uint32_t* node_off, uint64_t T, uint32_t N,
                  int chunked, uint64_t thr, uint32_t* rstart, uint32_t* rend, uint32_t* rcount,
                  uint32_t* needed, uint32_t* redundant) {
    if (chunked && thr == 0) return 3;
    uint64_t base = 0;
    uint32_t* ids = NULL;
    uint64_t cap = 0;
    for (uint64_t g = 0; g < T; ++g) {
        const uint32_t* off = node_off + g * (N + 1);
        for (uint32_t k = 0; k < N; ++k) {
            const uint64_t lo = base + off[k], n = off[k + 1] - off[k];
            if (n > cap) { cap = n; ids = (uint32_t*)realloc(ids, cap * sizeof(uint32_t)); }
            uint64_t f = 0;
            for (uint64_t q = 0; q < n; ++q)
                if (!(items[lo + q] & OR_HIT_BIT)) ids[f++] = items[lo + q];
            qsort(ids, f, sizeof(uint32_t), cmp_u32);
            uint64_t nr = 0, red = 0, need = f;
            if (chunked) {
                uint64_t u = 0;
                for (uint64_t q = 0; q < f; ++q) if (u == 0 || ids[u - 1] != ids[q]) ids[u++] = ids[q];
                need = u;
                uint64_t i = 0;
                while (i < u) {
                    uint64_t start = ids[i], j = i + 1;
                    while (j < u && ids[j] - start + 1 <= thr) ++j;
                    rstart[lo + nr] = (uint32_t)start;
                    rend[lo + nr] = ids[j - 1];
                    if (j - i > 1) red += (ids[j - 1] - start + 1) - (j - i);
                    ++nr;
                    i = j;
                }
            } else {
                for (uint64_t q = 0; q < f; ++q) { rstart[lo + nr] = ids[q]; rend[lo + nr] = ids[q]; ++nr; }
            }
            rcount[g * N + k] = (uint32_t)nr;
            needed[g * N + k] = (uint32_t)need;
            redundant[g * N + k] = (uint32_t)red;
        }
        base += off[N];
    }
    free(ids);
    return 0;
}
