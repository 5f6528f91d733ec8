/*
 * abmx_oracle.c — TEST INFRASTRUCTURE ONLY. Plain-C restatement of the reference's
 * CPU algorithm for the predation hot path; see abmx_oracle.h for the pinning story.
 * Every function cites the reference file:line (under /root/reference/proj) it follows.
 * Build: make -C oracle (gcc, default x86-64 target: no FMA contraction, matching the
 * reference's g++ build, which is what keeps frac*E bit-identical).
 */
#include "abmx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ RNG */
/* src/rng.cpp:9-10 */
#define K_DRAW 0x9E3779B97F4A7C15ULL
#define K_SPLIT 0xC2B2AE3D27D4EB4FULL

/* splitmix64 finalizer, src/rng.cpp:12-16 */
uint64_t orc_mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
/* src/rng.cpp:18-20 */
uint64_t orc_split(uint64_t key, uint64_t i) { return orc_mix64(key + K_SPLIT * (i + 1)); }
/* src/rng.cpp:22-24 */
uint64_t orc_draw(uint64_t key, uint64_t c) { return orc_mix64(key + K_DRAW * (c + 1)); }
/* src/rng.cpp:26-28 */
double orc_uniform_double(uint64_t key, uint64_t c) {
    return (double)(orc_draw(key, c) >> 11) * 0x1.0p-53;
}
/* src/rng.cpp:30-36 (lo < hi is the caller's contract here) */
int64_t orc_uniform_int(uint64_t key, uint64_t c, int64_t lo, int64_t hi) {
    const uint64_t span = (uint64_t)(hi - lo);
    const unsigned __int128 wide = (unsigned __int128)orc_draw(key, c) * span;
    return lo + (int64_t)(uint64_t)(wide >> 64);
}
/* src/rng.cpp:38-40 */
int orc_bernoulli(uint64_t key, uint64_t c, double p) { return orc_uniform_double(key, c) < p; }
/* src/batch.cpp:12-19: master.split(BatchReplica=2).split(r) */
uint64_t orc_replica_seed(uint64_t master, int64_t r) {
    return orc_split(orc_split(master, 2), (uint64_t)r);
}

/* ------------------------------------------------------------------ kernel table */
/* src/simd/kernels_scalar.cpp:7-13 */
void orc_rank_scan(const uint8_t* mask, int32_t* ranks, size_t n) {
    int32_t run = 0;
    for (size_t i = 0; i < n; ++i) {
        run += mask[i] ? 1 : 0;
        ranks[i] = mask[i] ? run : 0;
    }
}
/* src/simd/kernels_scalar.cpp:15-20 */
int64_t orc_count_true(const uint8_t* mask, size_t n) {
    int64_t c = 0;
    for (size_t i = 0; i < n; ++i) c += mask[i] ? 1 : 0;
    return c;
}
/* src/simd/kernels_scalar.cpp:22-31 */
void orc_compact_indices(const uint8_t* mask, int32_t* out, size_t n) {
    size_t f = 0;
    for (size_t i = 0; i < n; ++i)
        if (mask[i]) out[f++] = (int32_t)i;
    for (size_t i = 0; i < n; ++i)
        if (!mask[i]) out[f++] = (int32_t)i;
}
/* src/simd/kernels_scalar.cpp:33-48 */
void orc_match_first_equal(const int32_t* ra, size_t n, const int32_t* rb, size_t m,
                           int32_t* row_out) {
    for (size_t i = 0; i < n; ++i) {
        row_out[i] = -1;
        if (ra[i] == 0) continue;
        for (size_t j = 0; j < m; ++j)
            if (rb[j] == ra[i]) {
                row_out[i] = (int32_t)j;
                break;
            }
    }
}
/* src/simd/kernels_scalar.cpp:50-54 (bitwise select) */
void orc_blend_i64(const uint8_t* mask, const int64_t* a, const int64_t* b, int64_t* out,
                   size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = mask[i] ? a[i] : b[i];
}
void orc_blend_f64(const uint8_t* mask, const double* a, const double* b, double* out, size_t n) {
    for (size_t i = 0; i < n; ++i) memcpy(&out[i], mask[i] ? &a[i] : &b[i], 8);
}
void orc_blend_u8(const uint8_t* mask, const uint8_t* a, const uint8_t* b, uint8_t* out,
                  size_t n) {
    for (size_t i = 0; i < n; ++i) out[i] = mask[i] ? a[i] : b[i];
}

/* tests/support/oracle.cpp:11-31 */
int32_t orc_pair(const uint8_t* target, int32_t n, const uint8_t* valid, int32_t m,
                 int32_t* slots, int32_t* rows) {
    int32_t p = 0, q = 0;
    for (int32_t i = 0; i < n; ++i)
        if (target[i]) slots[p++] = i;
    for (int32_t j = 0; j < m; ++j)
        if (valid[j]) rows[q++] = j;
    return p < q ? p : q;
}

/* lifecycle.cpp:124-142 + agent_set.cpp:45-58 */
int32_t orc_remove_agents(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* e,
                          double* w, uint8_t* f, const uint8_t* kill, int recycle,
                          int64_t* retired, int32_t* n_retired) {
    int32_t killed = 0;
    for (int32_t i = 0; i < cap; ++i) {
        if (!(active[i] && kill[i])) continue;
        if (recycle) retired[(*n_retired)++] = ids[i];
        active[i] = 0;
        ids[i] = 0;
        ages[i] = 0;
        e[i] = 0;
        w[i] = 0.0;
        f[i] = 0;
        ++killed;
    }
    return killed;
}

/* lifecycle.cpp:144-195: pairs in ascending slot order (k-th free slot <-> k-th valid row) */
int32_t orc_spawn_agents(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* types,
                         int64_t* e, double* w, uint8_t* f, int64_t* next_id, int recycle,
                         int64_t* retired, int32_t* n_retired, int32_t m, const int64_t* re,
                         const double* rw, const uint8_t* rf, const uint8_t* valid, int set_type,
                         int64_t agent_type, int32_t* slots, int32_t* rows, int32_t* dropped) {
    int32_t q = 0, k = 0, j = 0;
    for (int32_t r = 0; r < m; ++r) q += valid[r] != 0;
    for (int32_t i = 0; i < cap; ++i) {
        if (active[i]) continue;
        while (j < m && !valid[j]) ++j;
        if (j >= m) break;
        slots[k] = i;
        rows[k] = j;
        e[i] = re[j];
        w[i] = rw[j];
        f[i] = rf[j];
        active[i] = 1;
        if (recycle && *n_retired > 0)
            ids[i] = retired[--(*n_retired)];
        else
            ids[i] = (*next_id)++;
        ages[i] = 0;
        if (set_type) types[i] = agent_type;
        ++k;
        ++j;
    }
    *dropped = q - k;
    return k;
}

/* kernels.cpp:52-73: std::stable_sort of the identity permutation by key; here a
 * bottom-up merge sort (also stable). */
int orc_sort_perm(const double* key, const uint8_t* active, int32_t n, int descending,
                  int32_t* perm) {
    for (int32_t i = 0; i < n; ++i)
        if (active[i] && !isfinite(key[i])) return 2;
    int32_t* tmp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
    for (int32_t i = 0; i < n; ++i) perm[i] = i;
    int32_t *src = perm, *dst = tmp;
    for (int32_t w = 1; w < n; w *= 2) {
        for (int32_t lo = 0; lo < n; lo += 2 * w) {
            int32_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
            int32_t a = lo, b = mid, k = lo;
            while (a < mid && b < hi) {
                const double ka = key[src[a]], kb = key[src[b]];
                /* take b first only when strictly before a (stability) */
                const int b_first = descending ? (kb > ka) : (kb < ka);
                dst[k++] = b_first ? src[b++] : src[a++];
            }
            while (a < mid) dst[k++] = src[a++];
            while (b < hi) dst[k++] = src[b++];
        }
        int32_t* t = src;
        src = dst;
        dst = t;
    }
    if (src != perm) memcpy(perm, src, sizeof(int32_t) * (size_t)n);
    free(tmp);
    return 0;
}

/* ------------------------------------------------------------------ predation */
/* src/models/predation.cpp:13-15 */
static const int kNeigh[8][2] = {{-1, -1}, {-1, 0}, {-1, 1}, {0, -1},
                                 {0, 1},   {1, -1}, {1, 0},  {1, 1}};

static void species_alloc(orc_species* s, int32_t cap) {
    size_t n = (size_t)(cap > 0 ? cap : 1);
    s->capacity = cap;
    s->active = (uint8_t*)calloc(n, 1);
    s->ids = (int64_t*)calloc(n, 8);
    s->types = (int64_t*)calloc(n, 8);
    s->ages = (int64_t*)calloc(n, 8);
    s->x = (int64_t*)calloc(n, 8);
    s->y = (int64_t*)calloc(n, 8);
    s->energy = (double*)calloc(n, 8);
}

static void species_free(orc_species* s) {
    free(s->active);
    free(s->ids);
    free(s->types);
    free(s->ages);
    free(s->x);
    free(s->y);
    free(s->energy);
}

/* agent_set.cpp:45-58: zero state, id, age, active; type kept */
static void reset_slot(orc_species* s, int32_t i) {
    s->active[i] = 0;
    s->ids[i] = 0;
    s->ages[i] = 0;
    s->x[i] = 0;
    s->y[i] = 0;
    s->energy[i] = 0.0;
}

/* predation.cpp:22-33 + lifecycle.cpp:11-85 (create_agents; field ordinals x=0,y=1,energy=2,
 * draws for ALL slots from seed.split(CreateField=1).split(ordinal), then reset slots>=n0) */
static void create_species(orc_species* s, int32_t cap, int32_t n0, int32_t W, int32_t H,
                           double gain, uint64_t seed, int64_t type) {
    species_alloc(s, cap);
    const uint64_t root = orc_split(seed, 1);
    const uint64_t sx = orc_split(root, 0), sy = orc_split(root, 1), se = orc_split(root, 2);
    const int64_t ehi = 2 * (int64_t)gain + 1;
    for (int32_t i = 0; i < cap; ++i) {
        s->x[i] = orc_uniform_int(sx, (uint64_t)i, 0, W);
        s->y[i] = orc_uniform_int(sy, (uint64_t)i, 0, H);
        s->energy[i] = (double)orc_uniform_int(se, (uint64_t)i, 1, ehi);
        s->types[i] = type;
    }
    for (int32_t i = 0; i < n0; ++i) {
        s->active[i] = 1;
        s->ids[i] = i;
    }
    for (int32_t i = n0; i < cap; ++i) reset_slot(s, i);
    s->num_active = n0;
    s->next_id = n0;
}

/* predation.cpp:154-165 */
/* predation.cpp:154-164: NULL where init_predation throws -- the initial counts
 * (CapacityError), a negative capacity (lifecycle.cpp:55-58), or an empty draw range for any
 * slot of a non-empty species (rng.cpp:30-36): x in [0, W), y in [0, H), energy in
 * [1, 2*trunc(gain) + 1). */
orc_pred* orc_pred_create(const orc_pred_config* cfg, uint64_t seed) {
    if (cfg->n_sheep0 > cfg->sheep_capacity || cfg->n_wolves0 > cfg->wolf_capacity) return NULL;
    {
        const int64_t cap[2] = {cfg->sheep_capacity, cfg->wolf_capacity};
        const double gain[2] = {cfg->energy_gain_sheep, cfg->energy_gain_wolf};
        for (int s = 0; s < 2; ++s) {
            if (cap[s] < 0) return NULL;
            if (cap[s] > 0 && (cfg->width < 1 || cfg->height < 1 || !(gain[s] >= 1.0))) return NULL;
        }
    }
    orc_pred* p = (orc_pred*)calloc(1, sizeof(orc_pred));
    p->cfg = *cfg;
    p->seed = seed;
    const size_t cells = (size_t)cfg->width * (size_t)cfg->height;
    p->ready = (uint8_t*)malloc(cells ? cells : 1);
    memset(p->ready, 1, cells);
    p->regrow = (int64_t*)calloc(cells ? cells : 1, 8);
    create_species(&p->sp[0], cfg->sheep_capacity, cfg->n_sheep0, cfg->width, cfg->height,
                   cfg->energy_gain_sheep, orc_split(seed, 20), 0);
    create_species(&p->sp[1], cfg->wolf_capacity, cfg->n_wolves0, cfg->width, cfg->height,
                   cfg->energy_gain_wolf, orc_split(seed, 21), 1);
    return p;
}

void orc_pred_free(orc_pred* p) {
    if (!p) return;
    species_free(&p->sp[0]);
    species_free(&p->sp[1]);
    free(p->ready);
    free(p->regrow);
    free(p);
}

/* predation.cpp:35-49 + lifecycle.cpp:87-122 (step_agents: transition, blend placeholders
 * to 0, age++ on active) */
static void move_species(orc_species* s, int32_t W, int32_t H, uint64_t stream) {
    for (int32_t i = 0; i < s->capacity; ++i) {
        if (s->active[i]) {
            const int64_t u = orc_uniform_int(stream, (uint64_t)i, 0, 8);
            s->x[i] = (s->x[i] + kNeigh[u][0] + W) % W;
            s->y[i] = (s->y[i] + kNeigh[u][1] + H) % H;
            s->ages[i] += 1;
        } else {
            s->x[i] = 0;
            s->y[i] = 0;
            s->energy[i] = 0.0;
        }
    }
}

/* lifecycle.cpp:124-142 */
static void remove_masked(orc_species* s, const uint8_t* kill) {
    int32_t killed = 0;
    for (int32_t i = 0; i < s->capacity; ++i)
        if (s->active[i] && kill[i]) {
            reset_slot(s, i);
            ++killed;
        }
    s->num_active -= killed;
}

/* predation.cpp:76-137 + lifecycle.cpp:144-195 (spawn via rank-match of !active vs valid) */
static void reproduce(orc_species* s, const orc_pred_config* cfg, double prob, uint64_t stream,
                      int64_t type, orc_species_events* ev) {
    const int32_t n = s->capacity;
    uint8_t* valid = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
    int64_t* cx = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t* cy = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double* ce = (double*)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    for (int32_t i = 0; i < n; ++i) {
        if (!s->active[i] || s->energy[i] <= cfg->metabolism) continue;
        if (!orc_bernoulli(stream, (uint64_t)i, prob)) continue;
        /* quantize_energy, predation.cpp:141-143 */
        const double child = floor((cfg->reproduce_energy_frac * s->energy[i]) / 0x1p-20) * 0x1p-20;
        s->energy[i] -= child;
        cx[i] = s->x[i];
        cy[i] = s->y[i];
        ce[i] = child;
        valid[i] = 1;
    }
    /* k-th free slot (ascending) <- k-th valid row (ascending) */
    int32_t q = 0;
    for (int32_t i = 0; i < n; ++i) q += valid[i] ? 1 : 0;
    int32_t row = 0, spawned = 0;
    for (int32_t slot = 0; slot < n && spawned < q; ++slot) {
        if (s->active[slot]) continue;
        while (!valid[row]) ++row;
        s->x[slot] = cx[row];
        s->y[slot] = cy[row];
        s->energy[slot] = ce[row];
        s->active[slot] = 1;
        s->ids[slot] = s->next_id++;
        s->ages[slot] = 0;
        s->types[slot] = type;
        ++row;
        ++spawned;
    }
    s->num_active += spawned;
    ev->births += spawned;
    ev->births_dropped += q - spawned;
    /* predation.cpp:121-135: energy of the dropped (highest-slot) rows */
    for (; row < n; ++row)
        if (valid[row]) ev->energy_dropped_births += ce[row];
    free(valid);
    free(cx);
    free(cy);
    free(ce);
}

/* predation.cpp:167-263 */
void orc_pred_step(orc_pred* p, int64_t t, orc_pred_events* ev_out) {
    const orc_pred_config* cfg = &p->cfg;
    orc_pred_events ev;
    memset(&ev, 0, sizeof ev);
    const int32_t W = cfg->width, H = cfg->height;
    orc_species* sh = &p->sp[0];
    orc_species* wo = &p->sp[1];
    const uint64_t ut = (uint64_t)t;

    /* 1. move (PredMove = 3) */
    const uint64_t move_root = orc_split(orc_split(p->seed, 3), ut);
    move_species(sh, W, H, orc_split(move_root, 0));
    move_species(wo, W, H, orc_split(move_root, 1));

    /* 2a. graze: ascending sheep slots, first on a ready cell eats (predation.cpp:178-195) */
    for (int32_t i = 0; i < sh->capacity; ++i) {
        if (!sh->active[i]) continue;
        const size_t c = (size_t)sh->y[i] * (size_t)W + (size_t)sh->x[i];
        if (p->ready[c]) {
            p->ready[c] = 0;
            p->regrow[c] = cfg->regrow_delay;
            sh->energy[i] += cfg->energy_gain_sheep;
            ++ev.grass_eaten;
        }
    }

    /* 2b. predation: k-th wolf (slot order) in a cell takes the k-th sheep (predation.cpp:197-239) */
    {
        const size_t cells = (size_t)W * (size_t)H;
        int32_t* head = (int32_t*)malloc(sizeof(int32_t) * (cells ? cells : 1));
        int32_t* tail = (int32_t*)malloc(sizeof(int32_t) * (cells ? cells : 1));
        int32_t* next = (int32_t*)malloc(sizeof(int32_t) * (size_t)(sh->capacity > 0 ? sh->capacity : 1));
        uint8_t* eaten = (uint8_t*)calloc((size_t)(sh->capacity > 0 ? sh->capacity : 1), 1);
        for (size_t c = 0; c < cells; ++c) head[c] = tail[c] = -1;
        for (int32_t i = 0; i < sh->capacity; ++i) next[i] = -1;
        for (int32_t i = 0; i < sh->capacity; ++i) {
            if (!sh->active[i]) continue;
            const size_t c = (size_t)sh->y[i] * (size_t)W + (size_t)sh->x[i];
            if (head[c] < 0)
                head[c] = i;
            else
                next[tail[c]] = i;
            tail[c] = i;
        }
        for (int32_t i = 0; i < wo->capacity; ++i) {
            if (!wo->active[i]) continue;
            const size_t c = (size_t)wo->y[i] * (size_t)W + (size_t)wo->x[i];
            const int32_t v = head[c];
            if (v < 0) continue;
            head[c] = next[v];
            eaten[v] = 1;
            ev.sheep.energy_removed_deaths += sh->energy[v];
            ++ev.sheep.deaths;
            ++ev.sheep_eaten_by_wolves;
            wo->energy[i] += cfg->energy_gain_wolf;
        }
        remove_masked(sh, eaten);
        free(head);
        free(tail);
        free(next);
        free(eaten);
    }

    /* 3+4. metabolize, then starve (predation.cpp:51-74, 241-245) */
    orc_species* sp[2] = {sh, wo};
    orc_species_events* se[2] = {&ev.sheep, &ev.wolves};
    for (int k = 0; k < 2; ++k)
        for (int32_t i = 0; i < sp[k]->capacity; ++i)
            if (sp[k]->active[i]) {
                sp[k]->energy[i] -= cfg->metabolism;
                ++se[k]->metabolized;
            }
    for (int k = 0; k < 2; ++k) {
        uint8_t* kill = (uint8_t*)calloc((size_t)(sp[k]->capacity > 0 ? sp[k]->capacity : 1), 1);
        for (int32_t i = 0; i < sp[k]->capacity; ++i)
            if (sp[k]->active[i] && sp[k]->energy[i] <= 0.0) {
                kill[i] = 1;
                se[k]->energy_removed_deaths += sp[k]->energy[i];
                ++se[k]->deaths;
            }
        remove_masked(sp[k], kill);
        free(kill);
    }

    /* 5. reproduce (PredReproduce = 4) */
    const uint64_t rep_root = orc_split(orc_split(p->seed, 4), ut);
    reproduce(sh, cfg, cfg->reproduce_prob_sheep, orc_split(rep_root, 0), 0, &ev.sheep);
    reproduce(wo, cfg, cfg->reproduce_prob_wolf, orc_split(rep_root, 1), 1, &ev.wolves);

    /* 6. regrow (predation.cpp:252-258) */
    const size_t cells = (size_t)W * (size_t)H;
    for (size_t c = 0; c < cells; ++c)
        if (p->regrow[c] > 0 && --p->regrow[c] == 0) p->ready[c] = 1;

    p->ev = ev;
    if (ev_out) *ev_out = ev;
}

/* predation.cpp:265-272, 281-287 */
void orc_pred_metrics(const orc_pred* p, int64_t* out4) {
    out4[0] = p->sp[0].num_active;
    out4[1] = p->sp[1].num_active;
    out4[2] = orc_count_true(p->ready, (size_t)p->cfg.width * (size_t)p->cfg.height);
    out4[3] = p->ev.sheep.births_dropped + p->ev.wolves.births_dropped;
}

static uint64_t fnv(uint64_t h, const void* d, size_t n) {
    const uint8_t* b = (const uint8_t*)d;
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

uint64_t orc_pred_hash(const orc_pred* p, int with_world) {
    uint64_t h = 0xcbf29ce484222325ULL;
    for (int k = 0; k < 2; ++k) {
        const orc_species* s = &p->sp[k];
        const size_t n = (size_t)s->capacity;
        h = fnv(h, s->active, n);
        h = fnv(h, s->ids, n * 8);
        h = fnv(h, s->ages, n * 8);
        h = fnv(h, s->x, n * 8);
        h = fnv(h, s->y, n * 8);
        h = fnv(h, s->energy, n * 8);
    }
    if (with_world) {
        const size_t cells = (size_t)p->cfg.width * (size_t)p->cfg.height;
        h = fnv(h, p->ready, cells);
        h = fnv(h, p->regrow, cells * 8);
    }
    return h;
}

orc_species* orc_pred_species(orc_pred* p, int species) { return &p->sp[species ? 1 : 0]; }
uint8_t* orc_pred_ready(orc_pred* p) { return p->ready; }
int64_t* orc_pred_regrow(orc_pred* p) { return p->regrow; }

/* batch.cpp:21-101 with one thread; rows in (replica, step) order, t = 1..steps */
int orc_run_batch(const orc_pred_config* cfg, uint64_t master, int32_t replicas, int64_t steps,
                  double* metrics_out) {
    for (int32_t r = 0; r < replicas; ++r) {
        orc_pred* p = orc_pred_create(cfg, orc_replica_seed(master, r));
        if (!p) return 1;
        for (int64_t t = 1; t <= steps; ++t) {
            orc_pred_step(p, t, NULL);
            int64_t m[4];
            orc_pred_metrics(p, m);
            double* o = metrics_out + ((size_t)r * (size_t)steps + (size_t)(t - 1)) * 4;
            for (int j = 0; j < 4; ++j) o[j] = (double)m[j];
        }
        orc_pred_free(p);
    }
    return 0;
}


/* ------------------------------------------------------------------ traffic */
/* rng.hpp:33-35 stream tags */
enum { ORC_TRAFFIC_SIGNAL = 5, ORC_TRAFFIC_PROPOSE = 6, ORC_TRAFFIC_SPAWN = 7 };

orc_traffic* orc_traffic_create(const orc_traffic_config* cfg, uint64_t seed) {
    if (cfg->period < 1 || cfg->length < 1) return NULL;
    orc_traffic* m = (orc_traffic*)calloc(1, sizeof(orc_traffic));
    m->length = cfg->length;
    m->period = cfg->period;
    /* SignalSchedule::from_config (traffic.cpp:8-17) */
    long long gl = llround((double)cfg->period * cfg->green_fraction);
    m->green_len = gl < 0 ? 0 : (gl > cfg->period ? cfg->period : gl);
    m->phase = orc_uniform_int(orc_split(seed, ORC_TRAFFIC_SIGNAL), 0, 0, cfg->period);
    m->seed = seed;
    /* Road::empty (traffic.cpp:19-29): capacity 3*length, lane/cell int columns */
    const size_t n = (size_t)(3 * cfg->length);
    m->capacity = (int32_t)n;
    m->active = (uint8_t*)calloc(n, 1);
    m->ids = (int64_t*)calloc(n, 8);
    m->ages = (int64_t*)calloc(n, 8);
    m->lane = (int64_t*)calloc(n, 8);
    m->cell = (int64_t*)calloc(n, 8);
    m->occupancy = (int32_t*)malloc(n * 4);
    for (size_t i = 0; i < n; ++i) m->occupancy[i] = -1;
    return m;
}

void orc_traffic_free(orc_traffic* m) {
    if (!m) return;
    free(m->active);
    free(m->ids);
    free(m->ages);
    free(m->lane);
    free(m->cell);
    free(m->occupancy);
    free(m);
}

int orc_traffic_rebuild(orc_traffic* m) {
    const int32_t n = m->capacity;
    for (int32_t c = 0; c < n; ++c) m->occupancy[c] = -1;
    for (int32_t i = 0; i < n; ++i) {
        if (!m->active[i]) continue;
        const int64_t c = m->lane[i] * m->length + m->cell[i];
        if (m->occupancy[c] != -1) return 1;
        m->occupancy[c] = i;
    }
    return 0;
}

void orc_traffic_propose(const orc_traffic* m, uint64_t stream, int green, uint8_t* kind,
                         int64_t* to_lane, int64_t* to_cell) {
    for (int32_t i = 0; i < m->capacity; ++i) {
        kind[i] = 0;
        to_lane[i] = 0;
        to_cell[i] = 0;
        if (!m->active[i]) continue;
        const int64_t lane = m->lane[i], cell = m->cell[i];
        if (cell == m->length - 1) { /* exit column: no draw */
            kind[i] = green ? 2 : 0;
            continue;
        }
        int64_t opt[3];
        int n = 0;
        opt[n++] = lane; /* forward, forward-left, forward-right */
        if (lane > 0) opt[n++] = lane - 1;
        if (lane < 2) opt[n++] = lane + 1;
        const int64_t pick = orc_uniform_int(stream, (uint64_t)i, 0, n);
        kind[i] = 1;
        to_lane[i] = opt[pick];
        to_cell[i] = cell + 1;
    }
}

int orc_traffic_resolve(const orc_traffic* m, const uint8_t* kind, const int64_t* to_lane,
                        const int64_t* to_cell, uint8_t* accepted) {
    const int32_t n = m->capacity;
    const size_t cells = (size_t)n;
    int32_t* winner = (int32_t*)malloc(cells * 4);
    int* prio_of = (int*)malloc(cells * sizeof(int));
    for (size_t c = 0; c < cells; ++c) {
        winner[c] = -1;
        prio_of[c] = 99;
    }
    int rc = 0;
    for (int32_t i = 0; i < n; ++i) {
        accepted[i] = 0;
    }
    for (int32_t i = 0; i < n && !rc; ++i) {
        if (!m->active[i]) continue;
        if (kind[i] == 2) {
            accepted[i] = 1; /* exit pseudo-cell: no capacity limit */
        } else if (kind[i] == 1) {
            const int64_t tl = to_lane[i], tc = to_cell[i];
            if (tl < 0 || tl >= 3 || tc < 0 || tc >= m->length) {
                rc = 2; /* ContractError */
                break;
            }
            const size_t target = (size_t)(tl * m->length + tc);
            const int prio = m->lane[i] == tl ? 0 : (m->lane[i] == tl - 1 ? 1 : 2);
            if (prio < prio_of[target]) {
                prio_of[target] = prio;
                winner[target] = i;
            }
        }
    }
    /* fixed point, in the reference's round / cell order (traffic.cpp:124-138) */
    for (int64_t round = 0; round < m->length && !rc; ++round) {
        int changed = 0;
        for (size_t c = 0; c < cells; ++c) {
            const int32_t w = winner[c];
            if (w < 0 || accepted[w]) continue;
            const int32_t occ = m->occupancy[c];
            if (occ < 0 || accepted[occ]) {
                accepted[w] = 1;
                changed = 1;
            }
        }
        if (!changed) break;
    }
    free(winner);
    free(prio_of);
    return rc;
}

/* spawn_cars (traffic.cpp:143-184) + spawn_agents' pairing (lifecycle.cpp:144-195) */
static int64_t orc_traffic_spawn(orc_traffic* m, uint64_t stream) {
    const int64_t k = orc_uniform_int(stream, 0, 0, 4);
    int64_t lanes[3] = {0, 1, 2};
    for (int64_t i = 0; i < (k < 2 ? k : 2); ++i) {
        const int64_t j = i + orc_uniform_int(stream, (uint64_t)(1 + i), 0, 3 - i);
        const int64_t tmp = lanes[i];
        lanes[i] = lanes[j];
        lanes[j] = tmp;
    }
    int64_t row_lane[3];
    int valid[3] = {0, 0, 0};
    for (int64_t r = 0; r < (k < 3 ? k : 3); ++r) {
        if (m->occupancy[lanes[r] * m->length] != -1) continue; /* occupied entry */
        row_lane[r] = lanes[r];
        valid[r] = 1;
    }
    int64_t spawned = 0;
    int r = 0;
    for (int32_t i = 0; i < m->capacity; ++i) {
        if (m->active[i]) continue;
        while (r < 3 && !valid[r]) ++r;
        if (r >= 3) break;
        m->active[i] = 1;
        m->lane[i] = row_lane[r];
        m->cell[i] = 0;
        m->ids[i] = m->next_id++;
        m->ages[i] = 0;
        ++spawned;
        ++r;
    }
    m->num_active += (int32_t)spawned;
    orc_traffic_rebuild(m);
    return spawned;
}

void orc_traffic_step(orc_traffic* m, int64_t t) {
    const int green = (((t + m->phase) % m->period + m->period) % m->period) < m->green_len;
    const size_t n = (size_t)m->capacity;
    uint8_t* kind = (uint8_t*)malloc(n);
    int64_t* tl = (int64_t*)malloc(n * 8);
    int64_t* tc = (int64_t*)malloc(n * 8);
    uint8_t* acc = (uint8_t*)malloc(n);
    orc_traffic_propose(m, orc_split(orc_split(m->seed, ORC_TRAFFIC_PROPOSE), (uint64_t)t), green,
                        kind, tl, tc);
    orc_traffic_resolve(m, kind, tl, tc, acc);
    int64_t exited = 0;
    for (size_t i = 0; i < n; ++i) {
        if (!acc[i]) continue;
        if (kind[i] == 1) { /* set_agents_mask: lane / cell <- target */
            m->lane[i] = tl[i];
            m->cell[i] = tc[i];
        } else if (kind[i] == 2 && m->active[i]) { /* remove_agents -> reset_slot */
            m->active[i] = 0;
            m->ids[i] = 0;
            m->ages[i] = 0;
            m->lane[i] = 0;
            m->cell[i] = 0;
            ++exited;
        }
    }
    m->num_active -= (int32_t)exited;
    orc_traffic_rebuild(m);
    m->spawned = orc_traffic_spawn(m, orc_split(orc_split(m->seed, ORC_TRAFFIC_SPAWN), (uint64_t)t));
    m->exited = exited;
    m->green = green;
    m->spawned_total += m->spawned;
    m->exited_total += exited;
    free(kind);
    free(tl);
    free(tc);
    free(acc);
}

void orc_traffic_metrics(const orc_traffic* m, double* out4) {
    out4[0] = (double)m->num_active;
    out4[1] = (double)m->spawned;
    out4[2] = (double)m->exited;
    out4[3] = m->green ? 1.0 : 0.0;
}

int orc_traffic_run_batch(const orc_traffic_config* cfg, uint64_t master, int32_t replicas,
                          int64_t steps, double* out) {
    for (int32_t r = 0; r < replicas; ++r) {
        orc_traffic* m = orc_traffic_create(cfg, orc_replica_seed(master, r));
        if (!m) return 1;
        for (int64_t t = 1; t <= steps; ++t) {
            orc_traffic_step(m, t);
            orc_traffic_metrics(m, out + ((size_t)r * (size_t)steps + (size_t)(t - 1)) * 4);
        }
        orc_traffic_free(m);
    }
    return 0;
}


/* ------------------------------------------------------------------ finance */
enum { ORC_FIN_PLACE = 8 }; /* rng.hpp:36-37 */
#define ORC_TICK 0x1p-7     /* finance.hpp:37 kPriceTick */

double orc_quantize_price(double raw) {
    double p = round(raw / ORC_TICK) * ORC_TICK;
    if (p < ORC_TICK) p = ORC_TICK;
    return p;
}

static void orc_book_init(orc_book* b, int32_t cap, double init_price) {
    b->capacity = cap;
    b->num_active = 0;
    b->next_id = 0;
    b->active = (uint8_t*)calloc((size_t)cap + 1, 1);
    b->ids = (int64_t*)calloc((size_t)cap + 1, 8);
    b->ages = (int64_t*)calloc((size_t)cap + 1, 8);
    b->trader = (int64_t*)calloc((size_t)cap + 1, 8);
    b->side = (int64_t*)calloc((size_t)cap + 1, 8);
    b->qty = (int64_t*)calloc((size_t)cap + 1, 8);
    b->placed = (int64_t*)calloc((size_t)cap + 1, 8);
    b->price = (double*)calloc((size_t)cap + 1, 8);
    b->last_price = orc_quantize_price(init_price);
    b->dropped = 0;
    b->volume = 0;
    b->clearing = 0.0;
}

static void orc_book_reset_slot(orc_book* b, int32_t i) { /* agent_set.cpp:45-58 */
    b->active[i] = 0;
    b->ids[i] = 0;
    b->ages[i] = 0;
    b->trader[i] = 0;
    b->side[i] = 0;
    b->qty[i] = 0;
    b->placed[i] = 0;
    b->price[i] = 0.0;
    b->num_active -= 1;
}

orc_fin* orc_fin_create(const orc_fin_config* cfg, uint64_t seed) {
    if (cfg->books < 1 || cfg->traders < 0 || cfg->book_capacity < 1 || cfg->qmax < 1) return NULL;
    orc_fin* m = (orc_fin*)calloc(1, sizeof(orc_fin));
    m->cfg = *cfg;
    m->seed = seed;
    m->cash = (double*)calloc((size_t)cfg->traders + 1, 8);
    m->holdings = (int64_t*)calloc((size_t)(cfg->books * cfg->traders) + 1, 8);
    m->books = (orc_book*)calloc((size_t)cfg->books, sizeof(orc_book));
    for (int64_t k = 0; k < cfg->books; ++k) orc_book_init(&m->books[k], (int32_t)cfg->book_capacity, cfg->init_price);
    return m;
}

void orc_fin_free(orc_fin* m) {
    if (!m) return;
    for (int64_t k = 0; k < m->cfg.books; ++k) {
        orc_book* b = &m->books[k];
        free(b->active);
        free(b->ids);
        free(b->ages);
        free(b->trader);
        free(b->side);
        free(b->qty);
        free(b->placed);
        free(b->price);
    }
    free(m->books);
    free(m->cash);
    free(m->holdings);
    free(m);
}

/* place_orders (finance.cpp:74-123): row i = trader i; spawn into the lowest free slots */
static void orc_fin_place(const orc_fin* m, orc_book* b, uint64_t stream, int64_t t) {
    const orc_fin_config* c = &m->cfg;
    int64_t q = 0, spawned = 0;
    int32_t slot = 0;
    for (int64_t i = 0; i < c->traders; ++i) {
        const uint64_t base = 4 * (uint64_t)i;
        if (!(orc_uniform_double(stream, base) < c->p_order)) continue;
        const int64_t side = orc_uniform_int(stream, base + 1, 0, 2);
        const double eps = -c->delta + 2.0 * c->delta * orc_uniform_double(stream, base + 2);
        const int64_t qty = orc_uniform_int(stream, base + 3, 1, c->qmax + 1);
        const double price = orc_quantize_price(b->last_price * (1.0 + eps));
        ++q;
        while (slot < b->capacity && b->active[slot]) ++slot;
        if (slot >= b->capacity) continue; /* no free slot left: dropped */
        b->active[slot] = 1;
        b->ids[slot] = b->next_id++;
        b->ages[slot] = 0;
        b->trader[slot] = i;
        b->side[slot] = side;
        b->price[slot] = price;
        b->qty[slot] = qty;
        b->placed[slot] = t;
        b->num_active += 1;
        ++spawned;
    }
    b->dropped = q - spawned;
}

/* sorted_side comparator (finance.cpp:27-36): price (desc for buys), placed, id */
static const orc_book* g_sort_book;
static int g_sort_desc;
static int orc_fin_before(int32_t a, int32_t bb) {
    const orc_book* b = g_sort_book;
    if (b->price[a] != b->price[bb]) return g_sort_desc ? b->price[a] > b->price[bb] : b->price[a] < b->price[bb];
    if (b->placed[a] != b->placed[bb]) return b->placed[a] < b->placed[bb];
    return b->ids[a] < b->ids[bb];
}
static void orc_fin_sort(int32_t* v, int32_t n) { /* stable insertion sort (n is small) */
    for (int32_t i = 1; i < n; ++i) {
        const int32_t x = v[i];
        int32_t j = i - 1;
        while (j >= 0 && orc_fin_before(x, v[j])) {
            v[j + 1] = v[j];
            --j;
        }
        v[j + 1] = x;
    }
}

int32_t orc_fin_match(orc_book* b, int64_t* f_trader, int64_t* f_side, int64_t* f_qty, double* f_amount) {
    const int32_t n = b->capacity;
    int32_t* buys = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int32_t* sells = (int32_t*)malloc(sizeof(int32_t) * (size_t)(n + 1));
    int64_t* bcum = (int64_t*)malloc(8 * (size_t)(n + 1));
    int64_t* scum = (int64_t*)malloc(8 * (size_t)(n + 1));
    int32_t nb = 0, ns = 0, nf = 0;
    for (int32_t i = 0; i < n; ++i) {
        if (!b->active[i]) continue;
        if (b->side[i] == 0)
            buys[nb++] = i;
        else if (b->side[i] == 1)
            sells[ns++] = i;
    }
    g_sort_book = b;
    g_sort_desc = 1;
    orc_fin_sort(buys, nb);
    g_sort_desc = 0;
    orc_fin_sort(sells, ns);
    int64_t run = 0;
    for (int32_t i = 0; i < nb; ++i) bcum[i] = (run += b->qty[buys[i]]);
    run = 0;
    for (int32_t j = 0; j < ns; ++j) scum[j] = (run += b->qty[sells[j]]);
    b->volume = 0;
    int64_t volume = 0;
    if (nb > 0 && ns > 0) {
        for (int32_t i = 0; i < nb; ++i) {
            int32_t feasible = 0; /* upper_bound of the buy price in the ascending sell prices */
            while (feasible < ns && !(b->price[buys[i]] < b->price[sells[feasible]])) ++feasible;
            if (feasible == 0) continue;
            const int64_t v = bcum[i] < scum[feasible - 1] ? bcum[i] : scum[feasible - 1];
            if (v > volume) volume = v;
        }
    }
    if (volume > 0) {
        int32_t mb = 0, ms = 0;
        while (bcum[mb] < volume) ++mb;
        while (scum[ms] < volume) ++ms;
        const double clearing = (b->price[buys[mb]] + b->price[sells[ms]]) / 2.0;
        uint8_t* exhausted = (uint8_t*)calloc((size_t)n + 1, 1);
        for (int side = 0; side < 2; ++side) {
            const int32_t* v = side == 0 ? buys : sells;
            const int32_t cnt = side == 0 ? nb : ns;
            int64_t remaining = volume;
            for (int32_t j = 0; j < cnt && remaining > 0; ++j) {
                const int32_t i = v[j];
                const int64_t f = b->qty[i] < remaining ? b->qty[i] : remaining;
                b->qty[i] -= f;
                remaining -= f;
                if (b->qty[i] == 0) exhausted[i] = 1;
                if (f_trader) {
                    f_trader[nf] = b->trader[i];
                    f_side[nf] = side;
                    f_qty[nf] = f;
                    f_amount[nf] = (double)f * clearing;
                }
                ++nf;
            }
        }
        for (int32_t i = 0; i < n; ++i)
            if (exhausted[i] && b->active[i]) orc_book_reset_slot(b, i);
        free(exhausted);
        b->last_price = clearing;
        b->volume = volume;
        b->clearing = clearing;
    }
    free(buys);
    free(sells);
    free(bcum);
    free(scum);
    return nf;
}

void orc_fin_step(orc_fin* m, int64_t t) {
    const orc_fin_config* c = &m->cfg;
    const uint64_t root = orc_split(orc_split(m->seed, ORC_FIN_PLACE), (uint64_t)t);
    for (int64_t k = 0; k < c->books; ++k) orc_fin_place(m, &m->books[k], orc_split(root, (uint64_t)k), t);
    const size_t cap = (size_t)c->book_capacity + 1;
    int64_t* ft = (int64_t*)malloc(8 * cap * 2);
    int64_t* fs = (int64_t*)malloc(8 * cap * 2);
    int64_t* fq = (int64_t*)malloc(8 * cap * 2);
    double* fa = (double*)malloc(8 * cap * 2);
    for (int64_t k = 0; k < c->books; ++k) { /* settlement folds books in order */
        const int32_t nf = orc_fin_match(&m->books[k], ft, fs, fq, fa);
        int64_t* h = m->holdings + k * c->traders;
        for (int32_t q = 0; q < nf; ++q) {
            if (fs[q] == 0) {
                m->cash[ft[q]] -= fa[q];
                h[ft[q]] += fq[q];
            } else {
                m->cash[ft[q]] += fa[q];
                h[ft[q]] -= fq[q];
            }
        }
    }
    free(ft);
    free(fs);
    free(fq);
    free(fa);
    for (int64_t k = 0; k < c->books; ++k) { /* cancel at the age limit (finance.cpp:236-245) */
        orc_book* b = &m->books[k];
        for (int32_t i = 0; i < b->capacity; ++i)
            if (b->active[i] && t - b->placed[i] >= c->max_order_age) orc_book_reset_slot(b, i);
    }
}

void orc_fin_metrics(const orc_fin* m, double* rows) {
    for (int64_t k = 0; k < m->cfg.books; ++k) {
        const orc_book* b = &m->books[k];
        int64_t nb = 0, ns = 0;
        for (int32_t i = 0; i < b->capacity; ++i) {
            if (!b->active[i]) continue;
            if (b->side[i] == 0)
                ++nb;
            else
                ++ns;
        }
        double* r = rows + k * 6;
        r[0] = (double)k;
        r[1] = b->last_price;
        r[2] = (double)nb;
        r[3] = (double)ns;
        r[4] = (double)b->volume;
        r[5] = (double)b->dropped;
    }
}

int orc_fin_run_batch(const orc_fin_config* cfg, uint64_t master, int32_t replicas, int64_t steps, double* rows) {
    for (int32_t r = 0; r < replicas; ++r) {
        orc_fin* m = orc_fin_create(cfg, orc_replica_seed(master, r));
        if (!m) return 1;
        for (int64_t t = 1; t <= steps; ++t) {
            orc_fin_step(m, t);
            orc_fin_metrics(m, rows + (((size_t)r * (size_t)steps + (size_t)(t - 1)) * (size_t)cfg->books) * 6);
        }
        orc_fin_free(m);
    }
    return 0;
}

/* FNV-1a-64 helper for state hashes (test bookkeeping, not a reference algorithm) */
uint64_t orc_fnv1a(uint64_t h, const void* data, size_t n) { return fnv(h, data, n); }
