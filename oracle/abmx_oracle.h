/*
 * abmx_oracle.h — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).
 *
 * A plain-C restatement of the reference's CPU algorithm for the predation hot path
 * (arxiv/paper_2508_16508, C++ "abmx" under /root/reference/proj). Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 *
 * Parity is PINNED: tests/test_oracle.py checks every function here against
 *   (1) the unmodified reference library built by oracle/Makefile (oracle/_ref), and
 *   (2) the committed golden vectors in tests/golden/ (generated from oracle/_ref by
 *       oracle/gen_golden.py) plus the known-answer values of SURVEY.md §8c.
 */
#ifndef ABMX_ORACLE_H
#define ABMX_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG (src/rng.cpp:12-40; schedule include/abmx/rng.hpp:7-38) ---- */
uint64_t orc_mix64(uint64_t z);
uint64_t orc_split(uint64_t key, uint64_t i);
uint64_t orc_draw(uint64_t key, uint64_t c);
double orc_uniform_double(uint64_t key, uint64_t c);
int64_t orc_uniform_int(uint64_t key, uint64_t c, int64_t lo, int64_t hi);
int orc_bernoulli(uint64_t key, uint64_t c, double p);
uint64_t orc_replica_seed(uint64_t master, int64_t r); /* batch.cpp:12-19 */

/* ---- KernelTable scalar semantics (src/simd/kernels_scalar.cpp:7-54) ---- */
void orc_rank_scan(const uint8_t* mask, int32_t* ranks, size_t n);
int64_t orc_count_true(const uint8_t* mask, size_t n);
void orc_compact_indices(const uint8_t* mask, int32_t* out, size_t n);
void orc_match_first_equal(const int32_t* ra, size_t n, const int32_t* rb, size_t m,
                           int32_t* row_out);
void orc_blend_i64(const uint8_t* mask, const int64_t* a, const int64_t* b, int64_t* out,
                   size_t n);
void orc_blend_f64(const uint8_t* mask, const double* a, const double* b, double* out, size_t n);
void orc_blend_u8(const uint8_t* mask, const uint8_t* a, const uint8_t* b, uint8_t* out,
                  size_t n);

/* Sequential pairing oracle (tests/support/oracle.cpp:11-31): the first min(p,q)
 * selected slots paired with the first min(p,q) valid rows, in order. Returns r. */
int32_t orc_pair(const uint8_t* target, int32_t n, const uint8_t* valid, int32_t m,
                 int32_t* slots, int32_t* rows);

/* remove_agents (lifecycle.cpp:124-142) on an e/w/f set: active &= !kill on live slots, killed
 * slots reset to placeholders (agent_set.cpp:45-58: active, id, age and state zeroed, type
 * kept). With recycle, killed ids are pushed on the retired stack in slot order. Returns the
 * number killed. */
int32_t orc_remove_agents(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* e,
                          double* w, uint8_t* f, const uint8_t* kill, int recycle,
                          int64_t* retired, int32_t* n_retired);

/* spawn_agents (lifecycle.cpp:144-195) with the copy apply: the k-th free slot receives the
 * k-th valid row; id = retired.pop() while the stack is non-empty (recycle), else next_id++;
 * age 0; type = agent_type when set_type. Returns spawned; writes dropped, slots, rows. */
int32_t orc_spawn_agents(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* types,
                         int64_t* e, double* w, uint8_t* f, int64_t* next_id, int recycle,
                         int64_t* retired, int32_t* n_retired, int32_t m, const int64_t* re,
                         const double* rw, const uint8_t* rf, const uint8_t* valid, int set_type,
                         int64_t agent_type, int32_t* slots, int32_t* rows, int32_t* dropped);

/* Stable sort permutation by an f64 key (kernels.cpp:52-73). Returns 0, or 2 when an
 * active slot has a non-finite key (DomainError). */
int orc_sort_perm(const double* key, const uint8_t* active, int32_t n, int descending,
                  int32_t* perm);

/* ---- predation (include/abmx/models/predation.hpp, src/models/predation.cpp) ---- */
typedef struct {
    int32_t width, height, n_sheep0, n_wolves0, sheep_capacity, wolf_capacity;
    double energy_gain_sheep, energy_gain_wolf, metabolism;
    double reproduce_prob_sheep, reproduce_prob_wolf, reproduce_energy_frac;
    int64_t regrow_delay;
} orc_pred_config;

typedef struct {
    int64_t metabolized, deaths, births, births_dropped;
    double energy_removed_deaths, energy_dropped_births;
} orc_species_events;

typedef struct {
    int64_t grass_eaten, sheep_eaten_by_wolves;
    orc_species_events sheep, wolves;
} orc_pred_events;

typedef struct {
    int32_t capacity, num_active;
    int64_t next_id;
    uint8_t* active;
    int64_t *ids, *types, *ages, *x, *y;
    double* energy;
} orc_species;

typedef struct {
    orc_pred_config cfg;
    uint64_t seed;
    orc_species sp[2]; /* 0 sheep, 1 wolves */
    uint8_t* ready;
    int64_t* regrow;
    orc_pred_events ev;
} orc_pred;

orc_pred* orc_pred_create(const orc_pred_config* cfg, uint64_t seed);
void orc_pred_free(orc_pred* p);
void orc_pred_step(orc_pred* p, int64_t t, orc_pred_events* ev);
void orc_pred_metrics(const orc_pred* p, int64_t* out4);
uint64_t orc_pred_hash(const orc_pred* p, int with_world);
/* direct pointers for tests (export/import through ctypes) */
orc_species* orc_pred_species(orc_pred* p, int species);
uint8_t* orc_pred_ready(orc_pred* p);
int64_t* orc_pred_regrow(orc_pred* p);

/* Whole ensemble (run_batch, batch.cpp:21-101) single-threaded: metrics [K][T][4]. */
int orc_run_batch(const orc_pred_config* cfg, uint64_t master, int32_t replicas, int64_t steps,
                  double* metrics_out);

/* ---- traffic (include/abmx/models/traffic.hpp, src/models/traffic.cpp) ---- */
typedef struct {
    int64_t length, period;
    double green_fraction;
} orc_traffic_config;

typedef struct {
    int64_t length, period, green_len, phase;
    uint64_t seed;
    int32_t capacity, num_active;
    int64_t next_id;
    uint8_t* active;
    int64_t *ids, *ages, *lane, *cell;
    int32_t* occupancy;                 /* [3*length]: slot or -1 */
    int64_t spawned, exited, green;     /* last step (RoadStepStats) */
    int64_t spawned_total, exited_total;
} orc_traffic;

/* NULL on DomainError (length < 1 or period < 1, traffic.cpp:8-9,20-21) */
orc_traffic* orc_traffic_create(const orc_traffic_config* cfg, uint64_t seed);
void orc_traffic_free(orc_traffic* m);
/* rebuild occupancy from the car columns; 1 if two cars share a cell (traffic.cpp:31-44) */
int orc_traffic_rebuild(orc_traffic* m);
/* propose_moves (traffic.cpp:47-80): kind 0 stay / 1 move / 2 exit */
void orc_traffic_propose(const orc_traffic* m, uint64_t stream, int green, uint8_t* kind,
                         int64_t* to_lane, int64_t* to_cell);
/* resolve_conflicts (traffic.cpp:82-140); returns 2 on a proposal outside the road */
int orc_traffic_resolve(const orc_traffic* m, const uint8_t* kind, const int64_t* to_lane,
                        const int64_t* to_cell, uint8_t* accepted);
/* step_road (traffic.cpp:186-222) + model totals (traffic.cpp:228-232) */
void orc_traffic_step(orc_traffic* m, int64_t t);
/* collect_metrics (traffic.cpp:234-238): n_cars, spawned, exited, signal_green */
void orc_traffic_metrics(const orc_traffic* m, double* out4);
/* run_batch of TrafficModel: metrics [K][T][4] */
int orc_traffic_run_batch(const orc_traffic_config* cfg, uint64_t master, int32_t replicas,
                          int64_t steps, double* metrics_out);

/* ---- finance (include/abmx/models/finance.hpp, src/models/finance.cpp) ---- */
typedef struct {
    int64_t books, traders, book_capacity;
    double p_order, delta;
    int64_t qmax, max_order_age;
    double init_price;
} orc_fin_config;

typedef struct {
    int32_t capacity, num_active;
    int64_t next_id;
    uint8_t* active;
    int64_t *ids, *ages, *trader, *side, *qty, *placed;
    double* price;
    double last_price;
    int64_t dropped, volume; /* dropped_this_step, last_trades.volume */
    double clearing;
} orc_book;

typedef struct {
    orc_fin_config cfg;
    uint64_t seed;
    double* cash;       /* [traders] */
    int64_t* holdings;  /* [books][traders] */
    orc_book* books;    /* [books] */
} orc_fin;

double orc_quantize_price(double raw);                 /* finance.cpp:56-61 */
orc_fin* orc_fin_create(const orc_fin_config* cfg, uint64_t seed);  /* init_market */
void orc_fin_free(orc_fin* m);
void orc_fin_step(orc_fin* m, int64_t t);             /* step_market */
void orc_fin_metrics(const orc_fin* m, double* rows); /* [books][6] collect_metrics */
/* match_book (finance.cpp:125-190) on one book; fills (trader, side, qty, amount) appended
 * into the arrays (capacity entries each, nullable); returns the number of fills */
int32_t orc_fin_match(orc_book* b, int64_t* f_trader, int64_t* f_side, int64_t* f_qty,
                      double* f_amount);
int orc_fin_run_batch(const orc_fin_config* cfg, uint64_t master, int32_t replicas,
                      int64_t steps, double* rows); /* [K][T][books][6] */

/* FNV-1a-64 continuation over raw bytes (start h = 0xcbf29ce484222325) */
uint64_t orc_fnv1a(uint64_t h, const void* data, size_t n);

#ifdef __cplusplus
}
#endif
#endif
