/*
 * abmx_cuda.h — C-ABI of the B200-native (sm_100a) engine for the Abmax hot path
 * (arXiv 2508.16508; reference C++ implementation "abmx" under /root/reference/proj).
 *
 * Plain pointers and sizes only. Three layers, each citing the reference interface it
 * replaces:
 *
 *  1. KernelTable drop-in (host pointers, synchronous, bit-identical to the scalar
 *     table) — replaces abmx::simd::KernelTable, include/abmx/simd/kernels.hpp:15-43.
 *     abmx_cuda_kernel_table() returns a struct with the SAME layout as KernelTable,
 *     so the reference's dispatch (src/simd/dispatch.cpp:16-58) can hand it out as a
 *     third backend; see INTEGRATION.md.
 *  2. The same entries on device pointers + a cudaStream_t (passed as void*).
 *  3. Fused model engines: the predation step (PredationModel, include/abmx/models/
 *     predation.hpp:76-107, src/models/predation.cpp:167-263) for one model or a batch
 *     of replicas, and the ensemble runner (run_batch, include/abmx/batch.hpp:48-54).
 *
 * Errors: int-returning entries give ABMX_OK or one of the codes below, mirroring the
 * reference exception taxonomy (include/abmx/errors.hpp:8-40); abmx_cuda_last_error()
 * holds the message (thread-local). The void KernelTable entries cannot report errors
 * (the reference's never fail); on a CUDA failure they print and abort().
 */
#ifndef ABMX_CUDA_H
#define ABMX_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ABMX_OK 0
#define ABMX_E_DOMAIN 1   /* DomainError   errors.hpp:26-28 */
#define ABMX_E_CAPACITY 2 /* CapacityError errors.hpp:21-23 */
#define ABMX_E_SCHEMA 3   /* SchemaError   errors.hpp:16-18 */
#define ABMX_E_BATCH 4    /* BatchError    errors.hpp:36-38 */
#define ABMX_E_CUDA 5     /* device / driver failure (no reference counterpart) */
#define ABMX_E_ARG 6      /* null handle or pointer */
#define ABMX_E_CONTRACT 7 /* ContractError errors.hpp:31-33 (e.g. a move proposal off the road) */

const char* abmx_cuda_last_error(void);
/* The synchronous KernelTable entries (section 1) return void, as KernelTable fixes their
 * signatures. A CUDA failure inside one is therefore recorded, not thrown and not fatal: the call
 * leaves its outputs unwritten (count_true returns -1), abmx_cuda_table_status() turns sticky
 * ABMX_E_CUDA until abmx_cuda_table_clear_status(), and abmx_cuda_last_error() holds the
 * calling thread's message. A caller that must fail fast checks the status after its calls. */
int abmx_cuda_table_status(void);
void abmx_cuda_table_clear_status(void);
const char* abmx_cuda_version(void);
/* FNV-1a-64 of n bytes continuing from h (start with 0xcbf29ce484222325): the checksum the
 * sharded benchmarks apply to gathered metrics rows (same definition as the reference-state
 * hashes of the test fixtures). Host-side utility. */
uint64_t abmx_fnv1a64(uint64_t h, const void* data, size_t n);
/* number of kernels this library has launched in this process (all threads) */
uint64_t abmx_cuda_launch_count(void);

/* ======================================================================= 1. KernelTable
 * Host pointers. Semantics of src/simd/kernels_scalar.cpp:7-54; any nonzero mask byte
 * is true; `out` may alias `a` or `b` in the blends (lifecycle.cpp:105-111). */
void abmx_cuda_rank_scan(const uint8_t* mask, int32_t* ranks, size_t n);
int64_t abmx_cuda_count_true(const uint8_t* mask, size_t n);
void abmx_cuda_compact_indices(const uint8_t* mask, int32_t* out, size_t n);
void abmx_cuda_match_first_equal(const int32_t* ra, size_t n, const int32_t* rb, size_t m,
                                 int32_t* row_out);
void abmx_cuda_blend_i64(const uint8_t* mask, const int64_t* a, const int64_t* b, int64_t* out,
                         size_t n);
void abmx_cuda_blend_f64(const uint8_t* mask, const double* a, const double* b, double* out,
                         size_t n);
void abmx_cuda_blend_u8(const uint8_t* mask, const uint8_t* a, const uint8_t* b, uint8_t* out,
                        size_t n);

/* Layout-identical to abmx::simd::KernelTable (kernels.hpp:15-43). */
typedef struct abmx_kernel_table {
    const char* name; /* "cuda" */
    void (*rank_scan)(const uint8_t*, int32_t*, size_t);
    int64_t (*count_true)(const uint8_t*, size_t);
    void (*compact_indices)(const uint8_t*, int32_t*, size_t);
    void (*match_first_equal)(const int32_t*, size_t, const int32_t*, size_t, int32_t*);
    void (*blend_i64)(const uint8_t*, const int64_t*, const int64_t*, int64_t*, size_t);
    void (*blend_f64)(const uint8_t*, const double*, const double*, double*, size_t);
    void (*blend_u8)(const uint8_t*, const uint8_t*, const uint8_t*, uint8_t*, size_t);
} abmx_kernel_table;

const abmx_kernel_table* abmx_cuda_kernel_table(void);

/* ======================================================================= 2. device variants
 * All pointers are device pointers; `stream` is a cudaStream_t (NULL = legacy default).
 * Stream-ordered and asynchronous; temporaries come from the stream-ordered pool. */
int abmx_cuda_rank_scan_async(const uint8_t* d_mask, int32_t* d_ranks, size_t n, void* stream);
int abmx_cuda_count_true_async(const uint8_t* d_mask, size_t n, int64_t* d_count, void* stream);
int abmx_cuda_compact_indices_async(const uint8_t* d_mask, int32_t* d_out, size_t n,
                                    int64_t* d_count, void* stream);
int abmx_cuda_match_first_equal_async(const int32_t* d_ra, size_t n, const int32_t* d_rb, size_t m,
                                      int32_t* d_row_out, void* stream);
int abmx_cuda_blend_i64_async(const uint8_t* d_mask, const int64_t* d_a, const int64_t* d_b,
                              int64_t* d_out, size_t n, void* stream);
int abmx_cuda_blend_f64_async(const uint8_t* d_mask, const double* d_a, const double* d_b,
                              double* d_out, size_t n, void* stream);
int abmx_cuda_blend_u8_async(const uint8_t* d_mask, const uint8_t* d_a, const uint8_t* d_b,
                             uint8_t* d_out, size_t n, void* stream);

/* ======================================================================= 3. predation
 * Field order identical to abmx::models::PredationConfig (predation.hpp:13-27). */
typedef struct abmx_predation_config {
    int32_t width, height, n_sheep0, n_wolves0, sheep_capacity, wolf_capacity;
    double energy_gain_sheep, energy_gain_wolf, metabolism;
    double reproduce_prob_sheep, reproduce_prob_wolf, reproduce_energy_frac;
    int64_t regrow_delay;
} abmx_predation_config;

/* SpeciesEvents / PredationEvents (predation.hpp:41-57) without the birth-pair vector
 * (see abmx_predation_birth_pairs). */
typedef struct abmx_species_events {
    int64_t metabolized, deaths, births, births_dropped;
    double energy_removed_deaths, energy_dropped_births;
} abmx_species_events;

typedef struct abmx_predation_events {
    int64_t grass_eaten, sheep_eaten_by_wolves;
    abmx_species_events sheep, wolves;
} abmx_predation_events;

typedef struct abmx_predation abmx_predation; /* opaque: R replicas resident in HBM */

/* init_predation (predation.cpp:154-165) for `replicas` models with the given replica
 * seeds (RngState keys). Errors: CAPACITY (n0 > capacity, capacity >= 2^24 per species),
 * DOMAIN (regrow_delay > 2^24, width/height < 1, grid too large). */
int abmx_predation_create(const abmx_predation_config* cfg, const uint64_t* seeds,
                          int32_t replicas, abmx_predation** out);
int abmx_predation_destroy(abmx_predation* h);
/* PredationModel::step(t) for every replica (predation.cpp:277-279). Asynchronous. */
int abmx_predation_step(abmx_predation* h, int64_t t);
/* steps t0 .. t0+steps-1; metrics_out (nullable, host) receives [replicas][steps][4]
 * rows n_sheep, n_wolves, n_grass, births_dropped (predation.cpp:281-287). Synchronous
 * iff metrics_out != NULL. */
int abmx_predation_run(abmx_predation* h, int64_t t0, int64_t steps, double* metrics_out);
int abmx_predation_sync(abmx_predation* h);
/* collect_metrics of the last step: [replicas][4] */
int abmx_predation_metrics(abmx_predation* h, int64_t* out);
/* events of the last step: [replicas] */
int abmx_predation_last_events(abmx_predation* h, abmx_predation_events* out);
/* (parent slot, child slot) pairs of the last step's births, ascending child slot */
int32_t abmx_predation_birth_pairs(abmx_predation* h, int32_t replica, int32_t species,
                                   int32_t* parent, int32_t* child, int32_t cap);
/* AgentSet export/import in the reference layout (agent_set.hpp:15-77). species 0 = sheep,
 * 1 = wolves. Import requires num_active == popcount(active) and x, y in range. */
int abmx_predation_export(abmx_predation* h, int32_t replica, int32_t species, uint8_t* active,
                          int64_t* ids, int64_t* types, int64_t* ages, int64_t* x, int64_t* y,
                          double* energy, int32_t* num_active, int64_t* next_id);
int abmx_predation_import(abmx_predation* h, int32_t replica, int32_t species,
                          const uint8_t* active, const int64_t* ids, const int64_t* ages,
                          const int64_t* x, const int64_t* y, const double* energy,
                          int32_t num_active, int64_t next_id);
int abmx_predation_export_world(abmx_predation* h, int32_t replica, uint8_t* grass_ready,
                                int64_t* regrow);
int abmx_predation_import_world(abmx_predation* h, int32_t replica, const uint8_t* grass_ready,
                                const int64_t* regrow);
/* the CUDA stream all of h's work is ordered on (cudaStream_t) */
void* abmx_predation_stream(abmx_predation* h);
/* Per-kernel timing: abmx_predation_bench(..., per_kernel = 1) brackets every kernel with CUDA
 * events; abmx_predation_kernel_times returns the accumulated device milliseconds and launch
 * counts per kernel (names via abmx_predation_kernel_name); abmx_predation_set_timing resets
 * the accumulators. */
int abmx_predation_set_timing(abmx_predation* h, int enabled);
int32_t abmx_predation_kernel_count(void);
const char* abmx_predation_kernel_name(int32_t k);
int abmx_predation_kernel_times(abmx_predation* h, double* ms, int64_t* launches);
/* diagnostics: the random-access ceiling of the predation kernels' cell-word pattern (see
 * DESIGN.md §4): `cells` 16-byte words, sheep_ctas + wolf_ctas CTAs of 256 threads x 4 slots
 * with the given live fractions; mode 0 = one returning atomicExch per live slot plus one
 * atomicMax per live sheep, mode 1 = one random 16-byte read per live slot; cold = L2 flushed
 * before every launch. Event-timed like the bench's per-kernel times (microseconds). */
int abmx_diag_random_access(int64_t cells, int32_t sheep_ctas, int32_t wolf_ctas, double live_sheep,
                            double live_wolves, int32_t mode, int32_t cold, int32_t reps,
                            double* min_us, double* mean_us);
/* diagnostics: per-CTA phase timestamps (%globaltimer ns) of k_move / k_update, recorded only
 * by builds compiled with -DABMX_PRED_TRACE; [2][CTAs][8], returns the number of entries */
int abmx_predation_set_trace(abmx_predation* h, int32_t enable);
int64_t abmx_predation_trace(abmx_predation* h, uint64_t* out, int64_t cap);
/* diagnostics: in a -DABMX_CHECKED build, the id of the first device bounds check that failed in
 * the predation kernels (0 = none); -1 in normal builds */
int abmx_predation_check_status(void);
/* device-resident bytes of h (state + scratch) */
int64_t abmx_predation_device_bytes(abmx_predation* h);
/* Device-timed steps t0..t0+steps-1 for benchmarking: before each step an (untimed) write
 * of flush_bytes evicts L2; CUDA events on h's stream bracket each step (per_kernel = 0,
 * CUDA-graph launch) or each kernel (per_kernel = 1, also accumulates kernel_times).
 * step_ms[steps] receives the device milliseconds of every step. Metrics of these steps
 * are then readable with abmx_predation_fetch_metrics ([replicas][steps][4]). */
int abmx_predation_bench(abmx_predation* h, int64_t t0, int64_t steps, int64_t flush_bytes,
                         int32_t per_kernel, double* step_ms);
int abmx_predation_fetch_metrics(abmx_predation* h, double* out);

/* ======================================================================= ensemble
 * run_batch (batch.cpp:21-101) for replicas [replica_begin, replica_begin+count) of
 * master seed `master` (seeds master.split(2).split(r), batch.cpp:12-19), t = 1..steps.
 * metrics_out: host [count][steps][4] in run_batch row order. `path`: 0 auto, 1 the
 * SMEM-resident CTA-per-replica kernel, 2 the batched HBM engine. kernel_ms (nullable)
 * receives the device time of the simulation kernels. */
int abmx_ensemble_run(const abmx_predation_config* cfg, uint64_t master, int32_t replica_begin,
                      int32_t count, int64_t steps, int32_t path, double* metrics_out,
                      double* kernel_ms);
/* 1 if the SMEM-resident path supports cfg */
int abmx_ensemble_smem_fits(const abmx_predation_config* cfg);

/* One species in the reference layout (predation.cpp:22-33 fields + AgentSet lifecycle
 * columns): caller-owned host arrays of the species capacity; num_active / next_id are out. */
typedef struct abmx_species_arrays {
    uint8_t* active;
    int64_t* ids;
    int64_t* ages;
    int64_t* x;
    int64_t* y;
    double* energy;
    int32_t num_active;
    int64_t next_id;
} abmx_species_arrays;

/* run_batch on the SMEM-resident path, then the final state of batch member `replica`
 * (0-based within [replica_begin, replica_begin+count)) in the reference layout: what the
 * reference's PredationModel of that replica holds after `steps` steps. grass_ready / regrow:
 * [width*height]. ABMX_E_DOMAIN when cfg does not fit the SMEM-resident path. */
int abmx_ensemble_replica_state(const abmx_predation_config* cfg, uint64_t master,
                                int32_t replica_begin, int32_t count, int64_t steps,
                                int32_t replica, abmx_species_arrays* sheep,
                                abmx_species_arrays* wolves, uint8_t* grass_ready,
                                int64_t* regrow);

/* ======================================================================= 4. agent sets
 * The generic lifecycle and subset operations on an AgentSet whose
 * columns live in device memory. Callbacks (std::function ApplyFn / SlotUpdateFn,
 * kernels.hpp:62-102) cannot cross a C-ABI, so the apply is a COLUMN COPY: state column c of
 * a paired slot receives column c of its row (a NULL row column leaves that state column
 * alone). All entries are stream-ordered on `stream` (cudaStream_t as void*); counts stay in
 * device memory. Element sizes are 1, 4 or 8 bytes (bool / int32 / int64 / f64 columns). */
typedef struct abmx_column {
    void* data;         /* device pointer, capacity (state) or m (rows) elements */
    int32_t elem_size;  /* 1, 4 or 8 */
    int32_t pad;
} abmx_column;

/* AgentSet (agent_set.hpp:15-77). counters: device int64[3] = {num_active, next_id,
 * retired count}; retired: device int64[capacity] id stack (used when recycle_ids). */
typedef struct abmx_agent_set {
    int32_t capacity;
    int32_t recycle_ids;          /* AgentSet::set_id_recycling (agent_set.hpp:45-52) */
    uint8_t* active;
    int64_t* ids;
    int64_t* types;
    int64_t* ages;
    int64_t* counters;
    int64_t* retired;
    int32_t n_state;
    int32_t n_extra;
    const abmx_column* state;     /* host array of n_state device columns (reset on removal) */
    const abmx_column* extra;     /* params / policy columns: moved by permute and sort only */
} abmx_agent_set;

/* remove_agents (lifecycle.cpp:124-142): live slots with kill[i] != 0 are reset (active, id,
 * age, state zeroed; type kept, agent_set.cpp:45-58); with recycle_ids their ids are pushed on
 * the retired stack in slot order. d_killed (nullable, device int64): number removed.
 * One cooperative launch when the set's tiles fit on the GPU at once (see lifecycle below). */
int abmx_agents_remove(const abmx_agent_set* s, const uint8_t* d_kill, int64_t* d_killed,
                       void* stream);
/* spawn_agents (lifecycle.cpp:144-195): the k-th free slot receives the k-th valid row
 * (copy apply), id = retired.pop() while recycling and non-empty else next_id++, age 0,
 * type = agent_type if set_type. d_slots[k] / d_rows[k] (nullable, device int32, capacity /
 * m entries): pair k, k < spawned. d_result (nullable, device int64[2]): {spawned, dropped}.
 * One cooperative launch when the set's tiles fit on the GPU at once (see lifecycle below). */
int abmx_agents_spawn(const abmx_agent_set* s, int32_t m, const uint8_t* d_valid,
                      const abmx_column* rows, int32_t set_type, int64_t agent_type,
                      int32_t* d_slots, int32_t* d_rows, int64_t* d_result, void* stream);
/* One lifecycle cycle: remove_agents(kill) then spawn_agents(rows, valid) (lifecycle.cpp:124-195)
 * fused: one cooperative kernel with one grid barrier (count + tile-local free/killed-id lists,
 * barrier, removal in place + rows placed into their free slots) when the set's tiles fit on the
 * GPU at once, else two kernels (one selection
 * pass with the removal applied in place, one pairing apply); results identical to
 * abmx_agents_remove followed by abmx_agents_spawn. d_killed (nullable, device int64) = removed;
 * d_result (nullable, device int64[2]) = {spawned, dropped}. */
int abmx_agents_lifecycle(const abmx_agent_set* s, const uint8_t* d_kill, int32_t m, const uint8_t* d_valid,
                          const abmx_column* rows, int32_t set_type, int64_t agent_type, int64_t* d_killed,
                          int64_t* d_result, void* stream);
/* set_agents_rm / set_agents_sci (kernels.cpp:116-153) with the copy apply: the k-th target
 * slot receives the k-th valid row, k < min(popcount(target), popcount(valid)). With a copy
 * apply RM and SCI coincide (kernels.hpp:96-99). d_result (nullable): {pairs, valid rows};
 * d_slots / d_rows (nullable): pair k, k < pairs. One cooperative launch when the set's tiles
 * fit on the GPU at once (lifecycle fields and counters untouched). */
int abmx_agents_set_rm(const abmx_agent_set* s, const uint8_t* d_target, int32_t m,
                       const uint8_t* d_valid, const abmx_column* rows, int32_t* d_slots,
                       int32_t* d_rows, int64_t* d_result, void* stream);
int abmx_agents_set_sci(const abmx_agent_set* s, const uint8_t* d_target, int32_t m,
                        const uint8_t* d_valid, const abmx_column* rows, int32_t* d_slots,
                        int32_t* d_rows, int64_t* d_result, void* stream);
/* set_agents_mask (kernels.cpp:155-167): state column c [i] = values[c][i] where mask[i]. */
int abmx_agents_set_mask(const abmx_agent_set* s, const uint8_t* d_mask,
                         const abmx_column* values, void* stream);
/* select_agents / compact_mask (kernels.cpp:23-35): stable partition, true indices first;
 * d_count (device int64) = number of true entries. */
int abmx_agents_select(const uint8_t* d_mask, int32_t n, int32_t* d_indices, int64_t* d_count,
                       void* stream);
/* sort_agents (kernels.cpp:52-73): stable permutation by an f64 key (ascending or
 * descending); ABMX_E_DOMAIN (nothing written) if an active slot has a non-finite key.
 * Synchronises `stream` once for that check. */
int abmx_agents_sort_perm(const double* d_key, const uint8_t* d_active, int32_t n,
                          int32_t descending, int32_t* d_perm, void* stream);
/* pinned_keys (kernels.cpp:37-50, kernels.hpp:73-79): out[i] = keys[i] on active slots, +inf
 * (ascending) or -inf (descending) on placeholders, so sort_agents moves them to the tail. */
int abmx_agents_pinned_keys(const double* d_keys, const uint8_t* d_active, int32_t n, int32_t descending,
                            double* d_out, void* stream);
/* permute_agents (agent_set.cpp:92-108): every column c[i] = c[perm[i]] (gather); indices
 * outside [0, capacity) give ABMX_E_DOMAIN. */
int abmx_agents_permute(const abmx_agent_set* s, const int32_t* d_perm, void* stream);
/* sort_perm + permute; d_perm (nullable) receives the permutation. */
int abmx_agents_sort(const abmx_agent_set* s, const double* d_key, int32_t descending,
                     int32_t* d_perm, void* stream);

/* ======================================================================= 5. traffic
 * TrafficModel (include/abmx/models/traffic.hpp:84-110, src/models/traffic.cpp) for `roads`
 * independent roads at once (seeds[r] = the replica seed). Capacity 3*length slots per road;
 * state exported in the reference layout (lane / cell as int64, occupancy slot-or--1).
 * abmx_traffic_config has the field order of abmx::models::TrafficConfig (traffic.hpp:13-17). */
typedef struct abmx_traffic_config {
    int64_t length;        /* cells per lane (3 lanes) */
    int64_t period;        /* signal period */
    double green_fraction;
} abmx_traffic_config;

typedef struct abmx_traffic abmx_traffic;

int abmx_traffic_create(const abmx_traffic_config* cfg, const uint64_t* seeds, int32_t roads,
                        abmx_traffic** out);
int abmx_traffic_destroy(abmx_traffic* h);
/* TrafficModel::step(t) on every road (traffic.cpp:228-232) */
int abmx_traffic_step(abmx_traffic* h, int64_t t);
/* steps t0 .. t0+steps-1; metrics_out (nullable, host) [roads][steps][4] */
int abmx_traffic_run(abmx_traffic* h, int64_t t0, int64_t steps, double* metrics_out);
int abmx_traffic_sync(abmx_traffic* h);
/* collect_metrics of the last step (traffic.cpp:234-238): [roads][4] n_cars, spawned, exited,
 * signal_green */
int abmx_traffic_metrics(abmx_traffic* h, double* out);
int abmx_traffic_totals(abmx_traffic* h, int32_t road, int64_t* spawned_total,
                        int64_t* exited_total);
/* SignalSchedule (traffic.hpp:21-32) of a road */
int abmx_traffic_schedule(abmx_traffic* h, int32_t road, int64_t* period, int64_t* green_len,
                          int64_t* phase);
int abmx_traffic_export(abmx_traffic* h, int32_t road, uint8_t* active, int64_t* ids,
                        int64_t* ages, int64_t* lane, int64_t* cell, int32_t* occupancy,
                        int64_t* next_id, int32_t* num_active);
/* replace a road's cars (DomainError if two cars share a cell, traffic.cpp:31-44) */
int abmx_traffic_import(abmx_traffic* h, int32_t road, const uint8_t* active,
                        const int64_t* ids, const int64_t* ages, const int64_t* lane,
                        const int64_t* cell, int64_t next_id);
/* resolve_conflicts (traffic.cpp:82-140) with explicit proposals, host arrays of 3*length:
 * kind 0 stay / 1 move / 2 exit. ABMX_E_CONTRACT on a move target off the road. Acceptance is
 * the least fixed point (pointer jumping on the device); identical to the reference whenever
 * its L-round iteration converges, which holds for every propose_moves proposal. */
int abmx_traffic_resolve(int64_t length, const uint8_t* active, const int64_t* lane,
                         const int64_t* cell, const uint8_t* kind, const int64_t* to_lane,
                         const int64_t* to_cell, uint8_t* accepted);
/* timed steps (see abmx_predation_bench) */
int abmx_traffic_bench(abmx_traffic* h, int64_t t0, int64_t steps, int64_t flush_bytes,
                       int32_t per_kernel, double* step_ms);
int32_t abmx_traffic_kernel_count(void);
const char* abmx_traffic_kernel_name(int32_t k);
int abmx_traffic_kernel_times(abmx_traffic* h, double* ms, int64_t* launches);
/* run_batch of TrafficModel for replicas [replica_begin, +count) of `master`: metrics_out
 * [count][steps][4]; kernel_ms (nullable) the device time of the run */
int abmx_traffic_run_batch(const abmx_traffic_config* cfg, uint64_t master,
                           int32_t replica_begin, int32_t count, int64_t steps,
                           double* metrics_out, double* kernel_ms);
/* the same with an explicit path: 0 auto, 1 one shared-memory-resident CTA per road (roads up
 * to 3*length <= 32767 cells), 2 the batched HBM engine */
int abmx_traffic_run_batch_path(const abmx_traffic_config* cfg, uint64_t master,
                                int32_t replica_begin, int32_t count, int64_t steps,
                                int32_t path, double* metrics_out, double* kernel_ms);

/* ======================================================================= 6. finance
 * FinanceModel (include/abmx/models/finance.hpp:21-97, src/models/finance.cpp) for `markets`
 * independent markets (seeds[m] = replica seed). abmx_finance_config has the field order of
 * FinanceConfig (finance.hpp:13-22). One CTA per (market, book) with the book resident in shared
 * memory: book_capacity and traders up to 4096 (CapacityError beyond). Metrics rows are
 * collect_metrics' (finance.cpp:262-276): book_id, price, n_active_buys, n_active_sells, volume,
 * orders_dropped — one row per book. */
typedef struct abmx_finance_config {
    int64_t books, traders, book_capacity;
    double p_order, delta;
    int64_t qmax, max_order_age;
    double init_price;
} abmx_finance_config;

typedef struct abmx_finance abmx_finance;

int abmx_finance_create(const abmx_finance_config* cfg, const uint64_t* seeds, int32_t markets,
                        abmx_finance** out);
int abmx_finance_destroy(abmx_finance* h);
/* step_market at t on every market (finance.cpp:203-247) */
int abmx_finance_step(abmx_finance* h, int64_t t);
/* steps t0 .. t0+steps-1 in one launch; rows (nullable, host) [markets][steps][books][6] */
int abmx_finance_run(abmx_finance* h, int64_t t0, int64_t steps, double* rows);
/* collect_metrics of the last step: [markets][books][6] */
int abmx_finance_metrics(abmx_finance* h, double* rows);
/* a book in the reference layout; scalars[6] = last_price, dropped_this_step, last volume,
 * last clearing price, next_id, num_active */
int abmx_finance_export_book(abmx_finance* h, int32_t market, int32_t book, uint8_t* active,
                             int64_t* ids, int64_t* trader, int64_t* side, double* price,
                             int64_t* qty, int64_t* placed, double* scalars);
int abmx_finance_import_book(abmx_finance* h, int32_t market, int32_t book,
                             const uint8_t* active, const int64_t* ids, const int64_t* trader,
                             const int64_t* side, const double* price, const int64_t* qty,
                             const int64_t* placed, int64_t next_id, double last_price);
/* traders' cash [traders] and holdings [books][traders] */
int abmx_finance_export_traders(abmx_finance* h, int32_t market, double* cash,
                                int64_t* holdings);
/* match_book (finance.cpp:125-190) on one host book (arrays updated in place); fills in the
 * reference order (buys in priority order, then sells); returns the fill count, or -code */
int32_t abmx_finance_match(int32_t capacity, double last_price, uint8_t* active, int64_t* ids,
                           int64_t* trader, int64_t* side, double* price, int64_t* qty,
                           int64_t* placed, int64_t* f_trader, int64_t* f_side, int64_t* f_qty,
                           double* f_amount, double* scalars);
double abmx_finance_quantize_price(double raw); /* finance.cpp:56-61 */
/* run_batch of FinanceModel: rows [count][steps][books][6]; kernel_ms nullable */
int abmx_finance_run_batch(const abmx_finance_config* cfg, uint64_t master, int32_t replica_begin,
                           int32_t count, int64_t steps, double* rows, double* kernel_ms);

#ifdef __cplusplus
}
#endif
#endif /* ABMX_CUDA_H */
