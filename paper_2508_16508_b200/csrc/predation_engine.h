// predation_engine.h — device data layout and the host-side engine object for the
// predation step (internal; the public surface is include/abmx_cuda.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/abmx_cuda.h"

namespace abmx_pred {

#ifndef ABMX_PRED_KT
#define ABMX_PRED_KT 256
#endif
#ifndef ABMX_PRED_KS
#define ABMX_PRED_KS 4
#endif
#ifndef ABMX_PRED_MINB
#define ABMX_PRED_MINB 4
#endif
constexpr int kT = ABMX_PRED_KT;      // threads per CTA
constexpr int kS = ABMX_PRED_KS;      // slots per thread (2, 4 or 8)
constexpr int kMinB = ABMX_PRED_MINB; // CTAs per SM the hot kernels are register-limited to
constexpr int kTile = kT * kS;   // slots per tile (k_move and k_update use the same tiling)
constexpr int kNumKernels = 3;   // k_move, k_cells (crowded grids only), k_update
constexpr int kGroup = 32;       // tiles per group counter (births fast path in k_move)
constexpr int kEpochClear = 128; // cell tags are cleared every kEpochClear steps (epoch8 period 255)

// Device control block (counters shared by the kernels of a step).
struct Ctl {
    unsigned occ;       // entries in the wolf-cell list this step (crowded grids)
    unsigned pool_top;  // bump allocator of the long-list sort pool (sized N_s + N_w: every
                        // agent sits in exactly one cell list, so it cannot overflow)
    unsigned pad[2];
};

// Per (replica, species) counters. next_id / num_active are double-buffered by step parity
// p = epoch & 1: the births of step e read next_id[p] and write next_id[p ^ 1].
struct SpeciesRep {
    long long next_id[2];
    int num_active[2];
    int pairs;  // births of the last step (min(free, valid))
    int Q;      // valid parent rows of the last step
};

// Per replica, per parity event accumulators (PredationEvents, predation.hpp:41-57).
// Energies are exact fixed-point multiples of 2^-20.
struct Events {
    unsigned long long grass_eaten, sheep_eaten;
    unsigned long long metabolized[2], deaths[2], births[2], dropped[2];
    long long e_removed_fx[2], e_dropped_fx[2];
};

struct Params {
    // per-step scalars (host-advanced kernel parameters)
    unsigned long long epoch;        // internal step counter (>= 1) tagging the per-cell words
    long long t;                     // the reference's step index t fed to the RNG streams
    long long* metrics;              // [R][metrics_stride][4]
    unsigned run_step, metrics_stride, needs_blend, pending;
    unsigned long long birth_epoch;  // step whose births k_move / k_finalize apply (if pending)
    unsigned birth_row;              // metrics row of that step
    unsigned book;                   // 1: the births pass also does that step's bookkeeping
    long long* host_row;             // k_book: mapped host copy of the metrics row (or null)
    long long* host_seq;             //   ... then this mapped sequence word = book_seq
    unsigned long long* book_count;  //   k_book CTAs done (device; the R-th of a call publishes)
    unsigned long long book_seq;
    // model constants
    int R, W, H, Cpad;
    long long C;
    int N[2], Npad[2], tiles[2];
    double gain[2], metab, prob[2], frac;
    int delay;     // regrow_delay if >= 1, else 0 (a grazed cell never regrows)
    int due_ring;  // due-epoch histogram ring length per replica (power of two > delay)
    int crowded;   // more slots than cells: sort-based pairing kernel instead of list walks
    int k2_ctas, status_stride;
    const unsigned long long* seeds;
    uint8_t* active[2];
    int* cell[2];
    int* age[2];
    double* energy[2];
    long long* id[2];
    int* next[2];
    uint8_t* flag[2];    // crowded grids: sheep eaten / wolf ate this step
    int* row_at[2];      // valid parent rows, tile-local compaction: parent slot
    int* rowcell[2];     //   ... its cell
    double* rowE[2];     //   ... the child's energy
    int* birth_child[2]; // child slot of birth k (for abmx_predation_birth_pairs)
    uint4* cw;               // per cell: sheep head, wolf head, lowest sheep slot, grass due epoch
    long long* n_grass;      // [R] ready cells after the last step
    unsigned* due_count;     // [R][due_ring] cells coming due at each epoch (mod ring)
    unsigned long long* status;  // [species][R][status_stride] packed (free, valid) per tile
    unsigned long long* group;   // [parity][species][R][groups] packed (free, valid) per kGroup tiles
    int groups;
    unsigned long long* occ;     // crowded grids: wolf cells (replica << 32 | cell)
    int* pool;
    long long pool_size;
    Ctl* ctl;
    SpeciesRep* rep;
    Events* ev;
    unsigned long long* trace;  // ABMX_PRED_TRACE builds: [kernel][CTA][8] %globaltimer stamps
};

const char* kernel_name(int k);

int check_create(const abmx_predation_config& c);  // init_predation's errors (predation.cu)
int check_status();  // checked builds: first failing device bounds check; -1 otherwise

struct Engine {
    abmx_predation_config cfg{};
    int R = 0;
    Params params{};
    cudaStream_t stream = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaGraphNode_t nodes[kNumKernels] = {};
    cudaGraph_t step_graph = nullptr;          // the API step: memset row, kernels, k_finalize
    cudaGraphExec_t step_exec = nullptr;
    cudaGraphNode_t step_nodes[kNumKernels + 1] = {};
    long long* h_metrics_pinned = nullptr;     // mapped pinned copy of the step() metrics row
    long long* h_metrics_dev = nullptr;        //   ... its device alias (written by k_book)
    bool host_row_valid = false;               // the mapped row holds the last step()'s row
    unsigned long long step_seq = 0;           // step() calls (the sequence k_book publishes)
    unsigned long long* d_book_count = nullptr;
    std::vector<void*> allocs;
    long long device_bytes = 0;
    unsigned long long* d_seeds = nullptr;
    long long* d_metrics_step = nullptr;  // [R][1][4]
    long long* d_run_metrics = nullptr;   // [R][steps][4]
    size_t run_metrics_bytes = 0;
    long long last_run_steps = 0;
    unsigned long long host_epoch = 1;    // epoch of the next step
    size_t move_smem = 0;                 // dynamic smem of k_move / k_finalize (tile-count prefix)
    double kernel_ms[kNumKernels] = {};
    long long kernel_launches[kNumKernels] = {};
    void* flush_buf = nullptr;
    size_t flush_cap = 0;
    unsigned long long* d_trace = nullptr;  // phase timeline (tracing builds only)
    size_t trace_n = 0;

    ~Engine();
    int create(const abmx_predation_config& c, const uint64_t* seeds, int replicas);
    int step(long long t);
    int run_async(long long t0, long long steps);  // metrics -> d_run_metrics
    int fetch_run_metrics(double* out);            // [R][last_run_steps][4]
    int last_metrics(long long* out);              // [R][4] of the last step
    int last_events(abmx_predation_events* out);
    int export_species(int r, int s, uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages,
                       int64_t* x, int64_t* y, double* energy, int32_t* num_active, int64_t* next_id);
    int import_species(int r, int s, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                       const int64_t* x, const int64_t* y, const double* energy, int32_t num_active,
                       int64_t next_id);
    int export_world(int r, uint8_t* ready, int64_t* regrow);
    int import_world(int r, const uint8_t* ready, const int64_t* regrow);
    int birth_pairs(int r, int s, int32_t* parent, int32_t* child, int32_t cap);
    // timed steps: optional L2 flush (untimed) before each step, CUDA events around each step
    // (graph) or around each kernel (per_kernel); step_ms[steps] receives device ms.
    int bench(long long t0, long long steps, size_t flush_bytes, bool per_kernel, double* step_ms);
    int finalize();  // apply the pending births of the last step

    // internals
    int alloc(void** p, size_t bytes);
    int set_t(long long t);
    int set_metrics_target(long long* d_metrics, unsigned stride);
    int prepare_run(long long t0, long long steps);
    int reserve_run(long long steps);  // allocate the run rows (before a timed region)
    int enqueue_step(cudaEvent_t* ev);
    int launch_steps(long long steps);
    int build_graph();
    unsigned grid(int k) const;
    size_t smem(int k) const;
    bool launched(int k) const;
};

}  // namespace abmx_pred
