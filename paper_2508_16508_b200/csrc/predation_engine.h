// predation_engine.h — device data layout and the host-side engine object for the
// predation step (internal; the public surface is include/abmx_cuda.h).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/abmx_cuda.h"

namespace abmx_pred {

constexpr int kT = 256;          // threads per slot-tile CTA
constexpr int kS = 4;            // slots per thread in the scanning kernel (k_update)
constexpr int kTile = kT * kS;   // slots per lookback tile
constexpr int kM = 4;            // slots per thread in k_move / k_cells
constexpr int kMTile = kT * kM;
constexpr int kNumKernels = 4;
constexpr int kEpochClear = 128;  // cell tags are cleared every kEpochClear steps (epoch8 period 255)

// Device control block: step bookkeeping shared by the four kernels of a step.
struct Ctl {
    unsigned pad0;
    unsigned pool_top;   // bump allocator of the long-list sort pool
    unsigned error;      // set if the sort pool overflowed (cannot happen: sized N_s + N_w)
    unsigned occ[2];     // entries in the occupied-cell lists (sheep, wolves) this step
};

// Per (replica, species) persistent counters + this step's spawn plan.
// Counters are double-buffered by step parity p = epoch & 1: k_spawn of a step reads
// next_id[p] and writes next_id[p ^ 1] / num_active[p ^ 1] for the next step.
struct SpeciesRep {
    long long next_id[2];
    int num_active[2];
    long long base_id;  // first fresh id of the last step's births
    int pairs;          // min(free, valid) of the last step
    int Q;              // valid rows of the last step
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
    unsigned long long epoch;  // internal step counter (>= 1) stamping the per-cell lists
    long long t;               // the reference's step index t fed to the RNG streams
    long long* metrics;        // [R][metrics_stride][4]
    unsigned run_step, metrics_stride, needs_blend, pad0;
    // model constants
    int R, W, H, Cpad;
    long long C;
    int N[2], Npad[2], tiles[2], mtiles[2];
    double gain[2], metab, prob[2], frac;
    int delay;     // regrow_delay if >= 1, else 0 (a grazed cell never regrows)
    int due_ring;  // due-epoch histogram ring length per replica (power of two > delay)
    int spawn_cps, spawn_ctas, k2_ctas, status_stride;
    const unsigned long long* seeds;
    uint8_t* active[2];
    int* cell[2];
    int* age[2];
    double* energy[2];
    long long* id[2];
    int* next[2];
    uint8_t* flag[2];   // sheep: eaten this step; wolves: ate this step
    int* free_at[2];
    int* row_at[2];
    int* rowcell[2];
    double* rowE[2];
    uint4* cw;             // per cell: sheep head, wolf head, lowest sheep slot, grass due epoch
    long long* n_grass;    // [R] ready cells after the last step
    unsigned* due_count;   // [R][due_ring] cells coming due at each epoch (mod ring)
    unsigned long long* status;  // [species][R][status_stride] packed (free, valid) per k_update tile
    unsigned long long* occ[2];  // occupied cells per species: (replica << 32) | cell
    int* pool;
    long long pool_size;
    Ctl* ctl;
    unsigned long long* phase_ns;  // optional: k_step accumulates per-phase ns (globaltimer)
    SpeciesRep* rep;
    Events* ev;
};

const char* kernel_name(int k);

struct Engine {
    abmx_predation_config cfg{};
    int R = 0;
    Params params{};
    cudaStream_t stream = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t graph_exec = nullptr;
    cudaGraphNode_t nodes[kNumKernels] = {};
    std::vector<void*> allocs;
    long long device_bytes = 0;
    unsigned long long* d_seeds = nullptr;
    long long* d_metrics_step = nullptr;   // [R][1][4]
    long long* d_run_metrics = nullptr;    // [R][steps][4]
    size_t run_metrics_bytes = 0;
    long long last_run_steps = 0;
    unsigned long long host_epoch = 1;     // epoch of the next step
    bool timing = false;
    bool fused = false;  // true: one cooperative k_step launch per step; false: the 4-kernel graph
    int coop_grid = 0;
    cudaEvent_t tev[2 * kNumKernels] = {};
    double kernel_ms[kNumKernels] = {};
    long long kernel_launches[kNumKernels] = {};
    size_t spawn_smem = 0;
    void* flush_buf = nullptr;
    size_t flush_cap = 0;

    ~Engine();
    int create(const abmx_predation_config& c, const uint64_t* seeds, int replicas);
    int step(long long t);
    int run_async(long long t0, long long steps);           // metrics -> d_run_metrics
    int fetch_run_metrics(double* out);                     // [R][last_run_steps][4]
    int last_metrics(long long* out);                       // [R][4] of the last step
    int last_events(abmx_predation_events* out);
    int export_species(int r, int s, uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages,
                       int64_t* x, int64_t* y, double* energy, int32_t* num_active, int64_t* next_id);
    int import_species(int r, int s, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                       const int64_t* x, const int64_t* y, const double* energy, int32_t num_active,
                       int64_t next_id);
    int export_world(int r, uint8_t* ready, int64_t* regrow);
    int import_world(int r, const uint8_t* ready, const int64_t* regrow);
    int birth_pairs(int r, int s, int32_t* parent, int32_t* child, int32_t cap);
    // timed steps: optional L2 flush (untimed) before each step, CUDA events around each
    // step (graph) or around each kernel (per_kernel); step_ms[steps] receives device ms.
    int bench(long long t0, long long steps, size_t flush_bytes, bool per_kernel, double* step_ms);

    // internals
    int alloc(void** p, size_t bytes);
    int set_t(long long t);
    int set_metrics_target(long long* d_metrics, unsigned stride);
    void launch_step_kernels(bool timed);
    unsigned grid(int k) const;
    int build_graph();
    int launch_steps(long long steps);
    int accumulate_times();
};

}  // namespace abmx_pred
