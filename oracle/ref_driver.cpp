// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A thin extern "C" shim over the UNMODIFIED reference library (compiled from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/libabmx_ref.so).
// It lets the Python test-suite, the golden-vector generator and bench.py's
// CPU arm call the reference's own code paths through ctypes:
//   * the reference KernelTable (scalar / avx2)     include/abmx/simd/kernels.hpp:15-43
//   * RngState                                      include/abmx/rng.hpp:40-51
//   * init_predation / step_predation / metrics     include/abmx/models/predation.hpp:76-88
//   * replica_seeds / run_batch                     include/abmx/batch.hpp:48-54
//   * set_agents_rm / _sci / _mask, select, sort     include/abmx/kernels.hpp:47-106
//   * spawn_agents / remove_agents / step_agents    include/abmx/lifecycle.hpp:54-86
//   * TrafficModel / step_road / resolve_conflicts  include/abmx/models/traffic.hpp:60-110
//   * FinanceModel / match_book / run_batch          include/abmx/models/finance.hpp:21-97
// Nothing here re-implements reference behaviour; every call forwards.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <vector>

#include "abmx/batch.hpp"
#include "abmx/csv.hpp"
#include "abmx/kernels.hpp"
#include "abmx/lifecycle.hpp"
#include "abmx/models/predation.hpp"
#include "abmx/models/traffic.hpp"
#include "abmx/models/finance.hpp"
#include "abmx/rng.hpp"
#include "abmx/simd/kernels.hpp"

using namespace abmx;
using namespace abmx::models;

extern "C" {

// Same field order as abmx::models::PredationConfig (predation.hpp:13-27).
struct ref_pred_config {
    int32_t width, height, n_sheep0, n_wolves0, sheep_capacity, wolf_capacity;
    double energy_gain_sheep, energy_gain_wolf, metabolism;
    double reproduce_prob_sheep, reproduce_prob_wolf, reproduce_energy_frac;
    int64_t regrow_delay;
};

struct ref_species_events {
    int64_t metabolized, deaths, births, births_dropped;
    double energy_removed_deaths, energy_dropped_births;
};

struct ref_pred_events {
    int64_t grass_eaten, sheep_eaten_by_wolves;
    ref_species_events sheep, wolves;
};

}  // extern "C"

namespace {

PredationConfig to_cfg(const ref_pred_config* c) {
    PredationConfig p;
    p.width = c->width;
    p.height = c->height;
    p.n_sheep0 = c->n_sheep0;
    p.n_wolves0 = c->n_wolves0;
    p.sheep_capacity = c->sheep_capacity;
    p.wolf_capacity = c->wolf_capacity;
    p.energy_gain_sheep = c->energy_gain_sheep;
    p.energy_gain_wolf = c->energy_gain_wolf;
    p.metabolism = c->metabolism;
    p.reproduce_prob_sheep = c->reproduce_prob_sheep;
    p.reproduce_prob_wolf = c->reproduce_prob_wolf;
    p.reproduce_energy_frac = c->reproduce_energy_frac;
    p.regrow_delay = c->regrow_delay;
    return p;
}

struct PredHandle {
    PredationConfig cfg;
    RngState seed;
    PredationState state;
    PredationEvents events;
};

void copy_events(const PredationEvents& e, ref_pred_events* o) {
    if (!o)
        return;
    o->grass_eaten = e.grass_eaten;
    o->sheep_eaten_by_wolves = e.sheep_eaten_by_wolves;
    const SpeciesEvents* src[2] = {&e.sheep, &e.wolves};
    ref_species_events* dst[2] = {&o->sheep, &o->wolves};
    for (int k = 0; k < 2; ++k) {
        dst[k]->metabolized = src[k]->metabolized;
        dst[k]->deaths = src[k]->deaths;
        dst[k]->births = src[k]->births;
        dst[k]->births_dropped = src[k]->births_dropped;
        dst[k]->energy_removed_deaths = src[k]->energy_removed_deaths;
        dst[k]->energy_dropped_births = src[k]->energy_dropped_births;
    }
}

inline uint64_t fnv_bytes(uint64_t h, const void* p, size_t n) {
    const auto* b = static_cast<const uint8_t*>(p);
    for (size_t i = 0; i < n; ++i) {
        h ^= b[i];
        h *= 0x100000001b3ULL;
    }
    return h;
}

uint64_t hash_set(uint64_t h, const AgentSet& s) {
    h = fnv_bytes(h, s.active().data(), s.active().size());
    h = fnv_bytes(h, s.ids().data(), s.ids().size() * 8);
    h = fnv_bytes(h, s.ages().data(), s.ages().size() * 8);
    h = fnv_bytes(h, s.state().ints("x").data(), s.state().ints("x").size() * 8);
    h = fnv_bytes(h, s.state().ints("y").data(), s.state().ints("y").size() * 8);
    h = fnv_bytes(h, s.state().reals("energy").data(), s.state().reals("energy").size() * 8);
    return h;
}

AgentSet& species_of(PredHandle* h, int species) {
    return species == 0 ? h->state.sheep : h->state.wolves;
}

// generic subset-update instances use the reference test schema e:int, w:real, f:bool
// (tests/support/oracle.cpp:33-99)
AgentSet make_ewf_set(int32_t cap, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                      const int64_t* e, const double* w, const uint8_t* f) {
    const auto n = static_cast<size_t>(cap);
    FieldBundle st(n);
    st.add("e", Column::of(std::vector<int64_t>(e, e + n)));
    st.add("w", Column::of(std::vector<double>(w, w + n)));
    st.add("f", Column::of(Mask(f, f + n)));
    AgentSet set(cap, std::move(st), FieldBundle(n));
    Index na = 0;
    for (size_t i = 0; i < n; ++i) {
        set.active_mut()[i] = active[i];
        set.ids_mut()[i] = ids[i];
        set.ages_mut()[i] = ages[i];
        na += active[i] ? 1 : 0;
    }
    set.set_num_active(na);
    return set;
}

UpdateBatch make_ewf_batch(int32_t m, const int64_t* e, const double* w, const uint8_t* f,
                           const uint8_t* valid) {
    const auto n = static_cast<size_t>(m);
    FieldBundle v(n);
    v.add("e", Column::of(std::vector<int64_t>(e, e + n)));
    v.add("w", Column::of(std::vector<double>(w, w + n)));
    v.add("f", Column::of(Mask(f, f + n)));
    return UpdateBatch(std::move(v), Mask(valid, valid + n));
}

void export_ewf(const AgentSet& s, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* e,
                double* w, uint8_t* f) {
    const auto n = static_cast<size_t>(s.capacity());
    if (n == 0)
        return;
    std::memcpy(active, s.active().data(), n);
    std::memcpy(ids, s.ids().data(), n * 8);
    std::memcpy(ages, s.ages().data(), n * 8);
    std::memcpy(e, s.state().ints("e").data(), n * 8);
    std::memcpy(w, s.state().reals("w").data(), n * 8);
    std::memcpy(f, s.state().bools("f").data(), n);
}

const ApplyFn& ewf_copy() {
    static const ApplyFn fn = [](StateWriter& w, const SlotView&, const RowView& row, Index) {
        w.set_int("e", row.get_int("e"));
        w.set_real("w", row.get_real("w"));
        w.set_bool("f", row.get_bool("f"));
    };
    return fn;
}

}  // namespace

extern "C" {

// ---------------------------------------------------------------- RNG
uint64_t ref_rng_split(uint64_t key, uint64_t i) { return RngState{key}.split(i).key; }
uint64_t ref_rng_draw(uint64_t key, uint64_t c) { return RngState{key}.draw(c); }
double ref_rng_uniform_double(uint64_t key, uint64_t c) { return RngState{key}.uniform_double(c); }
int64_t ref_rng_uniform_int(uint64_t key, uint64_t c, int64_t lo, int64_t hi) {
    return RngState{key}.uniform_int(c, lo, hi);
}
int ref_rng_bernoulli(uint64_t key, uint64_t c, double p) { return RngState{key}.bernoulli(c, p); }
uint64_t ref_replica_seed(uint64_t master, int32_t r) {
    return replica_seeds(RngState{master}, r + 1)[static_cast<size_t>(r)].seed.key;
}

// ---------------------------------------------------------------- KernelTable
// backend: 0 scalar, 1 avx2 (nullptr when unavailable). The returned pointer is
// the reference's own `const KernelTable*` (a C struct of function pointers).
const void* ref_kernel_table(int backend) {
    if (backend == 0)
        return &simd::scalar_table();
    return simd::avx2_table();
}
const void* ref_active_table() { return &simd::active(); }

// ---------------------------------------------------------------- predation
void* ref_pred_create(const ref_pred_config* c, uint64_t seed) {
    try {
        const PredationConfig cfg = to_cfg(c);
        return new PredHandle{cfg, RngState{seed}, init_predation(cfg, RngState{seed}), {}};
    } catch (const std::exception&) {
        return nullptr;
    }
}

void ref_pred_free(void* p) { delete static_cast<PredHandle*>(p); }

void ref_pred_step(void* p, int64_t t, ref_pred_events* ev) {
    auto* h = static_cast<PredHandle*>(p);
    h->state = step_predation(h->state, h->cfg, h->seed, t, &h->events);
    copy_events(h->events, ev);
}

// Runs `steps` steps from t0 (no events copied). Returns wall ms.
double ref_pred_run(void* p, int64_t t0, int64_t steps) {
    auto* h = static_cast<PredHandle*>(p);
    const auto a = std::chrono::steady_clock::now();
    for (int64_t t = t0; t < t0 + steps; ++t)
        h->state = step_predation(h->state, h->cfg, h->seed, t, &h->events);
    const auto b = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::milli>(b - a).count();
}

// n_sheep, n_wolves, n_grass, births_dropped (predation.cpp:281-287)
void ref_pred_metrics(void* p, int64_t* out4) {
    auto* h = static_cast<PredHandle*>(p);
    const PredationMetrics m = metrics_predation(h->state.world, h->state.sheep, h->state.wolves);
    out4[0] = m.n_sheep;
    out4[1] = m.n_wolves;
    out4[2] = m.n_grass;
    out4[3] = h->events.sheep.births_dropped + h->events.wolves.births_dropped;
}

// FNV-1a-64 over sheep then wolves of (active, ids, ages, x, y, energy); with_world
// appends grass_ready and regrow bytes.
uint64_t ref_pred_hash(void* p, int with_world) {
    auto* h = static_cast<PredHandle*>(p);
    uint64_t x = 0xcbf29ce484222325ULL;
    x = hash_set(x, h->state.sheep);
    x = hash_set(x, h->state.wolves);
    if (with_world) {
        x = fnv_bytes(x, h->state.world.grass_ready.data(), h->state.world.grass_ready.size());
        x = fnv_bytes(x, h->state.world.regrow.data(), h->state.world.regrow.size() * 8);
    }
    return x;
}

void ref_pred_export(void* p, int species, uint8_t* active, int64_t* ids, int64_t* types,
                     int64_t* ages, int64_t* x, int64_t* y, double* energy, int32_t* num_active,
                     int64_t* next_id) {
    const AgentSet& s = species_of(static_cast<PredHandle*>(p), species);
    const auto n = static_cast<size_t>(s.capacity());
    std::memcpy(active, s.active().data(), n);
    std::memcpy(ids, s.ids().data(), n * 8);
    std::memcpy(types, s.types().data(), n * 8);
    std::memcpy(ages, s.ages().data(), n * 8);
    std::memcpy(x, s.state().ints("x").data(), n * 8);
    std::memcpy(y, s.state().ints("y").data(), n * 8);
    std::memcpy(energy, s.state().reals("energy").data(), n * 8);
    *num_active = s.num_active();
    *next_id = s.next_id();
}

void ref_pred_import(void* p, int species, const uint8_t* active, const int64_t* ids,
                     const int64_t* types, const int64_t* ages, const int64_t* x, const int64_t* y,
                     const double* energy, int32_t num_active, int64_t next_id) {
    AgentSet& s = species_of(static_cast<PredHandle*>(p), species);
    const auto n = static_cast<size_t>(s.capacity());
    std::memcpy(s.active_mut().data(), active, n);
    std::memcpy(s.ids_mut().data(), ids, n * 8);
    std::memcpy(s.types_mut().data(), types, n * 8);
    std::memcpy(s.ages_mut().data(), ages, n * 8);
    std::memcpy(s.state_mut().ints("x").data(), x, n * 8);
    std::memcpy(s.state_mut().ints("y").data(), y, n * 8);
    std::memcpy(s.state_mut().reals("energy").data(), energy, n * 8);
    s.set_num_active(num_active);
    s.set_next_id(next_id);
}

void ref_pred_export_world(void* p, uint8_t* ready, int64_t* regrow) {
    const PredationWorld& w = static_cast<PredHandle*>(p)->state.world;
    std::memcpy(ready, w.grass_ready.data(), w.cells());
    std::memcpy(regrow, w.regrow.data(), w.cells() * 8);
}

void ref_pred_import_world(void* p, const uint8_t* ready, const int64_t* regrow) {
    PredationWorld& w = static_cast<PredHandle*>(p)->state.world;
    std::memcpy(w.grass_ready.data(), ready, w.cells());
    std::memcpy(w.regrow.data(), regrow, w.cells() * 8);
}

// Birth pairs of the last step: (parent slot, child slot) per species.
int32_t ref_pred_birth_pairs(void* p, int species, int32_t* parent, int32_t* child, int32_t cap) {
    const auto& ev = static_cast<PredHandle*>(p)->events;
    const auto& v = species == 0 ? ev.sheep.birth_pairs : ev.wolves.birth_pairs;
    const auto n = static_cast<int32_t>(v.size());
    for (int32_t k = 0; k < n && k < cap; ++k) {
        parent[k] = v[static_cast<size_t>(k)].first;
        child[k] = v[static_cast<size_t>(k)].second;
    }
    return n;
}

// ---------------------------------------------------------------- batch (E4)
// metrics_out: [K][steps][4] doubles in run_batch row order. Returns wall ms
// (the reference's own steady_clock measurement, batch.cpp:96-99), or -1 on error.
double ref_run_batch(const ref_pred_config* c, uint64_t master, int32_t replicas, int64_t steps,
                     int threads, double* metrics_out) {
    try {
        const auto model = PredationModel::descriptor(to_cfg(c));
        const auto seeds = replica_seeds(RngState{master}, replicas);
        double wall = 0.0;
        const Trajectory tr = run_batch(model, seeds, steps, threads, &wall);
        if (metrics_out) {
            size_t k = 0;
            for (const auto& row : tr.rows)
                for (double v : row.values)
                    metrics_out[k++] = v;
        }
        return wall;
    } catch (const std::exception&) {
        return -1.0;
    }
}

// ---------------------------------------------------------------- subset ops
// mode 0: set_agents_rm, 1: set_agents_sci (kernels.cpp:116-153), copy-apply on e/w/f.
int ref_set_agents(int mode, int32_t cap, const uint8_t* active, const int64_t* ids,
                   const int64_t* ages, const int64_t* e, const double* w, const uint8_t* f,
                   const uint8_t* target, int32_t m, const int64_t* re, const double* rw,
                   const uint8_t* rf, const uint8_t* valid, int64_t* oe, double* ow, uint8_t* of) {
    try {
        const AgentSet set = make_ewf_set(cap, active, ids, ages, e, w, f);
        const UpdateBatch b = make_ewf_batch(m, re, rw, rf, valid);
        const std::span<const uint8_t> tm(target, static_cast<size_t>(cap));
        const AgentSet out = mode == 0 ? set_agents_rm(set, tm, b, ewf_copy())
                                       : set_agents_sci(set, tm, b, ewf_copy());
        std::vector<uint8_t> a2(cap), f2(cap);
        std::vector<int64_t> i2(cap), g2(cap);
        export_ewf(out, a2.data(), i2.data(), g2.data(), oe, ow, of);
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// select_agents with a predicate that reads a mask (kernels.cpp:30-35).
int32_t ref_select_mask(const uint8_t* mask, int32_t n, int32_t* indices) {
    const SelectionResult r = compact_mask(std::span<const uint8_t>(mask, static_cast<size_t>(n)));
    std::memcpy(indices, r.indices.data(), static_cast<size_t>(n) * 4);
    return r.count;
}

// sort_agents (kernels.cpp:52-73): writes the permuted e/w/f, ids, active.
// Returns 0, or 2 on DomainError (non-finite key on an active slot).
int ref_sort_agents(int32_t cap, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                    const int64_t* e, const double* w, const uint8_t* f, const double* key,
                    int descending, uint8_t* oa, int64_t* oi, int64_t* og, int64_t* oe, double* ow,
                    uint8_t* of) {
    try {
        const AgentSet set = make_ewf_set(cap, active, ids, ages, e, w, f);
        const AgentSet out =
            sort_agents(set, std::span<const double>(key, static_cast<size_t>(cap)),
                        descending ? SortDirection::Descending : SortDirection::Ascending);
        export_ewf(out, oa, oi, og, oe, ow, of);
        return 0;
    } catch (const DomainError&) {
        return 2;
    } catch (const std::exception&) {
        return 1;
    }
}

// spawn_agents (lifecycle.cpp:144-195) with copy-apply; returns spawned, writes dropped.
int32_t ref_spawn_agents(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* e,
                         double* w, uint8_t* f, int64_t* next_id, int32_t m, const int64_t* re,
                         const double* rw, const uint8_t* rf, const uint8_t* valid,
                         int32_t* dropped) {
    AgentSet set = make_ewf_set(cap, active, ids, ages, e, w, f);
    set.set_next_id(*next_id);
    const UpdateBatch b = make_ewf_batch(m, re, rw, rf, valid);
    SpawnOutcome o = spawn_agents(set, b, ewf_copy());
    export_ewf(o.set, active, ids, ages, e, w, f);
    *next_id = o.set.next_id();
    *dropped = o.dropped;
    return o.spawned;
}

// remove_agents (lifecycle.cpp:124-142); returns new num_active.
int32_t ref_remove_agents(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* e,
                          double* w, uint8_t* f, const uint8_t* kill) {
    AgentSet set = make_ewf_set(cap, active, ids, ages, e, w, f);
    AgentSet out = remove_agents(set, std::span<const uint8_t>(kill, static_cast<size_t>(cap)));
    export_ewf(out, active, ids, ages, e, w, f);
    return out.num_active();
}

// One lifecycle cycle on the reference (lifecycle.cpp:124-195): remove_agents(kill) then
// spawn_agents(rows, copy apply), with optional id recycling. The retired-id stack is passed
// in and out so cycles chain. Returns spawned; writes dropped, slots, rows, num_active.
int32_t ref_lifecycle(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* types,
                      int64_t* e, double* w, uint8_t* f, int64_t* next_id, int recycle,
                      int64_t* retired, int32_t* n_retired, const uint8_t* kill, int32_t m,
                      const int64_t* re, const double* rw, const uint8_t* rf, const uint8_t* valid,
                      int set_type, int64_t agent_type, int32_t* slots, int32_t* rows,
                      int32_t* dropped, int32_t* num_active) {
    AgentSet set = make_ewf_set(cap, active, ids, ages, e, w, f);
    for (int32_t i = 0; i < cap; ++i) set.types_mut()[static_cast<size_t>(i)] = types[i];
    set.set_next_id(*next_id);
    set.set_id_recycling(recycle != 0);
    set.retired_ids().assign(retired, retired + *n_retired);
    AgentSet mid = remove_agents(set, std::span<const uint8_t>(kill, static_cast<size_t>(cap)));
    const UpdateBatch b = make_ewf_batch(m, re, rw, rf, valid);
    SpawnOutcome o = set_type ? spawn_agents(mid, b, ewf_copy(), agent_type)
                              : spawn_agents(mid, b, ewf_copy());
    export_ewf(o.set, active, ids, ages, e, w, f);
    for (int32_t i = 0; i < cap; ++i) types[i] = o.set.types()[static_cast<size_t>(i)];
    *next_id = o.set.next_id();
    *n_retired = static_cast<int32_t>(o.set.retired_ids().size());
    std::copy(o.set.retired_ids().begin(), o.set.retired_ids().end(), retired);
    for (size_t k = 0; k < o.slots.size(); ++k) {
        slots[k] = static_cast<int32_t>(o.slots[k]);
        rows[k] = static_cast<int32_t>(o.rows[k]);
    }
    *dropped = static_cast<int32_t>(o.dropped);
    *num_active = static_cast<int32_t>(o.set.num_active());
    return static_cast<int32_t>(o.spawned);
}

// Timed lifecycle cycles on the reference (bench.py's agents section): the set is built once,
// the K spawn batches up front; then K x (remove_agents(kill_k), spawn_agents(batch_k, copy
// apply)) chained by value as the reference's callers do. Returns wall ms per cycle; the final
// set is exported in place.
double ref_lifecycle_bench(int32_t cap, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* e,
                           double* w, uint8_t* f, int64_t next_id, int32_t K, const uint8_t* kills,
                           const int64_t* re, const double* rw, const uint8_t* rf, const uint8_t* valids) {
    try {
        AgentSet set = make_ewf_set(cap, active, ids, ages, e, w, f);
        set.set_next_id(next_id);
        std::vector<UpdateBatch> batches;
        batches.reserve(static_cast<size_t>(K));
        for (int32_t k = 0; k < K; ++k)
            batches.push_back(make_ewf_batch(cap, re, rw, rf, valids + static_cast<size_t>(k) * cap));
        const auto a = std::chrono::steady_clock::now();
        for (int32_t k = 0; k < K; ++k) {
            AgentSet mid = remove_agents(set, std::span<const uint8_t>(kills + static_cast<size_t>(k) * cap,
                                                                       static_cast<size_t>(cap)));
            SpawnOutcome o = spawn_agents(mid, batches[static_cast<size_t>(k)], ewf_copy());
            set = std::move(o.set);
        }
        const auto b = std::chrono::steady_clock::now();
        export_ewf(set, active, ids, ages, e, w, f);
        return std::chrono::duration<double, std::milli>(b - a).count() / (K > 0 ? K : 1);
    } catch (const std::exception&) {
        return -1.0;
    }
}

// ---------------------------------------------------------------- traffic (traffic.hpp)
// A road is passed as flat arrays over capacity 3*length: active, ids, ages, lane, cell,
// plus num_active / next_id; occupancy [3*length] is written on export.
namespace {
Road road_from(int64_t length, const uint8_t* active, const int64_t* ids, const int64_t* ages,
               const int64_t* lane, const int64_t* cell, int64_t next_id) {
    Road road = Road::empty(length);
    const auto n = static_cast<size_t>(road.cars.capacity());
    Index na = 0;
    for (size_t i = 0; i < n; ++i) {
        road.cars.active_mut()[i] = active[i];
        road.cars.ids_mut()[i] = ids[i];
        road.cars.ages_mut()[i] = ages[i];
        road.cars.state_mut().ints("lane")[i] = lane[i];
        road.cars.state_mut().ints("cell")[i] = cell[i];
        na += active[i] ? 1 : 0;
    }
    road.cars.set_num_active(na);
    road.cars.set_next_id(next_id);
    road.rebuild_occupancy();
    return road;
}
void road_to(const Road& road, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* lane,
             int64_t* cell, int32_t* occupancy, int64_t* next_id) {
    const auto n = static_cast<size_t>(road.cars.capacity());
    for (size_t i = 0; i < n; ++i) {
        active[i] = road.cars.active()[i];
        ids[i] = road.cars.ids()[i];
        ages[i] = road.cars.ages()[i];
        lane[i] = road.cars.state().ints("lane")[i];
        cell[i] = road.cars.state().ints("cell")[i];
        if (occupancy) occupancy[i] = road.occupancy[i];
    }
    *next_id = road.cars.next_id();
}
}  // namespace

void* ref_traffic_create(int64_t length, int64_t period, double green_fraction, uint64_t seed) {
    try {
        TrafficConfig cfg{static_cast<abmx::Index>(length), period, green_fraction};
        return new TrafficModel(cfg, RngState{seed});
    } catch (const std::exception&) {
        return nullptr;
    }
}
void ref_traffic_free(void* h) { delete static_cast<TrafficModel*>(h); }
void ref_traffic_step(void* h, int64_t t) { static_cast<TrafficModel*>(h)->step(t); }
void ref_traffic_metrics(void* h, double* out4) {
    std::vector<std::vector<double>> rows;
    static_cast<TrafficModel*>(h)->collect_metrics(rows);
    for (int k = 0; k < 4; ++k) out4[k] = rows[0][static_cast<size_t>(k)];
}
int64_t ref_traffic_phase(void* h) { return static_cast<TrafficModel*>(h)->schedule().phase; }
int64_t ref_traffic_green_len(void* h) { return static_cast<TrafficModel*>(h)->schedule().green_len; }
void ref_traffic_export(void* h, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* lane,
                        int64_t* cell, int32_t* occupancy, int64_t* next_id, int32_t* num_active) {
    const Road& road = static_cast<TrafficModel*>(h)->road();
    road_to(road, active, ids, ages, lane, cell, occupancy, next_id);
    *num_active = static_cast<int32_t>(road.cars.num_active());
}
// double wall ms of the steps t0..t0+steps-1
double ref_traffic_run(void* h, int64_t t0, int64_t steps) {
    auto* m = static_cast<TrafficModel*>(h);
    const auto a = std::chrono::steady_clock::now();
    for (int64_t t = t0; t < t0 + steps; ++t) m->step(t);
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}

// step_road on an arbitrary road (traffic.cpp:186-222): state in/out; stats out {spawned,
// exited, green}. Returns 0, or 1 on DomainError (two cars in one cell).
int ref_traffic_step_road(int64_t length, int64_t period, double green_fraction, uint64_t seed,
                          int64_t t, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* lane,
                          int64_t* cell, int32_t* occupancy, int64_t* next_id, int64_t* stats3) {
    try {
        const TrafficConfig cfg{static_cast<abmx::Index>(length), period, green_fraction};
        const SignalSchedule sched = SignalSchedule::from_config(cfg, RngState{seed});
        Road road = road_from(length, active, ids, ages, lane, cell, *next_id);
        RoadStepStats st;
        Road out = step_road(road, sched, RngState{seed}, t, &st);
        road_to(out, active, ids, ages, lane, cell, occupancy, next_id);
        stats3[0] = st.spawned;
        stats3[1] = st.exited;
        stats3[2] = st.signal_green ? 1 : 0;
        return 0;
    } catch (const std::exception&) {
        return 1;
    }
}

// resolve_conflicts with given proposals (kind 0 stay / 1 move / 2 exit). Returns 0, 1 on
// DomainError (bad road), 2 on ContractError (target outside the road).
int ref_traffic_resolve(int64_t length, const uint8_t* active, const int64_t* lane,
                        const int64_t* cell, const uint8_t* kind, const int64_t* to_lane,
                        const int64_t* to_cell, uint8_t* accepted) {
    const auto n = static_cast<size_t>(3 * length);
    std::vector<int64_t> z(n, 0);
    std::unique_ptr<Road> rp;
    try {
        rp = std::make_unique<Road>(road_from(length, active, z.data(), z.data(), lane, cell, 0));
    } catch (const std::exception&) {
        return 1;
    }
    const Road& road = *rp;
    Proposals p;
    p.kind.resize(n);
    p.to_lane.assign(to_lane, to_lane + n);
    p.to_cell.assign(to_cell, to_cell + n);
    for (size_t i = 0; i < n; ++i) p.kind[i] = static_cast<MoveKind>(kind[i]);
    try {
        const Mask acc = resolve_conflicts(road, p);
        std::memcpy(accepted, acc.data(), n);
        return 0;
    } catch (const ContractError&) {
        return 2;
    } catch (const std::exception&) {
        return 1;
    }
}

double ref_traffic_run_batch(int64_t length, int64_t period, double green_fraction,
                             uint64_t master, int32_t replicas, int64_t steps, int threads,
                             double* metrics_out) {
    try {
        const auto model = TrafficModel::descriptor(TrafficConfig{static_cast<abmx::Index>(length), period, green_fraction});
        const auto seeds = replica_seeds(RngState{master}, replicas);
        double wall = 0.0;
        const Trajectory tr = run_batch(model, seeds, steps, threads, &wall);
        if (metrics_out) {
            size_t k = 0;
            for (const auto& row : tr.rows)
                for (double v : row.values) metrics_out[k++] = v;
        }
        return wall;
    } catch (const std::exception&) {
        return -1.0;
    }
}


// ---------------------------------------------------------------- finance (finance.hpp)
struct ref_fin_config {
    int64_t books, traders, book_capacity;
    double p_order, delta;
    int64_t qmax, max_order_age;
    double init_price;
};
namespace {
FinanceConfig fin_cfg(const ref_fin_config* c) {
    FinanceConfig f;
    f.books = c->books;
    f.traders = c->traders;
    f.book_capacity = c->book_capacity;
    f.p_order = c->p_order;
    f.delta = c->delta;
    f.qmax = c->qmax;
    f.max_order_age = c->max_order_age;
    f.init_price = c->init_price;
    return f;
}
void book_to(const Book& b, uint8_t* active, int64_t* ids, int64_t* trader, int64_t* side, double* price,
             int64_t* qty, int64_t* placed, double* scalars /* last_price, dropped, volume, clearing, next_id, num_active */) {
    const auto n = static_cast<size_t>(b.orders.capacity());
    for (size_t i = 0; i < n; ++i) {
        active[i] = b.orders.active()[i];
        ids[i] = b.orders.ids()[i];
        trader[i] = b.orders.state().ints("trader")[i];
        side[i] = b.orders.state().ints("side")[i];
        price[i] = b.orders.state().reals("price")[i];
        qty[i] = b.orders.state().ints("qty")[i];
        placed[i] = b.orders.state().ints("placed")[i];
    }
    scalars[0] = b.last_price;
    scalars[1] = static_cast<double>(b.dropped_this_step);
    scalars[2] = static_cast<double>(b.last_trades.volume);
    scalars[3] = b.last_trades.clearing_price;
    scalars[4] = static_cast<double>(b.orders.next_id());
    scalars[5] = static_cast<double>(b.orders.num_active());
}
}  // namespace

void* ref_fin_create(const ref_fin_config* c, uint64_t seed) {
    try {
        return new FinanceModel(fin_cfg(c), RngState{seed});
    } catch (const std::exception&) {
        return nullptr;
    }
}
void ref_fin_free(void* h) { delete static_cast<FinanceModel*>(h); }
void ref_fin_step(void* h, int64_t t) { static_cast<FinanceModel*>(h)->step(t); }
double ref_fin_run(void* h, int64_t t0, int64_t steps) {
    auto* m = static_cast<FinanceModel*>(h);
    const auto a = std::chrono::steady_clock::now();
    for (int64_t t = t0; t < t0 + steps; ++t) m->step(t);
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - a).count();
}
void ref_fin_metrics(void* h, double* rows) {
    std::vector<std::vector<double>> out;
    static_cast<FinanceModel*>(h)->collect_metrics(out);
    size_t k = 0;
    for (const auto& row : out)
        for (double v : row) rows[k++] = v;
}
void ref_fin_export_book(void* h, int32_t book, uint8_t* active, int64_t* ids, int64_t* trader, int64_t* side,
                         double* price, int64_t* qty, int64_t* placed, double* scalars) {
    book_to(static_cast<FinanceModel*>(h)->market().books[static_cast<size_t>(book)], active, ids, trader, side,
            price, qty, placed, scalars);
}
void ref_fin_export_traders(void* h, double* cash, int64_t* holdings /* [books][traders] */) {
    const MarketState& s = static_cast<FinanceModel*>(h)->market();
    const auto n = static_cast<size_t>(s.traders.capacity());
    for (size_t i = 0; i < n; ++i) cash[i] = s.traders.state().reals("cash")[i];
    for (size_t k = 0; k < s.books.size(); ++k)
        for (size_t i = 0; i < n; ++i) holdings[k * n + i] = s.traders.state().ints("holdings_" + std::to_string(k))[i];
}
// match_book on a book given as arrays (capacity cap, last price); book arrays are updated,
// fills written (trader, side, qty, amount); returns the number of fills, -1 on error.
int32_t ref_fin_match(int32_t cap, double last_price, uint8_t* active, int64_t* ids, int64_t* trader, int64_t* side,
                      double* price, int64_t* qty, int64_t* placed, int64_t next_id, int64_t* f_trader,
                      int64_t* f_side, int64_t* f_qty, double* f_amount, double* scalars) {
    try {
        Book b = Book::empty(cap, 0, last_price);
        Index na = 0;
        for (int32_t i = 0; i < cap; ++i) {
            const auto u = static_cast<size_t>(i);
            b.orders.active_mut()[u] = active[i];
            b.orders.ids_mut()[u] = ids[i];
            b.orders.state_mut().ints("trader")[u] = trader[i];
            b.orders.state_mut().ints("side")[u] = side[i];
            b.orders.state_mut().reals("price")[u] = price[i];
            b.orders.state_mut().ints("qty")[u] = qty[i];
            b.orders.state_mut().ints("placed")[u] = placed[i];
            na += active[i] ? 1 : 0;
        }
        b.orders.set_num_active(na);
        b.orders.set_next_id(next_id);
        b.last_price = last_price;
        auto [out, summary] = match_book(b);
        book_to(out, active, ids, trader, side, price, qty, placed, scalars);
        for (size_t k = 0; k < summary.fills.size(); ++k) {
            f_trader[k] = summary.fills[k].trader;
            f_side[k] = summary.fills[k].side;
            f_qty[k] = summary.fills[k].qty;
            f_amount[k] = summary.fills[k].amount;
        }
        return static_cast<int32_t>(summary.fills.size());
    } catch (const std::exception&) {
        return -1;
    }
}
double ref_fin_quantize(double raw) { return quantize_price(raw); }
double ref_fin_run_batch(const ref_fin_config* c, uint64_t master, int32_t replicas, int64_t steps, int threads,
                         double* rows) {
    try {
        const auto model = FinanceModel::descriptor(fin_cfg(c));
        const auto seeds = replica_seeds(RngState{master}, replicas);
        double wall = 0.0;
        const Trajectory tr = run_batch(model, seeds, steps, threads, &wall);
        if (rows) {
            size_t k = 0;
            for (const auto& row : tr.rows)
                for (double v : row.values) rows[k++] = v;
        }
        return wall;
    } catch (const std::exception&) {
        return -1.0;
    }
}


// ---------------------------------------------------------------- CSV (csv.cpp)
// trajectory_to_csv of run_batch for one of the three batch models; returns the text length
// (the text is written only if it fits `cap`), -1 on error. kind 0 predation, 1 traffic,
// 2 finance; the matching config pointer is used.
int64_t ref_run_csv(int kind, const ref_pred_config* pc, int64_t length, int64_t period, double green_fraction,
                    const ref_fin_config* fc, uint64_t master, int32_t replicas, int64_t steps, char* out,
                    int64_t cap) {
    try {
        ModelDescriptor model = kind == 0   ? PredationModel::descriptor(to_cfg(pc))
                                : kind == 1 ? TrafficModel::descriptor(TrafficConfig{static_cast<abmx::Index>(length), period, green_fraction})
                                            : FinanceModel::descriptor(fin_cfg(fc));
        const auto seeds = replica_seeds(RngState{master}, replicas);
        const Trajectory tr = run_batch(model, seeds, steps, 1, nullptr);
        const std::string csv = trajectory_to_csv(tr);
        if (static_cast<int64_t>(csv.size()) <= cap) std::memcpy(out, csv.data(), csv.size());
        return static_cast<int64_t>(csv.size());
    } catch (const std::exception&) {
        return -1;
    }
}
void ref_format_real(double v, char* out) {
    const std::string s = format_real(v);
    std::memcpy(out, s.c_str(), s.size() + 1);
}

}  // extern "C"
