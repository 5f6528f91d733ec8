// abmx_cuda.hpp — header-only C++ host mirror of the reference interface over the C-ABI
// in abmx_cuda.h. A reference user keeps the reference's names and argument meaning:
//
//   abmx::models::PredationModel (include/abmx/models/predation.hpp:91-107)
//       -> abmx::cuda::PredationModel   step(t), collect_metrics(rows), last_events()
//   abmx::run_batch / replica_seeds (include/abmx/batch.hpp:48-54)
//       -> abmx::cuda::run_batch / replica_seeds
//   abmx::simd::KernelTable (include/abmx/simd/kernels.hpp:15-43)
//       -> abmx::cuda::kernel_table()  (same layout)
//   abmx::models::TrafficModel / FinanceModel (traffic.hpp:84-110, finance.hpp:80-97)
//       -> abmx::cuda::TrafficModel / FinanceModel, traffic_run_batch / finance_run_batch,
//          resolve_conflicts, match_book, quantize_price
//   AgentSet + remove/spawn/set_agents/select/sort/permute (agent_set.hpp, lifecycle.hpp,
//   kernels.hpp) -> abmx::cuda::DeviceAgentSet (columns resident in device memory)
//
// Errors are thrown as the reference's exception types (errors.hpp:8-40), re-declared here
// under abmx::cuda so this header does not need the reference tree.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "abmx_cuda.h"

namespace abmx::cuda {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct SchemaError : Error {
    using Error::Error;
};
struct CapacityError : Error {
    using Error::Error;
};
struct DomainError : Error {
    using Error::Error;
};
struct BatchError : Error {
    using Error::Error;
};
struct ContractError : Error {
    using Error::Error;
};
struct DeviceError : Error {
    using Error::Error;
};

inline void check(int rc) {
    if (rc == ABMX_OK) return;
    const std::string msg = abmx_cuda_last_error();
    switch (rc) {
        case ABMX_E_DOMAIN: throw DomainError(msg);
        case ABMX_E_CAPACITY: throw CapacityError(msg);
        case ABMX_E_SCHEMA: throw SchemaError(msg);
        case ABMX_E_BATCH: throw BatchError(msg);
        case ABMX_E_CUDA: throw DeviceError(msg);
        case ABMX_E_CONTRACT: throw ContractError(msg);
        default: throw Error(msg);
    }
}

inline const abmx_kernel_table& kernel_table() { return *abmx_cuda_kernel_table(); }

// RngState::split (src/rng.cpp:18-20), for seed plumbing on the host.
inline std::uint64_t split(std::uint64_t key, std::uint64_t i) {
    std::uint64_t z = key + 0xC2B2AE3D27D4EB4FULL * (i + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// replica_seeds (batch.cpp:12-19): master.split(BatchReplica = 2).split(r)
inline std::vector<std::uint64_t> replica_seeds(std::uint64_t master, std::int32_t count) {
    std::vector<std::uint64_t> out;
    out.reserve(static_cast<std::size_t>(count > 0 ? count : 0));
    const std::uint64_t root = split(master, 2);
    for (std::int32_t r = 0; r < count; ++r) out.push_back(split(root, static_cast<std::uint64_t>(r)));
    return out;
}

// Reference defaults of PredationConfig (predation.hpp:13-27).
inline abmx_predation_config default_predation_config() {
    abmx_predation_config c{};
    c.width = 100;
    c.height = 100;
    c.n_sheep0 = 600;
    c.n_wolves0 = 400;
    c.sheep_capacity = 20000;
    c.wolf_capacity = 20000;
    c.energy_gain_sheep = 4.0;
    c.energy_gain_wolf = 20.0;
    c.metabolism = 1.0;
    c.reproduce_prob_sheep = 0.04;
    c.reproduce_prob_wolf = 0.05;
    c.reproduce_energy_frac = 0.5;
    c.regrow_delay = 30;
    return c;
}

// The device-resident drop-in for abmx::models::PredationModel (one replica).
class PredationModel {
public:
    PredationModel(const abmx_predation_config& cfg, std::uint64_t seed) {
        check(abmx_predation_create(&cfg, &seed, 1, &h_));
    }
    ~PredationModel() { abmx_predation_destroy(h_); }
    PredationModel(const PredationModel&) = delete;
    PredationModel& operator=(const PredationModel&) = delete;

    // Model::step (batch.hpp:18)
    void step(std::int64_t t) { check(abmx_predation_step(h_, t)); }

    // Model::collect_metrics: n_sheep, n_wolves, n_grass, births_dropped (predation.cpp:281-287)
    void collect_metrics(std::vector<std::vector<double>>& rows) const {
        std::int64_t m[4];
        check(abmx_predation_metrics(h_, m));
        rows.push_back({static_cast<double>(m[0]), static_cast<double>(m[1]), static_cast<double>(m[2]),
                        static_cast<double>(m[3])});
    }

    abmx_predation_events last_events() const {
        abmx_predation_events e{};
        check(abmx_predation_last_events(h_, &e));
        return e;
    }

    abmx_predation* handle() const { return h_; }

private:
    abmx_predation* h_ = nullptr;
};

// run_batch (batch.cpp:21-101) for PredationModel replicas: rows [replicas][steps][4] in
// (replica, step) order, t = 1..steps.
inline std::vector<double> run_batch(const abmx_predation_config& cfg, std::uint64_t master,
                                     std::int32_t replicas, std::int64_t steps, std::int32_t first = 0) {
    std::vector<double> rows(static_cast<std::size_t>(replicas > 0 ? replicas : 0) *
                             static_cast<std::size_t>(steps > 0 ? steps : 0) * 4);
    check(abmx_ensemble_run(&cfg, master, first, replicas, steps, 0, rows.data(), nullptr));
    return rows;
}

// ------------------------------------------------------------------------------ traffic
// TrafficConfig defaults (traffic.hpp:13-17)
inline abmx_traffic_config default_traffic_config() { return abmx_traffic_config{100, 10, 0.5}; }

// The device-resident drop-in for abmx::models::TrafficModel (one road).
class TrafficModel {
public:
    TrafficModel(const abmx_traffic_config& cfg, std::uint64_t seed) : cap_(3 * cfg.length) {
        check(abmx_traffic_create(&cfg, &seed, 1, &h_));
    }
    ~TrafficModel() { abmx_traffic_destroy(h_); }
    TrafficModel(const TrafficModel&) = delete;
    TrafficModel& operator=(const TrafficModel&) = delete;

    void step(std::int64_t t) { check(abmx_traffic_step(h_, t)); }
    // n_cars, spawned, exited, signal_green (traffic.cpp:234-238)
    void collect_metrics(std::vector<std::vector<double>>& rows) const {
        std::vector<double> m(4);
        check(abmx_traffic_metrics(h_, m.data()));
        rows.push_back(m);
    }
    std::int64_t spawned_total() const {
        std::int64_t s = 0, e = 0;
        check(abmx_traffic_totals(h_, 0, &s, &e));
        return s;
    }
    std::int64_t exited_total() const {
        std::int64_t s = 0, e = 0;
        check(abmx_traffic_totals(h_, 0, &s, &e));
        return e;
    }
    // occupancy in the reference layout (lane * length + cell -> slot or -1)
    std::vector<std::int32_t> occupancy() const {
        std::vector<std::uint8_t> act(cap_);
        std::vector<std::int64_t> ids(cap_), ages(cap_), lane(cap_), cell(cap_), nid(1);
        std::vector<std::int32_t> occ(cap_);
        std::int32_t na = 0;
        check(abmx_traffic_export(h_, 0, act.data(), ids.data(), ages.data(), lane.data(), cell.data(),
                                  occ.data(), nid.data(), &na));
        return occ;
    }
    abmx_traffic* handle() const { return h_; }

private:
    abmx_traffic* h_ = nullptr;
    std::size_t cap_;
};

// run_batch of TrafficModel: rows [replicas][steps][4]
inline std::vector<double> traffic_run_batch(const abmx_traffic_config& cfg, std::uint64_t master,
                                             std::int32_t replicas, std::int64_t steps, std::int32_t first = 0) {
    std::vector<double> rows(static_cast<std::size_t>(replicas > 0 ? replicas : 0) *
                             static_cast<std::size_t>(steps > 0 ? steps : 0) * 4);
    check(abmx_traffic_run_batch(&cfg, master, first, replicas, steps, rows.data(), nullptr));
    return rows;
}

// resolve_conflicts (traffic.cpp:82-140) with explicit proposals (kind 0 stay, 1 move, 2 exit)
inline std::vector<std::uint8_t> resolve_conflicts(std::int64_t length, const std::vector<std::uint8_t>& active,
                                                   const std::vector<std::int64_t>& lane,
                                                   const std::vector<std::int64_t>& cell,
                                                   const std::vector<std::uint8_t>& kind,
                                                   const std::vector<std::int64_t>& to_lane,
                                                   const std::vector<std::int64_t>& to_cell) {
    std::vector<std::uint8_t> acc(static_cast<std::size_t>(3 * length));
    check(abmx_traffic_resolve(length, active.data(), lane.data(), cell.data(), kind.data(), to_lane.data(),
                               to_cell.data(), acc.data()));
    return acc;
}

// ------------------------------------------------------------------------------ finance
// FinanceConfig defaults (finance.hpp:13-22)
inline abmx_finance_config default_finance_config() {
    return abmx_finance_config{5, 10, 1000, 0.5, 0.05, 10, 20, 100.0};
}

inline double quantize_price(double raw) { return abmx_finance_quantize_price(raw); }

// The device-resident drop-in for abmx::models::FinanceModel (one market).
class FinanceModel {
public:
    FinanceModel(const abmx_finance_config& cfg, std::uint64_t seed) : books_(cfg.books) {
        check(abmx_finance_create(&cfg, &seed, 1, &h_));
    }
    ~FinanceModel() { abmx_finance_destroy(h_); }
    FinanceModel(const FinanceModel&) = delete;
    FinanceModel& operator=(const FinanceModel&) = delete;

    void step(std::int64_t t) { check(abmx_finance_step(h_, t)); }
    // one row per book: book_id, price, n_active_buys, n_active_sells, volume, orders_dropped
    void collect_metrics(std::vector<std::vector<double>>& rows) const {
        std::vector<double> m(static_cast<std::size_t>(books_) * 6);
        check(abmx_finance_metrics(h_, m.data()));
        for (std::int64_t k = 0; k < books_; ++k)
            rows.emplace_back(m.begin() + k * 6, m.begin() + (k + 1) * 6);
    }
    abmx_finance* handle() const { return h_; }

private:
    abmx_finance* h_ = nullptr;
    std::int64_t books_;
};

// run_batch of FinanceModel: rows [replicas][steps][books][6]
inline std::vector<double> finance_run_batch(const abmx_finance_config& cfg, std::uint64_t master,
                                             std::int32_t replicas, std::int64_t steps, std::int32_t first = 0) {
    std::vector<double> rows(static_cast<std::size_t>(replicas > 0 ? replicas : 0) *
                             static_cast<std::size_t>(steps > 0 ? steps : 0) * static_cast<std::size_t>(cfg.books) * 6);
    check(abmx_finance_run_batch(&cfg, master, first, replicas, steps, rows.data(), nullptr));
    return rows;
}

// ------------------------------------------------------------------------------ agent sets
// A thin RAII view over abmx_agent_set: the caller owns the device columns (any allocator);
// the operations mirror lifecycle.hpp / kernels.hpp with the column-copy apply.
class DeviceAgentSet {
public:
    explicit DeviceAgentSet(const abmx_agent_set& s, void* stream = nullptr) : s_(s), stream_(stream) {}
    void remove(const std::uint8_t* d_kill, std::int64_t* d_killed = nullptr) {
        check(abmx_agents_remove(&s_, d_kill, d_killed, stream_));
    }
    void spawn(std::int32_t m, const std::uint8_t* d_valid, const abmx_column* rows, bool set_type = false,
               std::int64_t agent_type = 0, std::int32_t* d_slots = nullptr, std::int32_t* d_rows = nullptr,
               std::int64_t* d_result = nullptr) {
        check(abmx_agents_spawn(&s_, m, d_valid, rows, set_type ? 1 : 0, agent_type, d_slots, d_rows, d_result,
                                stream_));
    }
    void set_rm(const std::uint8_t* d_target, std::int32_t m, const std::uint8_t* d_valid, const abmx_column* rows) {
        check(abmx_agents_set_rm(&s_, d_target, m, d_valid, rows, nullptr, nullptr, nullptr, stream_));
    }
    void set_sci(const std::uint8_t* d_target, std::int32_t m, const std::uint8_t* d_valid, const abmx_column* rows) {
        check(abmx_agents_set_sci(&s_, d_target, m, d_valid, rows, nullptr, nullptr, nullptr, stream_));
    }
    void set_mask(const std::uint8_t* d_mask, const abmx_column* values) {
        check(abmx_agents_set_mask(&s_, d_mask, values, stream_));
    }
    void sort(const double* d_key, bool descending, std::int32_t* d_perm = nullptr) {
        check(abmx_agents_sort(&s_, d_key, descending ? 1 : 0, d_perm, stream_));
    }
    void permute(const std::int32_t* d_perm) { check(abmx_agents_permute(&s_, d_perm, stream_)); }
    const abmx_agent_set& raw() const { return s_; }

private:
    abmx_agent_set s_;
    void* stream_;
};

}  // namespace abmx::cuda
