// abmx_cuda.hpp — header-only C++ host mirror of the reference interface over the C-ABI
// in abmx_cuda.h. A reference user keeps the reference's names and argument meaning:
//
//   abmx::models::PredationModel (include/abmx/models/predation.hpp:91-107)
//       -> abmx::cuda::PredationModel   step(t), collect_metrics(rows), last_events()
//   abmx::run_batch / replica_seeds (include/abmx/batch.hpp:48-54)
//       -> abmx::cuda::run_batch / replica_seeds
//   abmx::simd::KernelTable (include/abmx/simd/kernels.hpp:15-43)
//       -> abmx::cuda::kernel_table()  (same layout)
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

}  // namespace abmx::cuda
