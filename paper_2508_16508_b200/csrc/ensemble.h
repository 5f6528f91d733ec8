// ensemble.h — the SMEM/register-resident CTA-per-replica ensemble runner (internal).
#pragma once

#include <cstdint>

#include "../../include/abmx_cuda.h"

namespace abmx_ens {

bool smem_fits(const abmx_predation_config& cfg);

// Final state of one replica in the reference layout (for parity tests).
struct Dump {
    int32_t replica;  // relative to the run's first replica
    uint8_t* active[2];
    int64_t* ids[2];
    int64_t* ages[2];
    int64_t* x[2];
    int64_t* y[2];
    double* energy[2];
    int32_t num_active[2];
    int64_t next_id[2];
    uint8_t* grass_ready;
    int64_t* regrow;
};

int run_smem(const abmx_predation_config& cfg, const uint64_t* seeds, int count, long long steps,
             double* metrics_out, double* kernel_ms, Dump* dump = nullptr);

}  // namespace abmx_ens
