// abmx_internal.h — declarations shared by the .cu translation units (not public).
#pragma once

#include <cstddef>
#include <cstdint>
#include <string>

#include <cuda_runtime.h>

#include "../../include/abmx_cuda.h"

namespace abmx_internal {

constexpr int kMaxDevices = 64;
int num_sms();  // of the current device
// stream-ordered scratch from the library's own per-device pool, kept cached (up to 1 GiB)
// across synchronisations (177 -> 52 us per agent-set lifecycle cycle)
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s);
// raise (never lower) a kernel's dynamic shared-memory limit on the current device
cudaError_t raise_dyn_smem(const void* fn, size_t bytes);
template <class F>
cudaError_t raise_dyn_smem(F* fn, size_t bytes) {
    return raise_dyn_smem(reinterpret_cast<const void*>(fn), bytes);
}
template <class T>
cudaError_t malloc_async(T** p, size_t bytes, cudaStream_t s) {
    return malloc_async(reinterpret_cast<void**>(p), bytes, s);
}
void count_launch(int k = 1);          // launches of our own kernels (gpu_launches)
unsigned long long launches();

void set_error(const std::string& msg);  // thread-local last error
const char* last_error();

// KernelTable launchers (device pointers, stream-ordered); table.cu
cudaError_t launch_rank_scan(const uint8_t* d_mask, int32_t* d_ranks, size_t n, cudaStream_t s);
cudaError_t launch_count_true(const uint8_t* d_mask, size_t n, unsigned long long* d_out,
                              cudaStream_t s);
cudaError_t launch_compact_indices(const uint8_t* d_mask, int32_t* d_out, size_t n,
                                   unsigned long long* d_count, cudaStream_t s);
cudaError_t launch_match_first_equal(const int32_t* d_ra, size_t n, const int32_t* d_rb, size_t m,
                                     int32_t* d_out, cudaStream_t s);
template <class T>
cudaError_t launch_blend(const uint8_t* d_mask, const T* d_a, const T* d_b, T* d_out, size_t n,
                         cudaStream_t s);

// traffic run_batch on the SMEM-resident path (traffic_ens.cu)
bool traffic_ens_fits(const struct abmx_traffic_config& cfg);
int traffic_ensemble_run(const struct abmx_traffic_config& cfg, const uint64_t* seeds, int count, long long steps,
                         double* metrics_out, double* kernel_ms);

}  // namespace abmx_internal
