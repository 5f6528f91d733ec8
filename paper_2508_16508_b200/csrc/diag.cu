// diag.cu — measured ceilings for the roofline of the predation kernels.
//
// k_move and k_update are bound by random accesses to the 16-byte cell words, not by streaming
// HBM bandwidth. This file replays exactly that access pattern, with nothing else, in the same
// launch shape (R x (tiles) CTAs x 256 threads x 4 slots): every live slot does one returning
// atomicExch on a random cell word of a cells-sized array, and every sheep slot also does one
// fire-and-forget atomicMax (mode 0), or the live slots read a random 16-byte cell word
// (mode 1). Timed with CUDA events exactly like the bench's per-kernel times, with or without
// an L2 flush before each launch, so `bench.py` can state the kernels' share of the ceiling.
#include <cstdint>
#include <string>

#include "../../include/abmx_cuda.h"
#include "abmx_internal.h"

namespace {

constexpr int kT = 256, kS = 4;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// blocks [0, sheep_ctas) are sheep tiles (live fraction live_s / 1024), the rest wolf tiles
__global__ void __launch_bounds__(kT, 4) k_access(uint4* cw, unsigned cells, int* out, unsigned salt, int mode,
                                                   unsigned sheep_ctas, unsigned live_s, unsigned live_w) {
    const bool sheep = blockIdx.x < sheep_ctas;
    unsigned* w = reinterpret_cast<unsigned*>(cw);
    unsigned c[kS];
    bool act[kS];
#pragma unroll
    for (int k = 0; k < kS; ++k) {
        const unsigned slot = blockIdx.x * kT * kS + threadIdx.x * kS + k;
        const unsigned long long h = mix(slot * 0x9E3779B97F4A7C15ULL + salt);
        act[k] = (h & 1023) < (sheep ? live_s : live_w);
        c[k] = static_cast<unsigned>((h >> 20) % cells);
    }
    int acc = 0;
    if (mode == 0) {
        unsigned old[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) old[k] = atomicExch(&w[4 * c[k] + (sheep ? 0 : 1)], salt + k);
        if (sheep) {
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (act[k]) atomicMax(&w[4 * c[k] + 2], salt ^ k);
        }
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) acc += old[k];
    } else if (mode == 2) {  // no access: the launch shape, the hashing and the store only
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) acc += static_cast<int>(c[k]);
    } else {
        uint4 v[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) v[k] = cw[c[k]];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) acc += v[k].x ^ v[k].z;
    }
    out[blockIdx.x * kT + threadIdx.x] = acc;
}

__global__ void k_flush_d(uint4* p, size_t n, unsigned s) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = make_uint4(s, static_cast<unsigned>(i), 0, 0);
}
// then read it back, so L2 holds clean lines (as bench.py's flush: no write-backs in the timed kernel)
__global__ void k_flush_read_d(const uint4* p, size_t n, int* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        acc += p[i].x;
    if (acc == 0x12345678u) *out = static_cast<int>(acc);
}

}  // namespace

extern "C" int abmx_diag_random_access(int64_t cells, int32_t sheep_ctas, int32_t wolf_ctas, double live_sheep,
                                       double live_wolves, int32_t mode, int32_t cold, int32_t reps,
                                       double* min_us, double* mean_us) {
    if (cells < 1 || sheep_ctas < 0 || wolf_ctas < 0 || reps < 1 || !min_us) {
        abmx_internal::set_error("bad diag arguments");
        return ABMX_E_ARG;
    }
    const unsigned grid = static_cast<unsigned>(sheep_ctas + wolf_ctas);
    const size_t flush_n = (static_cast<size_t>(256) << 20) / 16;
    uint4 *cw = nullptr, *fl = nullptr;
    int* out = nullptr;
    cudaEvent_t a = nullptr, b = nullptr;
    int rc = ABMX_OK;
    if (cudaMalloc(&cw, static_cast<size_t>(cells) * 16) != cudaSuccess || cudaMalloc(&fl, flush_n * 16) != cudaSuccess ||
        cudaMalloc(&out, static_cast<size_t>(grid) * kT * 4) != cudaSuccess) {
        abmx_internal::set_error("diag: cudaMalloc failed");
        rc = ABMX_E_CUDA;
    } else {
        cudaMemset(cw, 0, static_cast<size_t>(cells) * 16);
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        const unsigned ls = static_cast<unsigned>(live_sheep * 1024.0), lw = static_cast<unsigned>(live_wolves * 1024.0);
        double best = 1e30, sum = 0.0;
        for (int r = 0; r < reps + 3; ++r) {
            const unsigned salt = cold ? 1000u + static_cast<unsigned>(r) : 77u;
            if (cold) {
                k_flush_d<<<abmx_internal::num_sms() * 4, 256>>>(fl, flush_n, static_cast<unsigned>(r));
                k_flush_read_d<<<abmx_internal::num_sms() * 4, 256>>>(fl, flush_n, out);
            } else
                k_access<<<grid, kT>>>(cw, static_cast<unsigned>(cells), out, salt, mode, sheep_ctas, ls, lw);
            cudaEventRecord(a);
            k_access<<<grid, kT>>>(cw, static_cast<unsigned>(cells), out, salt, mode, sheep_ctas, ls, lw);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) {
                best = ms < best ? ms : best;
                sum += ms;
            }
        }
        abmx_internal::count_launch((cold ? 3 : 2) * (reps + 3));
        if (cudaGetLastError() != cudaSuccess) {
            abmx_internal::set_error("diag: launch failed");
            rc = ABMX_E_CUDA;
        }
        *min_us = best * 1e3;
        if (mean_us) *mean_us = sum / reps * 1e3;
    }
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaFree(cw);
    cudaFree(fl);
    cudaFree(out);
    return rc;
}
