// Random-atomic ceiling of the B200 for the C2 access pattern (the bound DESIGN.md §4 uses for
// k_move / k_update): ~330k agents each do one returning atomicExch and (sheep) one
// fire-and-forget atomicMax on a random 16-byte cell word of a 64 MB array (4.19M cells), in
// the same launch shape as k_move (1024 CTAs x 256 threads x 4 slots, ~32% of slots live).
// Also: the same number of random 16-byte reads (k_update's cell-word reads).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o atomic_ceiling tools/atomic_ceiling.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int kT = 256, kS = 4;
constexpr unsigned kCells = 2048u * 2048u;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// mode 0: exch (+ max for half the grid = "sheep" tiles); mode 1: random 16-byte loads
__global__ void __launch_bounds__(kT, 4) k_pattern(uint4* cw, int* out, unsigned salt, int mode, unsigned live_per_1024) {
    const bool sheep = blockIdx.x < gridDim.x / 2;
    unsigned* w = reinterpret_cast<unsigned*>(cw);
    unsigned old[kS];
    unsigned c[kS];
    bool act[kS];
#pragma unroll
    for (int k = 0; k < kS; ++k) {
        const unsigned slot = blockIdx.x * kT * kS + threadIdx.x * kS + k;
        const unsigned long long h = mix(slot * 0x9E3779B97F4A7C15ULL + salt);
        act[k] = (h & 1023) < live_per_1024 && (sheep || (h >> 10 & 15) == 0);
        c[k] = static_cast<unsigned>((h >> 20) % kCells);
    }
    if (mode == 2) {  // L2 prefetch of every target line first, then the same atomics
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) asm volatile("prefetch.global.L2 [%0];" :: "l"(&cw[c[k]]));
    }
    if (mode == 0 || mode == 2) {
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) old[k] = atomicExch(&w[4 * c[k] + (sheep ? 0 : 1)], salt + k);
        if (sheep) {
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (act[k]) atomicMax(&w[4 * c[k] + 2], salt ^ k);
        }
        int acc = 0;
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) acc += old[k];
        out[blockIdx.x * kT + threadIdx.x] = acc;
    } else {
        uint4 v[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) v[k] = cw[c[k]];
        int acc = 0;
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) acc += v[k].x ^ v[k].z;
        out[blockIdx.x * kT + threadIdx.x] = acc;
    }
}

__global__ void k_flush(uint4* p, size_t n, unsigned s) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(s, (unsigned)i, 0, 0);
}

int main() {
    uint4 *cw, *fl;
    int* out;
    const size_t flush_n = (256u << 20) / 16;
    cudaMalloc(&cw, (size_t)kCells * 16);
    cudaMalloc(&fl, flush_n * 16);
    cudaMalloc(&out, 1024 * kT * 4);
    cudaMemset(cw, 0, (size_t)kCells * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned live = 700;  // C2: ~70% of the sheep slots live (~370k of 524k), wolves ~4%
    const char* names[3] = {"atomics (exch + max)", "random 16B loads", "prefetch + atomics"};
    for (int mode = 0; mode < 3; ++mode)
        for (int cold = 1; cold >= 0; --cold) {
            float best = 1e9f, sum = 0.f;
            const int reps = 20;
            for (int r = 0; r < reps + 3; ++r) {
                if (cold) k_flush<<<148 * 4, 256>>>(fl, flush_n, r);
                else k_pattern<<<1024, kT>>>(cw, out, 77u + r, mode, live);  // warm the same lines
                cudaEventRecord(a);
                k_pattern<<<1024, kT>>>(cw, out, cold ? 1000u + r : 77u + r, mode, live);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) {
                    best = ms < best ? ms : best;
                    sum += ms;
                }
            }
            std::printf("%-22s %s: min %.2f us  mean %.2f us\n", names[mode], cold ? "cold (L2 flushed)" : "warm", best * 1e3,
                        sum / reps * 1e3);
        }
    // empty-kernel floor of the same launch shape
    float best = 1e9f;
    for (int r = 0; r < 20; ++r) {
        cudaEventRecord(a);
        k_pattern<<<1024, kT>>>(cw, out, 5u, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    std::printf("%-22s: min %.2f us\n", "launch floor (no live)", best * 1e3);
    return 0;
}
