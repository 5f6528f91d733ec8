// Peak rate of random accesses to HBM on the B200: the ceiling for C2's cell-word accesses
// (profiles/r02_c2_cost_model.md §6). A 1 GiB array of 16-byte cells (64M cells: every access is
// an L2 miss, like C2's flushed cell words, which each step touches ~0.1 times per cell); every
// thread issues kDepth independent accesses per round to hashed cells; 4M accesses per launch
// (~30-80 us, so the ~6 us launch floor is a small share); L2 flushed clean before each launch.
// Arguments: array MiB (default 1024), accesses per launch (default 4M); "none" is the launch-shape
// baseline (hashing only). C2-like: `64 419430` (0.1 access per cell, as in a step).
// Accesses: 16-byte load, RED.max (32-bit, fire and forget), atomicExch (32-bit, returning).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/random_peak tools/random_peak.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

size_t kCells = size_t{64} << 20;  // cells of 16 bytes (argv[1] MiB of array)
unsigned kTotal = 4u << 20;        // accesses per launch (argv[2])

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

template <int kOp, int kDepth>
__global__ void __launch_bounds__(256) k_rand(uint4* arr, size_t cells, unsigned rounds, unsigned salt, unsigned* sink) {
    const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned acc = 0;
    for (unsigned r = 0; r < rounds; ++r) {
        size_t c[kDepth];
#pragma unroll
        for (int k = 0; k < kDepth; ++k)
            c[k] = mix((static_cast<unsigned long long>(t) * rounds + r) * kDepth + k + salt * 0x9E3779B97F4A7C15ULL) % cells;
        if constexpr (kOp == 3) {  // nothing: the launch-shape baseline
            acc += static_cast<unsigned>(c[0]);
        } else if constexpr (kOp == 0) {  // 16-byte loads, all issued before any use
            uint4 v[kDepth];
#pragma unroll
            for (int k = 0; k < kDepth; ++k) v[k] = __ldcg(arr + c[k]);
#pragma unroll
            for (int k = 0; k < kDepth; ++k) acc += v[k].x ^ v[k].w;
        } else if constexpr (kOp == 1) {  // RED.max
#pragma unroll
            for (int k = 0; k < kDepth; ++k) atomicMax(reinterpret_cast<unsigned*>(arr + c[k]), salt + k);
        } else {  // returning exchange
            unsigned o[kDepth];
#pragma unroll
            for (int k = 0; k < kDepth; ++k) o[k] = atomicExch(reinterpret_cast<unsigned*>(arr + c[k]), salt + k);
#pragma unroll
            for (int k = 0; k < kDepth; ++k) acc += o[k];
        }
    }
    if (acc == 0x12345678u) *sink = acc;
}

__global__ void k_fill(uint4* p, size_t n, unsigned v) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = make_uint4(v, v, v, v);
}
__global__ void k_read(const uint4* p, size_t n, unsigned* sink) {
    unsigned a = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * blockDim.x)
        a += p[i].x;
    if (a == 0x12345678u) *sink = a;
}

int main(int argc, char** argv) {
    if (argc > 1) kCells = (static_cast<size_t>(atoi(argv[1])) << 20) / 16;
    if (argc > 2) kTotal = static_cast<unsigned>(atoi(argv[2]));
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    uint4* arr;
    uint4* fl;
    unsigned* sink;
    const size_t flush_n = (size_t{256} << 20) / 16;
    cudaMalloc(&arr, kCells * 16);
    cudaMalloc(&fl, flush_n * 16);
    cudaMalloc(&sink, 4);
    cudaMemset(arr, 0, kCells * 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto flush = [&] {
        k_fill<<<sms * 8, 256>>>(fl, flush_n, 1);
        k_read<<<sms * 8, 256>>>(fl, flush_n, sink);
    };
    printf("array %zu MiB, %u accesses per launch\n", kCells * 16 >> 20, kTotal);
    printf("%-10s %6s %8s %9s %10s %12s\n", "access", "depth", "threads", "rounds", "us", "Gaccess/s");
    auto run = [&](const char* name, auto kern, int depth, unsigned threads) {
        const unsigned rounds = kTotal / (threads * depth) > 0 ? kTotal / (threads * depth) : 1;
        float best = 1e9f;
        for (int rep = 0; rep < 5; ++rep) {
            flush();
            cudaEventRecord(a);
            kern<<<threads / 256, 256>>>(arr, kCells, rounds, 17u + rep, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms = 0;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        const double acc = static_cast<double>(rounds) * threads * depth;
        printf("%-10s %6d %8u %9u %10.2f %12.1f\n", name, depth, threads, rounds, best * 1e3, acc / (best * 1e-3) / 1e9);
    };
    const unsigned full = static_cast<unsigned>(sms) * 2048;  // every SM full (8 CTAs of 256)
    for (unsigned thr : {full / 4, full}) {
        run("none", k_rand<3, 1>, 1, thr);
        run("load16", k_rand<0, 1>, 1, thr);
        run("load16", k_rand<0, 4>, 4, thr);
        run("red.max", k_rand<1, 1>, 1, thr);
        run("red.max", k_rand<1, 4>, 4, thr);
        run("exch", k_rand<2, 1>, 1, thr);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
