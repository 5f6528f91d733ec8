// microbench.cu — B200 access-pattern probes for the predation step design (not product code).
// Measures, with CUDA events after an L2 flush (write 256 MiB + read 256 MiB):
//   stream  : 1M slots x (1 B + 4 B + 4 B read, 4 B + 4 B write)  — k_move's dense columns
//   atom    : 400k random atomicExch on a 32 MiB array (cold)
//   load    : 400k random 4-byte loads from a 32 MiB array (cold)
//   load_l2 : the same loads with the array L2-resident
//   chain2  : 400k x 2 dependent random loads (cold)
//   empty   : an empty kernel of 1024 x 256 threads
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <vector>

#include <cuda_runtime.h>

#define CK(x)                                                                           \
    do {                                                                                \
        cudaError_t e = (x);                                                            \
        if (e != cudaSuccess) {                                                         \
            printf("%s failed: %s\n", #x, cudaGetErrorString(e));                       \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

__global__ void k_empty() {}

__global__ void k_stream(const uint8_t* act, int* cell, int* age, int n) {
    const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    if (i0 >= n) return;
    const uint32_t a = *reinterpret_cast<const uint32_t*>(act + i0);
    int4 c = *reinterpret_cast<int4*>(cell + i0);
    int4 g = *reinterpret_cast<int4*>(age + i0);
    if (a) {
        c.x += 1; c.y += 1; c.z += 1; c.w += 1;
        g.x += 1; g.y += 1; g.z += 1; g.w += 1;
        *reinterpret_cast<int4*>(cell + i0) = c;
        *reinterpret_cast<int4*>(age + i0) = g;
    }
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__global__ void k_atom(unsigned* arr, uint32_t mask, int n, int* out) {
    const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    unsigned acc = 0;
    unsigned old[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i0 + k < n) old[k] = atomicExch(&arr[hash32(i0 + k) & mask], i0 + k);
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i0 + k < n) acc += old[k];
    if (acc == 0xFFFFFFFF) *out = 1;
}

__global__ void k_load(const unsigned* arr, uint32_t mask, int n, int* out) {
    const int i0 = (blockIdx.x * blockDim.x + threadIdx.x) * 4;
    unsigned acc = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k)
        if (i0 + k < n) acc += arr[hash32(i0 + k) & mask];
    if (acc == 0xFFFFFFFF) *out = 1;
}

__global__ void k_chain2(const unsigned* arr, uint32_t mask, int n, int* out) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const unsigned a = arr[hash32(i) & mask];
    const unsigned b = arr[hash32(a + i) & mask];
    if (b == 0xFFFFFFFF) *out = 1;
}

__global__ void k_flush(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(i, 0, 0, 0);
}
__global__ void k_flush_read(const uint4* p, size_t n, int* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= p[i].x;
    if (acc == 0x12345) *out = 1;
}

int main() {
    const int N = 1 << 20, A = 400000;
    const size_t FB = 256u << 20;
    uint8_t* act;
    int *cell, *age, *out;
    unsigned* arr;
    uint4* fb;
    CK(cudaMalloc(&act, N));
    CK(cudaMalloc(&cell, N * 4));
    CK(cudaMalloc(&age, N * 4));
    CK(cudaMalloc(&arr, 32u << 20));
    CK(cudaMalloc(&out, 4));
    CK(cudaMalloc(&fb, 2 * FB));
    CK(cudaMemset(act, 1, N));
    CK(cudaMemset(cell, 0, N * 4));
    CK(cudaMemset(age, 0, N * 4));
    CK(cudaMemset(arr, 0, 32u << 20));
    CK(cudaMemset(fb, 0, 2 * FB));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint32_t mask = (8u << 20) - 1;  // 8M u32 = 32 MiB
    auto flush = [&]() {
        k_flush<<<592, 256>>>(fb, FB / 16);
        k_flush_read<<<592, 256>>>(fb + FB / 16, FB / 16, out);
    };
    for (int rep = 0; rep < 2; ++rep) {
        float ms;
        const char* names[] = {"empty", "stream", "atom", "load", "load_l2", "chain2"};
        for (int t = 0; t < 6; ++t) {
            float best = 1e9;
            for (int it = 0; it < 5; ++it) {
                if (t != 4) flush();
                else k_load<<<(A / 4 + 255) / 256, 256>>>(arr, mask, A, out);  // warm
                cudaEventRecord(e0);
                switch (t) {
                    case 0: k_empty<<<1024, 256>>>(); break;
                    case 1: k_stream<<<N / 4 / 256, 256>>>(act, cell, age, N); break;
                    case 2: k_atom<<<(A / 4 + 255) / 256, 256>>>(arr, mask, A, out); break;
                    case 3: k_load<<<(A / 4 + 255) / 256, 256>>>(arr, mask, A, out); break;
                    case 4: k_load<<<(A / 4 + 255) / 256, 256>>>(arr, mask, A, out); break;
                    case 5: k_chain2<<<(A + 255) / 256, 256>>>(arr, mask, A, out); break;
                }
                cudaEventRecord(e1);
                CK(cudaEventSynchronize(e1));
                cudaEventElapsedTime(&ms, e0, e1);
                if (ms < best) best = ms;
            }
            if (rep == 1) printf("%-8s %8.2f us\n", names[t], best * 1000);
        }
    }
    return 0;
}
