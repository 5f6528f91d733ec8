// Cold-code probe: what does a kernel pay to fetch its instructions after the bench's L2 flush?
// Each kernel runs the same ~N straight-line (unrolled) or looped ALU instructions per thread,
// no memory traffic, 296 CTAs x 256 threads; event-timed, median of 50, after either an
// L2-evicting write + read (cold: code lines come from DRAM) or nothing (warm).
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/icache_probe tools/icache_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

template <int kN>
__global__ void k_straight(unsigned* out, unsigned seed) {
    unsigned a = threadIdx.x ^ seed, b = blockIdx.x + seed;
#pragma unroll
    for (int i = 0; i < kN; ++i) {  // distinct constants: no folding into a loop
        a = a * 0x9E3779B1u + (b ^ static_cast<unsigned>(i * 0x85EBCA6B));
        b = __funnelshift_l(b, a, (i * 7) & 31) + static_cast<unsigned>(i);
    }
    if ((a ^ b) == 0x12345678u) out[0] = a;
}
template <int kN>
__global__ void k_looped(unsigned* out, unsigned seed) {
    unsigned a = threadIdx.x ^ seed, b = blockIdx.x + seed;
#pragma unroll 1
    for (int i = 0; i < kN; ++i) {
        a = a * 0x9E3779B1u + (b ^ static_cast<unsigned>(i * 0x85EBCA6B));
        b = __funnelshift_l(b, a, (i * 7) & 31) + static_cast<unsigned>(i);
    }
    if ((a ^ b) == 0x12345678u) out[0] = a;
}
__global__ void k_flush(int* p, size_t n, int v) {
    for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 256ull * gridDim.x) p[i] += v;
}

int main() {
    const size_t fn = (256u << 20) / 4;
    int* fl;
    unsigned* o;
    cudaMalloc(&fl, fn * 4);
    cudaMalloc(&o, 64);
    cudaMemset(fl, 0, fn * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    struct K {
        const char* name;
        void (*fn)(unsigned*, unsigned);
    } ks[] = {{"straight 256", k_straight<256>}, {"looped 256", k_looped<256>},
              {"straight 1024", k_straight<1024>}, {"looped 1024", k_looped<1024>},
              {"straight 2048", k_straight<2048>}, {"looped 2048", k_looped<2048>}};
    for (auto& k : ks) {
        cudaFuncAttributes at{};
        cudaFuncGetAttributes(&at, k.fn);
        for (int cold = 0; cold < 2; ++cold) {
            std::vector<float> v;
            for (int r = 0; r < 53; ++r) {
                if (cold) k_flush<<<1184, 256>>>(fl, fn, r);  // 256 MB read-modify-write
                cudaEventRecord(a);
                k.fn<<<296, 256>>>(o, r);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) v.push_back(ms * 1000.f);
            }
            std::sort(v.begin(), v.end());
            printf("%-14s %-4s p50 %7.2f us  p10 %7.2f  p90 %7.2f\n", k.name, cold ? "cold" : "warm",
                   v[v.size() / 2], v[v.size() / 10], v[v.size() * 9 / 10]);
        }
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
