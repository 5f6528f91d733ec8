// Launch-overhead probe for the fused lifecycle cycle (bench.py `agents`): event-timed, after an
// L2-flushing write, median of 50 reps each:
//   memset8        cudaMemsetAsync of 8 bytes (the barrier counters)
//   empty          256 x 256 empty kernel, plain launch
//   empty_coop     the same with cudaLaunchAttributeCooperative
//   memset+coop    both, as abmx_agents_lifecycle issues them
//   coop_2bar      memset + cooperative kernel that only crosses two grid barriers
//   plain_2bar     the same two barriers, plain launch (co-residency not guaranteed by the API)
//   empty_smem33k  the empty kernel with 33 KB of static shared memory (a carveout change after the
//                  flush kernel); smem33k_coop the same, memset + cooperative
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/launch_probe tools/launch_probe.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <vector>

__global__ void k_empty() {}
__global__ void k_empty_smem() {  // 33 KB of static shared memory, like k_life_coop
    __shared__ unsigned long long buf[4100];
    if (threadIdx.x == 1024) buf[threadIdx.x] = 1;  // never true: keeps the array
    __syncthreads();
    if (threadIdx.x == 1025) asm volatile("" ::"l"(buf[0]));
}
__global__ void k_flush(int* p, size_t n, int v) {
    for (size_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += 256ull * gridDim.x) p[i] = v;
}
__device__ __forceinline__ void bar(unsigned* c, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(c) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
        } while (v < G);
    }
    __syncthreads();
}
__global__ void k_2bar(unsigned* c) {
    bar(c, gridDim.x);
    bar(c + 1, gridDim.x);
}

int main() {
    const size_t fn = (256u << 20) / 4;
    int* fl;
    unsigned* ctr;
    cudaMalloc(&fl, fn * 4);
    cudaMalloc(&ctr, 64);
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto launch = [&](void (*k)(), bool coop) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(256);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = coop ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k);
    };
    auto launch2 = [&](bool coop) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(256);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeCooperative;
        at[0].val.cooperative = 1;
        cfg.attrs = at;
        cfg.numAttrs = coop ? 1 : 0;
        cudaLaunchKernelEx(&cfg, k_2bar, ctr);
    };
    const char* names[] = {"memset8", "empty", "empty_coop", "memset+coop", "coop_2bar", "plain_2bar", "empty_smem33k",
                           "smem33k_coop"};
    for (int t = 0; t < 8; ++t) {
        std::vector<float> v;
        for (int r = 0; r < 53; ++r) {
            k_flush<<<1184, 256, 0, st>>>(fl, fn, r);
            cudaEventRecord(a, st);
            switch (t) {
                case 0: cudaMemsetAsync(ctr, 0, 8, st); break;
                case 1: launch(k_empty, false); break;
                case 2: launch(k_empty, true); break;
                case 3: cudaMemsetAsync(ctr, 0, 8, st); launch(k_empty, true); break;
                case 4: cudaMemsetAsync(ctr, 0, 8, st); launch2(true); break;
                case 5: cudaMemsetAsync(ctr, 0, 8, st); launch2(false); break;
                case 6: launch(k_empty_smem, false); break;
                case 7: cudaMemsetAsync(ctr, 0, 8, st); launch(k_empty_smem, true); break;
            }
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) v.push_back(ms * 1000.f);
        }
        std::sort(v.begin(), v.end());
        printf("%-12s p50 %6.2f us  p10 %6.2f  p90 %6.2f\n", names[t], v[v.size() / 2], v[v.size() / 10],
               v[v.size() * 9 / 10]);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return e != cudaSuccess;
}
