// Event-bracketed launch overhead on the B200 for the ways a C2 predation step can be issued
// (DESIGN.md §4): direct launches, a CUDA graph (with and without per-launch node-parameter
// updates), a cooperative launch. Kernels are empty (1024 x 256, the step's grid) and the GPU
// is kept busy before each bracket, so host submission latency is not inside it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/launch_overhead tools/launch_overhead.cu
#include <cstdio>
#include <cuda_runtime.h>

struct P {
    unsigned long long a, b;
    int c[16];
};
__global__ void k_empty(P p) {
    if (p.a == 0xFFFFFFFFFFFFFFFFull && threadIdx.x == 1000) p.c[0] = 1;
}
__global__ void k_spin(long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < (unsigned long long)ns);
}

int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    P p{};
    void* args[1] = {&p};
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphNode_t n[2];
    cudaKernelNodeParams kp{};
    kp.func = reinterpret_cast<void*>(k_empty);
    kp.gridDim = dim3(1024);
    kp.blockDim = dim3(256);
    kp.kernelParams = args;
    cudaGraphAddKernelNode(&n[0], g, nullptr, 0, &kp);
    cudaGraphAddKernelNode(&n[1], g, &n[0], 1, &kp);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphUpload(ge, st);
    const char* names[] = {"events only", "1 kernel", "2 kernels", "graph(2)", "graph(2) + node param updates",
                           "cooperative 1 kernel (592 CTAs)", "1 kernel 148 CTAs"};
    for (int v = 0; v < 7; ++v) {
        float sum = 0.f, best = 1e9f;
        const int reps = 50;
        for (int r = 0; r < reps + 5; ++r) {
            k_spin<<<1, 32, 0, st>>>(30000);
            cudaEventRecord(a, st);
            switch (v) {
                case 1: k_empty<<<1024, 256, 0, st>>>(p); break;
                case 2:
                    k_empty<<<1024, 256, 0, st>>>(p);
                    k_empty<<<1024, 256, 0, st>>>(p);
                    break;
                case 3: cudaGraphLaunch(ge, st); break;
                case 4:
                    p.a = r;
                    cudaGraphExecKernelNodeSetParams(ge, n[0], &kp);
                    cudaGraphExecKernelNodeSetParams(ge, n[1], &kp);
                    cudaGraphLaunch(ge, st);
                    break;
                case 5: {
                    cudaLaunchConfig_t cfg{};
                    cfg.gridDim = dim3(592);
                    cfg.blockDim = dim3(256);
                    cfg.stream = st;
                    cudaLaunchAttribute at[1];
                    at[0].id = cudaLaunchAttributeCooperative;
                    at[0].val.cooperative = 1;
                    cfg.attrs = at;
                    cfg.numAttrs = 1;
                    cudaLaunchKernelEx(&cfg, k_empty, p);
                    break;
                }
                case 6: k_empty<<<148, 256, 0, st>>>(p); break;
                default: break;
            }
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 5) {
                sum += ms;
                best = ms < best ? ms : best;
            }
        }
        std::printf("%-36s mean %6.2f us  min %6.2f us\n", names[v], sum / reps * 1e3f, best * 1e3f);
    }
    std::printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
