// Host API latency probe for the per-call (step + metrics) path: how much each runtime call
// costs on the host, and the launch-to-completion round trip of a tiny graph.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o api_lat tools/api_lat.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

struct Big {
    long long v[50];  // a 400-byte kernel parameter block, like the engine's Params
};
__global__ void k_touch(Big b, long long* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) out[0] += b.v[0];
}
__global__ void k_flag(volatile long long* host_flag, long long v) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        __threadfence_system();
        *host_flag = v;
    }
}

static double now_us() {
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    long long* d;
    cudaMalloc(&d, 64);
    cudaMemset(d, 0, 64);
    Big b{};
    void* args[2] = {&b, &d};
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphNode_t nodes[4], prev = nullptr;
    cudaKernelNodeParams kp{};
    kp.func = reinterpret_cast<void*>(k_touch);
    kp.gridDim = dim3(1024);
    kp.blockDim = dim3(256);
    kp.kernelParams = args;
    for (int k = 0; k < 4; ++k) {
        cudaGraphAddKernelNode(&nodes[k], g, prev ? &prev : nullptr, prev ? 1 : 0, &kp);
        prev = nodes[k];
    }
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    const int N = 2000;
    for (int i = 0; i < 10; ++i) cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);

    double a = now_us();
    for (int i = 0; i < N; ++i) cudaGraphExecKernelNodeSetParams(ge, nodes[i & 3], &kp);
    printf("SetParams (400 B)         %7.2f us/call\n", (now_us() - a) / N);

    a = now_us();
    for (int i = 0; i < N; ++i) {
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
    }
    printf("graph(4 nodes)+sync       %7.2f us/iter\n", (now_us() - a) / N);

    a = now_us();
    for (int i = 0; i < N; ++i) {
        for (int k = 0; k < 4; ++k) cudaGraphExecKernelNodeSetParams(ge, nodes[k], &kp);
        cudaGraphLaunch(ge, s);
        cudaStreamSynchronize(s);
    }
    printf("4xSetParams+graph+sync    %7.2f us/iter\n", (now_us() - a) / N);

    a = now_us();
    for (int i = 0; i < N; ++i) {
        for (int k = 0; k < 4; ++k) cudaLaunchKernel(reinterpret_cast<void*>(k_touch), dim3(1024), dim3(256), args, 0, s);
        cudaStreamSynchronize(s);
    }
    printf("4 direct launches+sync    %7.2f us/iter\n", (now_us() - a) / N);

    long long* h;
    cudaHostAlloc(&h, 4096, cudaHostAllocMapped);
    long long* hd;
    cudaHostGetDevicePointer(reinterpret_cast<void**>(&hd), h, 0);
    a = now_us();
    for (int i = 0; i < N; ++i) {
        cudaMemcpyAsync(h, d, 32, cudaMemcpyDeviceToHost, s);
        cudaStreamSynchronize(s);
    }
    printf("D2H 32 B pinned + sync    %7.2f us/iter\n", (now_us() - a) / N);

    a = now_us();
    for (int i = 0; i < N; ++i) {
        cudaMemcpyAsync(d, h, 64, cudaMemcpyHostToDevice, s);
    }
    cudaStreamSynchronize(s);
    printf("H2D 64 B pinned (enqueue) %7.2f us/call\n", (now_us() - a) / N);

    a = now_us();
    for (int i = 0; i < N; ++i) cudaStreamSynchronize(s);
    printf("sync idle stream          %7.2f us/call\n", (now_us() - a) / N);

    a = now_us();
    for (int i = 0; i < N; ++i) {
        k_flag<<<1, 32, 0, s>>>(reinterpret_cast<volatile long long*>(hd), i + 1);
        while (*reinterpret_cast<volatile long long*>(h) != i + 1) {
        }
    }
    printf("kernel -> mapped flag spin %6.2f us/iter\n", (now_us() - a) / N);
    cudaStreamSynchronize(s);

    a = now_us();
    for (int i = 0; i < N; ++i) {
        k_flag<<<1, 32, 0, s>>>(reinterpret_cast<volatile long long*>(hd), i + 1);
        cudaStreamSynchronize(s);
    }
    printf("kernel + sync             %7.2f us/iter\n", (now_us() - a) / N);

    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    a = now_us();
    for (int i = 0; i < N; ++i) {
        k_flag<<<1, 32, 0, s>>>(reinterpret_cast<volatile long long*>(hd), i + 1);
        cudaEventRecord(ev, s);
        while (cudaEventQuery(ev) != cudaSuccess) {
        }
    }
    printf("kernel + event poll       %7.2f us/iter\n", (now_us() - a) / N);
    return 0;
}
