// Cost model of the C2 predation step's memory operations on the B200: each
// access class the step performs, alone, in the step's launch shape (1M slots: 524,288 sheep
// slots ~70% live, 524,288 wolf slots with ~35k live packed low), cold (L2 flushed) and warm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/c2_floor tools/c2_floor.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kT = 256, kS = 4;
constexpr unsigned kN = 524288u;          // slots per species
constexpr unsigned kCells = 2048u * 2048u;
constexpr unsigned kWolfLive = 45000u;    // wolves live in [0, kWolfLive) at ~78%

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

struct Buf {
    uint8_t* act[2];
    int* cell[2];
    int* age[2];
    double* E[2];
    int* next[2];
    uint4* cw;         // 16 B per cell
    unsigned* cw4;     // 4 B per cell
    unsigned short* g2;  // 2 B per cell
    int* out;
};

enum Mode {
    kStreamMove, kStreamUpdate, kAtomCur, kRedMin, kRedMinMax, kLoad16, kRed4Warm, kLoad2, kPrefetchLoad2,
    kMoveFull, kMoveRed, kNumModes
};
static const char* kNames[kNumModes] = {
    "stream k_move cols (act,cell,age r; cell,age w)",
    "stream k_update cols (act,cell,E r; E,act w)",
    "atoms: exch/live + max/sheep (current)",
    "atoms: RED.max/sheep + exch/wolf",
    "atoms: 2x RED.max/sheep + exch/wolf",
    "random 16B load/live",
    "RED.max on 4B/cell array (16.8MB)",
    "random 2B load/sheep from 8.4MB",
    "stream 8.4MB (2B/cell) then random 2B loads",
    "k_move-like: stream + current atoms + next[] write",
    "k_move-like: stream + RED.max sheep + exch wolf",
};

template <int M>
__global__ void __launch_bounds__(kT, 4) k_pat(Buf B, unsigned salt) {
    const int s = blockIdx.x < gridDim.x / 2 ? 0 : 1;
    const unsigned tile = s == 0 ? blockIdx.x : blockIdx.x - gridDim.x / 2;
    const unsigned i0 = tile * kT * kS + threadIdx.x * kS;
    uint8_t act[kS];
    int cell[kS];
    {
        const uint32_t w = *reinterpret_cast<const uint32_t*>(B.act[s] + i0);
        for (int k = 0; k < kS; ++k) act[k] = (w >> (8 * k)) & 0xFF;
    }
    bool any = false;
    for (int k = 0; k < kS; ++k) any |= act[k] != 0;
    if constexpr (M == kStreamMove || M == kMoveFull || M == kMoveRed) {
        if (!any) return;
        int4 c = *reinterpret_cast<const int4*>(B.cell[s] + i0);
        int4 a = *reinterpret_cast<const int4*>(B.age[s] + i0);
        cell[0] = c.x; cell[1] = c.y; cell[2] = c.z; cell[3] = c.w;
        for (int k = 0; k < kS; ++k) cell[k] = act[k] ? (int)((cell[k] + 2049u + salt) % kCells) : cell[k];
        a.x += act[0]; a.y += act[1]; a.z += act[2]; a.w += act[3];
        if constexpr (M == kMoveFull || M == kMoveRed) {
            unsigned* w = reinterpret_cast<unsigned*>(B.cw);
            unsigned old[kS];
            const bool exch = M == kMoveFull || s == 1;
            if (exch)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) old[k] = atomicExch(&w[4 * cell[k] + s], salt + i0 + k);
            if (s == 0)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) atomicMax(&w[4 * cell[k] + 2], salt ^ (i0 + k));
            if (exch)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) B.next[s][i0 + k] = (int)old[k];
        }
        *reinterpret_cast<int4*>(B.cell[s] + i0) = make_int4(cell[0], cell[1], cell[2], cell[3]);
        *reinterpret_cast<int4*>(B.age[s] + i0) = a;
        return;
    }
    if constexpr (M == kStreamUpdate) {
        if (!any) return;
        int4 c = *reinterpret_cast<const int4*>(B.cell[s] + i0);
        double2 e0 = reinterpret_cast<const double2*>(B.E[s] + i0)[0];
        double2 e1 = reinterpret_cast<const double2*>(B.E[s] + i0)[1];
        e0.x -= 1.0 + (c.x & 1); e0.y -= 1.0; e1.x -= 1.0; e1.y -= 1.0 + (c.w & 1);
        reinterpret_cast<double2*>(B.E[s] + i0)[0] = e0;
        reinterpret_cast<double2*>(B.E[s] + i0)[1] = e1;
        if ((c.y & 255) == 7) *reinterpret_cast<uint32_t*>(B.act[s] + i0) = 0x01010101u;
        return;
    }
    // synthetic random cells for the pure-access modes
    for (int k = 0; k < kS; ++k) cell[k] = (int)(mix((unsigned long long)(s * kN + i0 + k) * 0x9E3779B97F4A7C15ULL + salt) % kCells);
    int acc = 0;
    if constexpr (M == kAtomCur || M == kRedMin || M == kRedMinMax) {
        unsigned* w = reinterpret_cast<unsigned*>(B.cw);
        unsigned old[kS];
        const bool exch = M == kAtomCur || s == 1;
        if (exch)
            for (int k = 0; k < kS; ++k)
                if (act[k]) old[k] = atomicExch(&w[4 * cell[k] + s], salt + k);
        if (s == 0) {
            for (int k = 0; k < kS; ++k)
                if (act[k]) atomicMax(&w[4 * cell[k] + 2], salt ^ k);
            if (M == kRedMinMax)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) atomicMax(&w[4 * cell[k] + 3], salt + k);
        }
        if (exch)
            for (int k = 0; k < kS; ++k)
                if (act[k]) acc += old[k];
    } else if constexpr (M == kLoad16) {
        uint4 v[kS];
        for (int k = 0; k < kS; ++k)
            if (act[k]) v[k] = B.cw[cell[k]];
        for (int k = 0; k < kS; ++k)
            if (act[k]) acc += v[k].x ^ v[k].z;
    } else if constexpr (M == kRed4Warm) {
        for (int k = 0; k < kS; ++k)
            if (act[k]) atomicMax(&B.cw4[cell[k]], salt ^ k);
    } else if constexpr (M == kLoad2 || M == kPrefetchLoad2) {
        if (s == 0) {
            unsigned short v[kS];
            for (int k = 0; k < kS; ++k)
                if (act[k]) v[k] = B.g2[cell[k]];
            for (int k = 0; k < kS; ++k)
                if (act[k]) acc += v[k];
        }
    }
    if (acc == 0x7654321) B.out[0] = acc;
}

__global__ void k_stream_read(const uint4* p, size_t n, int* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = p[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9E3779B9u) *out = acc;
}

__global__ void k_flush(uint4* p, size_t n, unsigned s) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(s, (unsigned)i, 0, 0);
}

__global__ void k_init(Buf B) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < 2ull * kN; q += (size_t)gridDim.x * blockDim.x) {
        const int s = q >= kN;
        const unsigned i = (unsigned)(q - s * kN);
        const unsigned long long h = mix(q * 0x9E3779B97F4A7C15ULL + 12345);
        const bool live = s == 0 ? (h & 1023) < 717 : (i < kWolfLive && (h & 1023) < 800);
        B.act[s][i] = live;
        B.cell[s][i] = (int)((h >> 20) % kCells);
        B.age[s][i] = 1;
        B.E[s][i] = 10.0;
    }
}

template <int M>
void launch(Buf B, unsigned salt, cudaStream_t st) {
    k_pat<M><<<2 * kN / (kT * kS), kT, 0, st>>>(B, salt);
}
using LaunchFn = void (*)(Buf, unsigned, cudaStream_t);
static LaunchFn kFns[kNumModes] = {launch<0>, launch<1>, launch<2>, launch<3>, launch<4>, launch<5>,
                                   launch<6>, launch<7>, launch<8>, launch<9>, launch<10>};

int main() {
    Buf B{};
    for (int s = 0; s < 2; ++s) {
        cudaMalloc(&B.act[s], kN);
        cudaMalloc(&B.cell[s], kN * 4);
        cudaMalloc(&B.age[s], kN * 4);
        cudaMalloc(&B.E[s], kN * 8);
        cudaMalloc(&B.next[s], kN * 4);
    }
    cudaMalloc(&B.cw, (size_t)kCells * 16);
    cudaMalloc(&B.cw4, (size_t)kCells * 4);
    cudaMalloc(&B.g2, (size_t)kCells * 2);
    cudaMalloc(&B.out, 64);
    cudaMemset(B.cw, 0, (size_t)kCells * 16);
    cudaMemset(B.cw4, 0, (size_t)kCells * 4);
    cudaMemset(B.g2, 0, (size_t)kCells * 2);
    k_init<<<148 * 8, 256>>>(B);
    uint4* fl;
    const size_t flush_n = (256u << 20) / 16;
    cudaMalloc(&fl, 2 * flush_n * 16);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 20;
    std::printf("%-52s %10s %10s\n", "mode", "cold us", "warm us");
    for (int m = 0; m < kNumModes; ++m) {
        float res[2];
        for (int cold = 1; cold >= 0; --cold) {
            float sum = 0.f;
            for (int r = 0; r < reps + 3; ++r) {
                if (cold) {
                    k_flush<<<148 * 4, 256, 0, st>>>(fl, flush_n, r);
                    k_stream_read<<<148 * 4, 256, 0, st>>>(fl + flush_n, flush_n, B.out);
                } else {
                    kFns[m](B, 77u + r, st);
                }
                if (m == kRed4Warm) cudaMemsetAsync(B.cw4, 0, (size_t)kCells * 4, st);  // L2-resident scratch
                cudaEventRecord(a, st);
                if (m == kPrefetchLoad2)
                    k_stream_read<<<148 * 4, 256, 0, st>>>(reinterpret_cast<const uint4*>(B.g2), (size_t)kCells * 2 / 16, B.out);
                kFns[m](B, 1000u + r, st);
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms = 0.f;
                cudaEventElapsedTime(&ms, a, b);
                if (r >= 3) sum += ms;
            }
            res[cold] = sum / reps * 1e3f;
        }
        std::printf("%-52s %10.2f %10.2f\n", kNames[m], res[1], res[0]);
    }
    // memset of the 4 B/cell scratch alone, and a 16.8 MB streaming read
    float sum = 0.f;
    for (int r = 0; r < reps + 3; ++r) {
        k_flush<<<148 * 4, 256, 0, st>>>(fl, flush_n, r);
        cudaEventRecord(a, st);
        cudaMemsetAsync(B.cw4, 0, (size_t)kCells * 4, st);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) sum += ms;
    }
    std::printf("%-52s %10.2f\n", "memset 16.8 MB (4 B/cell)", sum / reps * 1e3f);
    std::printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
