// Random-access cost vs per-cell footprint for the C2 grid (4.19M cells) on the B200: the same
// ~370k sheep / ~35k wolf accesses (C2 live counts, random cells) as RED.max or loads on a cell
// array of 2, 4, 8 or 16 B per cell. Cold (L2 flushed, clean) and warm (same cells as the
// previous launch). Each line subtracts nothing: compare against the "none" baseline line of the
// same launch shape (mask load only).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/cell_layout tools/cell_layout.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int kT = 256, kS = 4;
constexpr unsigned kN = 524288u;
constexpr unsigned kCells = 2048u * 2048u;
constexpr unsigned kWolfLive = 45000u;

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

// op: 0 none, 1 RED.max 32-bit at word (cell * W/4), 2 load of W bytes, 3 exch (returning)
template <int kOp, int kW>
__global__ void __launch_bounds__(kT, 4) k_acc(const uint8_t* act0, const uint8_t* act1, unsigned char* arr, unsigned salt,
                                               int* out) {
    const int s = blockIdx.x < gridDim.x / 2 ? 0 : 1;
    const unsigned tile = s == 0 ? blockIdx.x : blockIdx.x - gridDim.x / 2;
    const unsigned i0 = tile * kT * kS + threadIdx.x * kS;
    const uint32_t aw = *reinterpret_cast<const uint32_t*>((s ? act1 : act0) + i0);
    if (!aw) return;
    unsigned acc = 0;
    unsigned c[kS];
#pragma unroll
    for (int k = 0; k < kS; ++k) c[k] = static_cast<unsigned>(mix((s * kN + i0 + k) * 0x9E3779B97F4A7C15ULL + salt) % kCells);
    if constexpr (kOp == 1) {
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if ((aw >> (8 * k)) & 0xFF) atomicMax(reinterpret_cast<unsigned*>(arr + static_cast<size_t>(c[k]) * kW), salt + k);
    } else if constexpr (kOp == 3) {
        unsigned o[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if ((aw >> (8 * k)) & 0xFF) o[k] = atomicExch(reinterpret_cast<unsigned*>(arr + static_cast<size_t>(c[k]) * kW), salt + k);
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if ((aw >> (8 * k)) & 0xFF) acc += o[k];
    } else if constexpr (kOp == 2) {
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if ((aw >> (8 * k)) & 0xFF) {
                const unsigned char* p = arr + static_cast<size_t>(c[k]) * (kW == 17 ? 16 : kW);
                if constexpr (kW == 16) {
                    const uint4 v = *reinterpret_cast<const uint4*>(p);
                    acc += v.x ^ v.w;
                } else if constexpr (kW == 17) {  // 16 B via ld.global.cg (L2 only)
                    const uint4 v = __ldcg(reinterpret_cast<const uint4*>(arr + static_cast<size_t>(c[k]) * 16));
                    acc += v.x ^ v.w;
                } else if constexpr (kW == 8) {
                    const uint2 v = *reinterpret_cast<const uint2*>(p);
                    acc += v.x ^ v.y;
                } else if constexpr (kW == 4) {
                    acc += *reinterpret_cast<const unsigned*>(p);
                } else {
                    acc += *reinterpret_cast<const unsigned short*>(p);
                }
            }
    }
    if (acc == 0x7654321u) *out = acc;
}

__global__ void k_flush(uint4* p, size_t n, unsigned s) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(s, (unsigned)i, 0, 0);
}
__global__ void k_stream_read(const uint4* p, size_t n, int* out) {
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = p[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9E3779B9u) *out = acc;
}
__global__ void k_init(uint8_t* a0, uint8_t* a1) {
    for (size_t q = blockIdx.x * (size_t)blockDim.x + threadIdx.x; q < 2ull * kN; q += (size_t)gridDim.x * blockDim.x) {
        const int s = q >= kN;
        const unsigned i = (unsigned)(q - s * kN);
        const unsigned long long h = mix(q * 0x9E3779B97F4A7C15ULL + 12345);
        (s ? a1 : a0)[i] = s == 0 ? (h & 1023) < 717 : (i < kWolfLive && (h & 1023) < 800);
    }
}
__global__ void k_spin(long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    } while (t - t0 < (unsigned long long)ns);
}

template <int kOp, int kW>
void measure(const char* name, uint8_t* a0, uint8_t* a1, unsigned char* arr, uint4* fl, size_t fn, int* out, cudaStream_t st, int smem = 0) {
    cudaFuncSetAttribute(k_acc<kOp, kW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float res[2];
    for (int cold = 1; cold >= 0; --cold) {
        float sum = 0.f;
        const int reps = 20;
        for (int r = 0; r < reps + 3; ++r) {
            const unsigned salt = cold ? 1000u + r : 77u;
            if (cold) {
                k_flush<<<148 * 4, 256, 0, st>>>(fl, fn, r);
                k_stream_read<<<148 * 4, 256, 0, st>>>(fl + fn, fn, out);
            } else {
                k_acc<kOp, kW><<<2 * kN / (kT * kS), kT, 0, st>>>(a0, a1, arr, salt, out);
                k_spin<<<1, 32, 0, st>>>(20000);
            }
            cudaEventRecord(a, st);
            k_acc<kOp, kW><<<2 * kN / (kT * kS), kT, smem, st>>>(a0, a1, arr, salt, out);
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (r >= 3) sum += ms;
        }
        res[cold] = sum / reps * 1e3f;
    }
    std::printf("%-40s %8.2f %8.2f\n", name, res[1], res[0]);
}

int main() {
    setvbuf(stdout, nullptr, _IONBF, 0);
    uint8_t *a0, *a1;
    unsigned char* arr;
    int* out;
    cudaMalloc(&a0, kN);
    cudaMalloc(&a1, kN);
    cudaMalloc(&arr, (size_t)kCells * 16);
    cudaMemset(arr, 0, (size_t)kCells * 16);
    cudaMalloc(&out, 64);
    k_init<<<148 * 8, 256>>>(a0, a1);
    uint4* fl;
    const size_t fn = (256u << 20) / 16;
    cudaMalloc(&fl, 2 * fn * 16);
    cudaStream_t st;
    cudaStreamCreate(&st);
    std::printf("%-40s %8s %8s\n", "access (all live agents, random cells)", "cold us", "warm us");
    measure<0, 4>("none (mask load only)", a0, a1, arr, fl, fn, out, st);
    measure<1, 4>("RED.max, 4 B/cell (16.8 MB)", a0, a1, arr, fl, fn, out, st);
    measure<1, 8>("RED.max, 8 B/cell (33.5 MB)", a0, a1, arr, fl, fn, out, st);
    measure<1, 16>("RED.max, 16 B/cell (67 MB)", a0, a1, arr, fl, fn, out, st);
    measure<3, 4>("exch, 4 B/cell (16.8 MB)", a0, a1, arr, fl, fn, out, st);
    measure<3, 16>("exch, 16 B/cell (67 MB)", a0, a1, arr, fl, fn, out, st);
    measure<2, 2>("load 2 B, 2 B/cell (8.4 MB)", a0, a1, arr, fl, fn, out, st);
    measure<2, 4>("load 4 B, 4 B/cell (16.8 MB)", a0, a1, arr, fl, fn, out, st);
    measure<2, 8>("load 8 B, 8 B/cell (33.5 MB)", a0, a1, arr, fl, fn, out, st);
    measure<2, 16>("load 16 B, 16 B/cell (67 MB)", a0, a1, arr, fl, fn, out, st);
    measure<2, 16>("load 16 B + 34 KB dyn smem/CTA", a0, a1, arr, fl, fn, out, st, 34816);
    measure<2, 16>("load 16 B + 48 KB dyn smem/CTA", a0, a1, arr, fl, fn, out, st, 49152);
    measure<2, 17>("ld.cg 16 B", a0, a1, arr, fl, fn, out, st);
    measure<2, 17>("ld.cg 16 B + 34 KB dyn smem/CTA", a0, a1, arr, fl, fn, out, st, 34816);
    measure<3, 16>("exch 16 B + 34 KB dyn smem/CTA", a0, a1, arr, fl, fn, out, st, 34816);
    measure<1, 16>("RED 16 B + 34 KB dyn smem/CTA", a0, a1, arr, fl, fn, out, st, 34816);
    std::printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
