// Memory skeleton of a PERSISTENT, SMEM-staged C2 predation step: each CTA
// stages its tiles' columns with cp.async.bulk (TMA bulk copies) into shared memory, moves the
// agents and posts the cell-word atomics, passes ONE grid barrier, reads the cell words back
// and writes the tiles out with bulk stores. No model logic; C2 shapes (1M slots, ~370k live
// sheep, ~35k live wolves packed low, 4.19M cells of 16 B). Cold (L2 flushed) and warm.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fused_skeleton tools/fused_skeleton.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

constexpr int kT = 256, kS = 4, kTile = kT * kS;
constexpr unsigned kN = 524288u;
constexpr unsigned kCells = 2048u * 2048u;
constexpr unsigned kWolfLive = 45000u;
constexpr int kTileBytes = kTile * (1 + 4 + 4 + 8);

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ unsigned sa(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

struct Buf {
    uint8_t* act[2];
    int* cell[2];
    int* age[2];
    double* E[2];
    int* next[2];
    uint8_t* tile_live;  // [2][512]
    uint4* cw;
    unsigned long long* bar;
    int* out;
};

#ifndef BACKOFF
#define BACKOFF 0
#endif
constexpr unsigned kBackoff = BACKOFF;
__device__ __forceinline__ void grid_sync(unsigned long long* ctr, unsigned long long target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned long long v;
        long long spins = 0;
        for (;;) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(ctr) : "memory");
            if (v >= target || ++spins >= (1LL << 22)) break;
            __nanosleep(kBackoff);
        }
    }
    __syncthreads();
}

// mode 0: staging + barrier + write-back only; 1: + move, exch/live + max/sheep, next[], random
// 16 B read/live; 2: as 1 with RED.max only for sheep (exch for wolves)
template <int kTpc, int kMode>
__global__ void __launch_bounds__(kT, kTpc == 1 ? 7 : 4) k_fused(Buf B, unsigned salt, unsigned long long target) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) unsigned long long mbar;
    const int tiles_per_species = kN / kTile;
    int s_[kTpc], t_[kTpc];
    bool live_[kTpc];
    for (int j = 0; j < kTpc; ++j) {
        const int g = blockIdx.x * kTpc + j;
        s_[j] = g >= tiles_per_species;
        t_[j] = g - s_[j] * tiles_per_species;
        live_[j] = B.tile_live[g];
    }
    auto tile_act = [&](int j) { return reinterpret_cast<uint8_t*>(sm + j * kTileBytes); };
    auto tile_cell = [&](int j) { return reinterpret_cast<int*>(sm + j * kTileBytes + kTile); };
    auto tile_age = [&](int j) { return reinterpret_cast<int*>(sm + j * kTileBytes + 5 * kTile); };
    auto tile_E = [&](int j) { return reinterpret_cast<double*>(sm + j * kTileBytes + 9 * kTile); };
    if (kMode == 4) {
        grid_sync(B.bar, target);
        return;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
        unsigned bytes = 0;
        for (int j = 0; j < kTpc; ++j) bytes += live_[j] ? kTileBytes : 0;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&mbar)), "r"(bytes));
        for (int j = 0; j < kTpc; ++j) {
            if (!live_[j]) continue;
            const size_t o = static_cast<size_t>(t_[j]) * kTile;
            const int s = s_[j];
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(tile_act(j))),
                         "l"(B.act[s] + o), "r"(kTile), "r"(sa(&mbar)) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(tile_cell(j))),
                         "l"(B.cell[s] + o), "r"(4 * kTile), "r"(sa(&mbar)) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(tile_age(j))),
                         "l"(B.age[s] + o), "r"(4 * kTile), "r"(sa(&mbar)) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(sa(tile_E(j))),
                         "l"(B.E[s] + o), "r"(8 * kTile), "r"(sa(&mbar)) : "memory");
        }
    }
    __syncthreads();
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT_%=;\n }" ::"r"(sa(&mbar))
        : "memory");
    // ---- phase A: move + atomics
    if (kMode == 1 || kMode == 2 || kMode == 5 || kMode == 6) {
        unsigned* w = reinterpret_cast<unsigned*>(B.cw);
#pragma unroll
        for (int j = 0; j < kTpc; ++j) {
            if (!live_[j]) continue;
            const int s = s_[j];
            const int i0 = threadIdx.x * kS;
            const uint32_t aw = *reinterpret_cast<const uint32_t*>(tile_act(j) + i0);
            int4 c = *reinterpret_cast<const int4*>(tile_cell(j) + i0);
            int4 a = *reinterpret_cast<const int4*>(tile_age(j) + i0);
            int cell[kS] = {c.x, c.y, c.z, c.w};
            bool act[kS];
            for (int k = 0; k < kS; ++k) {
                act[k] = (aw >> (8 * k)) & 0xFF;
                if (act[k]) cell[k] = static_cast<int>((cell[k] + 2049u + salt) % kCells);
            }
            a.x += act[0]; a.y += act[1]; a.z += act[2]; a.w += act[3];
            unsigned old[kS];
            const bool exch = kMode == 1 || (s == 1 && kMode == 2);
            const unsigned gslot = t_[j] * kTile + i0;
            if (exch)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) old[k] = atomicExch(&w[4 * cell[k] + s], salt + gslot + k);
            if (s == 0 || kMode >= 5)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) asm volatile("red.relaxed.gpu.global.max.u32 [%0], %1;" ::"l"(&w[4 * cell[k] + 2 + s]), "r"(salt ^ (gslot + k)) : "memory");
            *reinterpret_cast<int4*>(tile_cell(j) + i0) = make_int4(cell[0], cell[1], cell[2], cell[3]);
            *reinterpret_cast<int4*>(tile_age(j) + i0) = a;
            if (exch)
                for (int k = 0; k < kS; ++k)
                    if (act[k]) B.next[s][gslot + k] = static_cast<int>(old[k]);
        }
    }
    if (kMode != 3) grid_sync(B.bar, target);
    // ---- phase B: cell-word reads + energy update
    if (kMode == 1 || kMode == 2 || kMode == 6) {
#pragma unroll
        for (int j = 0; j < kTpc; ++j) {
            if (!live_[j]) continue;
            const int i0 = threadIdx.x * kS;
            const uint32_t aw = *reinterpret_cast<const uint32_t*>(tile_act(j) + i0);
            const int4 c = *reinterpret_cast<const int4*>(tile_cell(j) + i0);
            const int cell[kS] = {c.x, c.y, c.z, c.w};
            uint4 v[kS];
            for (int k = 0; k < kS; ++k)
                if ((aw >> (8 * k)) & 0xFF) v[k] = B.cw[cell[k]];
            double2* E = reinterpret_cast<double2*>(tile_E(j) + i0);
            double2 e0 = E[0], e1 = E[1];
            if (aw & 0xFF) e0.x -= 1.0 + (v[0].x & 1);
            if (aw & 0xFF00) e0.y -= 1.0 + (v[1].x & 1);
            if (aw & 0xFF0000) e1.x -= 1.0 + (v[2].x & 1);
            if (aw & 0xFF000000) e1.y -= 1.0 + (v[3].x & 1);
            E[0] = e0;
            E[1] = e1;
        }
    }
    // ---- write back (bulk stores)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int j = 0; j < kTpc; ++j) {
            if (!live_[j]) continue;
            const size_t o = static_cast<size_t>(t_[j]) * kTile;
            const int s = s_[j];
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(B.act[s] + o), "r"(sa(tile_act(j))), "r"(kTile) : "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(B.cell[s] + o), "r"(sa(tile_cell(j))), "r"(4 * kTile) : "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(B.age[s] + o), "r"(sa(tile_age(j))), "r"(4 * kTile) : "memory");
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(B.E[s] + o), "r"(sa(tile_E(j))), "r"(8 * kTile) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
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
        if (i % kTile == 0) B.tile_live[s * (kN / kTile) + i / kTile] = s == 0 || i < kWolfLive;
    }
}
__global__ void k_empty() {}
__global__ void k_spin(long long ns) {
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    do { asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); } while (t - t0 < (unsigned long long)ns);
}

template <int kTpc, int kMode>
float run(Buf B, uint4* fl, size_t flush_n, cudaStream_t st, bool cold, unsigned long long& target) {
    const int grid = 2 * kN / kTile / kTpc;
    const size_t smem = static_cast<size_t>(kTpc) * kTileBytes;
    cudaFuncSetAttribute(k_fused<kTpc, kMode>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_fused<kTpc, kMode>, kT, smem);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int reps = 20;
    float sum = 0.f;
    for (int r = 0; r < reps + 3; ++r) {
        if (cold) {
            k_flush<<<148 * 4, 256, 0, st>>>(fl, flush_n, r);
            k_stream_read<<<148 * 4, 256, 0, st>>>(fl + flush_n, flush_n, B.out);
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(kT);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (kMode != 3) target += grid;
        if (!cold) k_spin<<<1, 32, 0, st>>>(20000);
        cudaEventRecord(a, st);
        cudaError_t e = cudaLaunchKernelEx(&cfg, k_fused<kTpc, kMode>, B, 1000u + r, target);
        cudaEventRecord(b, st);
        cudaEventSynchronize(b);
        if (e != cudaSuccess) {
            std::printf("launch error %s (occ %d grid %d)\n", cudaGetErrorString(e), occ, grid);
            return -1.f;
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) sum += ms;
    }
    return sum / reps * 1e3f;
}

int main(int argc, char** argv) {
    setvbuf(stdout, nullptr, _IONBF, 0);
    const int only = argc > 1 ? atoi(argv[1]) : -1;
    int idx = 0;
    Buf B{};
    for (int s = 0; s < 2; ++s) {
        cudaMalloc(&B.act[s], kN);
        cudaMalloc(&B.cell[s], kN * 4);
        cudaMalloc(&B.age[s], kN * 4);
        cudaMalloc(&B.E[s], kN * 8);
        cudaMalloc(&B.next[s], kN * 4);
    }
    cudaMalloc(&B.tile_live, 2 * kN / kTile);
    cudaMalloc(&B.cw, (size_t)kCells * 16);
    cudaMalloc(&B.bar, 8);
    cudaMalloc(&B.out, 64);
    cudaMemset(B.bar, 0, 8);
    cudaMemset(B.cw, 0, (size_t)kCells * 16);
    k_init<<<148 * 8, 256>>>(B);
    uint4* fl;
    const size_t flush_n = (256u << 20) / 16;
    cudaMalloc(&fl, 2 * flush_n * 16);
    cudaStream_t st;
    cudaStreamCreate(&st);
    unsigned long long target = 0;
    {  // empty launch floor
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e9f;
        for (int r = 0; r < 20; ++r) {
            k_spin<<<1, 32, 0, st>>>(20000);
            cudaEventRecord(a, st);
            k_empty<<<512, 256, 0, st>>>();
            cudaEventRecord(b, st);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        std::printf("empty launch 512 CTAs (events): %.2f us\n", best * 1e3f);
        for (int variant = 0; variant < 3; ++variant) {
            best = 1e9f;
            for (int r = 0; r < 20; ++r) {
                k_spin<<<1, 32, 0, st>>>(20000);
                cudaEventRecord(a, st);
                if (variant == 0) k_empty<<<1, 32, 0, st>>>();
                if (variant == 1) { k_empty<<<512, 256, 0, st>>>(); k_empty<<<512, 256, 0, st>>>(); }
                cudaEventRecord(b, st);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            std::printf("%s: %.2f us\n", variant == 0 ? "empty launch 1 CTA" : variant == 1 ? "2 empty launches 512 CTAs" : "events only", best * 1e3f);
        }
    }
    std::printf("%-60s %8s %8s\n", "variant", "cold us", "warm us");
#define RUN(TPC, M, NAME)                                                                                  \
    if (only < 0 || only == idx++) {                                                                       \
        float c = run<TPC, M>(B, fl, flush_n, st, true, target);                                           \
        float w = run<TPC, M>(B, fl, flush_n, st, false, target);                                          \
        std::printf("%-60s %8.2f %8.2f\n", NAME, c, w);                                                    \
    }
    RUN(2, 4, "tpc2: grid barrier only (cooperative launch)")
    RUN(2, 3, "tpc2: TMA stage + bulk store, no barrier")
    RUN(2, 0, "tpc2: TMA stage + grid barrier + bulk store")
    RUN(2, 1, "tpc2: + move, exch/live + max/sheep, next[], 16B read/live")
    RUN(2, 2, "tpc2: + move, RED.max/sheep + exch/wolf, 16B read/live")
    RUN(4, 1, "tpc4: + move, exch/live + max/sheep, next[], 16B read/live")
    RUN(1, 1, "tpc1: + move, exch/live + max/sheep, next[], 16B read/live")
    RUN(2, 5, "tpc2: + move, RED.max/live, no reads")
    RUN(2, 6, "tpc2: + move, RED.max/live, 16B read/live")
    std::printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
    return 0;
}
