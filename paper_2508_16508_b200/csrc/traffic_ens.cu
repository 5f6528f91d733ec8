// traffic_ens.cu — run_batch of TrafficModel for many short roads (C4 roads variant: 3496 roads
// x L=100, 1000 steps): ONE CTA per road with the whole road resident in shared memory for all
// steps; HBM sees only the metrics rows. Same step as traffic.cu (propose + bid, acceptance as
// the suffix composition of 3-lane column maps, mover-written occupancy, spawn), bit-exact with
// src/models/traffic.cpp:47-238.
//
// Shared memory per road (C = 3L slots = cells): bid u32[C] (min of prio<<16 | slot), occupancy
// i16[C], proposal i16[C], position i16[C], accepted u8[C], active u8[C], lane u8[C], target lane
// u8[C]: 16 bytes x C. Lanes are stored, never divided out of cell indices.
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/abmx_cuda.h"
#include "abmx_device.cuh"
#include "abmx_internal.h"

using namespace abmx_dev;

namespace abmx_trfe {

constexpr unsigned kNoBid = 0xFFFFFFFFu;
constexpr int kStay = -1, kExit = -2;
constexpr unsigned kIdentityFn = 2u | (3u << 3) | (4u << 6);

struct EnsP {
    int L, C;
    long long period, green_len, steps;
    const unsigned long long* seeds;  // [roads]
    const long long* phase;           // [roads]
    double* metrics;                  // [roads][steps][4]
};

__device__ __forceinline__ unsigned mode_of(unsigned f, int l) { return (f >> (3 * l)) & 7u; }
__device__ __forceinline__ unsigned compose(unsigned f, unsigned g) {  // f ∘ g
    unsigned h = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const unsigned m = mode_of(f, l);
        h |= (m < 2 ? m : mode_of(g, static_cast<int>(m) - 2)) << (3 * l);
    }
    return h;
}
__device__ __forceinline__ unsigned apply_fn(unsigned f, unsigned v) {
    unsigned out = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const unsigned m = mode_of(f, l);
        out |= (m < 2 ? m : (v >> (m - 2)) & 1u) << l;
    }
    return out;
}

struct Road {
    unsigned* bid;
    short* occ;
    short* X;
    short* pos;
    uint8_t* acc;
    uint8_t* act;
    uint8_t* lane;  // lane of the car in slot i
    uint8_t* tl;    // target lane of its move proposal
};

// the column map of column c (see traffic.cu k_accept); m3 = occupied lanes
__device__ __forceinline__ unsigned column_map(const Road& R, int L, int c, unsigned& m3) {
    unsigned f = 0;
    m3 = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        unsigned m = 0;
        const int o = R.occ[l * L + c];
        if (o >= 0) {
            m3 |= 1u << l;
            const int X = R.X[o];
            if (X == kExit) {
                m = 1;
            } else if (X >= 0 && R.bid[X] != kNoBid && static_cast<int>(R.bid[X] & 0xFFFFu) == o) {
                m = R.occ[X] < 0 ? 1u : 2u + static_cast<unsigned>(R.tl[o]);
            }
        }
        f |= m << (3 * l);
    }
    return f;
}

template <int kNT>
__global__ void __launch_bounds__(kNT, 1536 / kNT) k_traffic_ens(EnsP P) {  // 24 roads of 64 threads per SM: C4 roads in one wave
    extern __shared__ unsigned char sm[];
    const int L = P.L, C = P.C;
    Road R;
    R.bid = reinterpret_cast<unsigned*>(sm);
    R.occ = reinterpret_cast<short*>(R.bid + C);
    R.X = R.occ + C;
    R.pos = R.X + C;
    R.acc = reinterpret_cast<uint8_t*>(R.pos + C);
    R.act = R.acc + C;
    R.lane = R.act + C;
    R.tl = R.lane + C;
    __shared__ unsigned s_warp[kNT / 32];
    __shared__ int s_exited;
    __shared__ long long s_active;
    const int road = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long seed = P.seeds[road];
    const long long phase = P.phase[road];
    for (int x = tid; x < C; x += kNT) {  // Road::empty (traffic.cpp:19-29)
        R.occ[x] = -1;
        R.act[x] = 0;
        R.pos[x] = 0;
        R.acc[x] = 0;
        R.lane[x] = 0;
    }
    if (tid == 0) {
        s_active = 0;
        s_exited = 0;
    }
    const int nc = (L + kNT - 1) / kNT;  // columns per thread in the acceptance scan
    // SignalSchedule::green(t) = ((t + phase) mod period) < green_len, advanced incrementally
    long long gm = ((1 + phase) % P.period + P.period) % P.period;
    __syncthreads();
    // per-road stream roots (TrafficPropose = 6, TrafficSpawn = 7); each step's two keys are
    // derived once per warp (lane 0 propose, lane 1 spawn) and shuffled out
    const unsigned long long root6 = split(seed, 6), root7 = split(seed, 7);
    for (long long t = 1; t <= P.steps; ++t, gm = gm + 1 == P.period ? 0 : gm + 1) {
        const bool green = gm < P.green_len;
        const unsigned long long kk = split(lane & 1 ? root7 : root6, static_cast<unsigned long long>(t));
        const unsigned long long kp = __shfl_sync(0xffffffffu, kk, 0);
        const unsigned long long ks_step = __shfl_sync(0xffffffffu, kk, 1);
        // (a) propose (traffic.cpp:47-80) and bid for the target cell (priority, then slot)
        for (int x = tid; x < C; x += kNT) R.bid[x] = kNoBid;
        __syncthreads();
        for (int i = tid; i < C; i += kNT) {
            if (!R.act[i]) continue;
            const int p = R.pos[i];
            const int lane_i = R.lane[i], cell = p - lane_i * L;
            int X;
            if (cell == L - 1) {
                X = green ? kExit : kStay;
            } else {
                const int n = 1 + (lane_i > 0) + (lane_i < 2);
                const int pick = static_cast<int>(uniform_span(kp, static_cast<unsigned long long>(i),
                                                               static_cast<unsigned long long>(n)));
                const int tl = pick == 0 ? lane_i : (pick == 1 ? (lane_i > 0 ? lane_i - 1 : lane_i + 1) : lane_i + 1);
                X = tl * L + cell + 1;
                R.tl[i] = static_cast<uint8_t>(tl);
                const int prio = lane_i == tl ? 0 : (lane_i == tl - 1 ? 1 : 2);
                atomicMin(&R.bid[X], (static_cast<unsigned>(prio) << 16) | static_cast<unsigned>(i));
            }
            R.X[i] = static_cast<short>(X);
        }
        __syncthreads();
        // (b) acceptance: suffix composition of the column maps (thread 0 holds the last columns)
        const int c_hi = L - tid * nc;
        unsigned T = kIdentityFn;
        // a thread's column maps, kept from the composition for the apply pass (nc <= kCache)
        constexpr int kCache = 4;
        unsigned fcache[kCache], mcache[kCache];
        {
            int j = 0;
            for (int c = c_hi - 1; c >= c_hi - nc && c >= 0; --c, ++j) {
                unsigned m3;
                const unsigned f = column_map(R, L, c, m3);
                if (nc <= kCache) {
#pragma unroll
                    for (int q = 0; q < kCache; ++q)
                        if (q == j) {
                            fcache[q] = f;
                            mcache[q] = m3;
                        }
                }
                T = compose(f, T);
            }
        }
        unsigned I = T;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned o = __shfl_up_sync(0xffffffffu, I, d);
            if (lane >= d) I = compose(I, o);
        }
        if (lane == 31) s_warp[warp] = I;
        __syncthreads();
        unsigned wex = kIdentityFn;
        for (int w = 0; w < warp; ++w) wex = compose(s_warp[w], wex);
        const unsigned up = __shfl_up_sync(0xffffffffu, I, 1);
        unsigned v = apply_fn(lane > 0 ? compose(up, wex) : wex, 0u);
        int j = 0;
        for (int c = c_hi - 1; c >= c_hi - nc && c >= 0; --c, ++j) {
            unsigned m3, f = 0;
            if (nc <= kCache) {
#pragma unroll
                for (int q = 0; q < kCache; ++q)
                    if (q == j) {
                        f = fcache[q];
                        m3 = mcache[q];
                    }
            } else {
                f = column_map(R, L, c, m3);
            }
            v = apply_fn(f, v);
#pragma unroll
            for (int l = 0; l < 3; ++l)
                if (m3 & (1u << l)) R.acc[l * L + c] = static_cast<uint8_t>((v >> l) & 1u);
        }
        __syncthreads();
        // (c) accepted moves and exits; movers write their new cell, vacated cells are cleared
        // unless an accepted winner enters them
        for (int i = tid; i < C; i += kNT) {
            if (!R.act[i]) continue;
            const int p = R.pos[i];
            if (!R.acc[p]) continue;
            const int X = R.X[i];
            const int lp = R.lane[i];
            if (X == kExit) {
                R.act[i] = 0;
                R.pos[i] = 0;
                R.lane[i] = 0;
                atomicAdd(&s_exited, 1);
            } else {
                R.pos[i] = static_cast<short>(X);
                R.lane[i] = R.tl[i];
                R.occ[X] = static_cast<short>(i);
            }
            const unsigned w = R.bid[p];
            bool keep = false;
            if (w != kNoBid) {
                const int prio = static_cast<int>(w >> 16);
                const int src = (prio == 0 ? lp : (prio == 1 ? lp - 1 : lp + 1)) * L + (p - lp * L) - 1;
                keep = R.acc[src] != 0;
            }
            if (!keep) R.occ[p] = -1;
        }
        __syncthreads();
        // (d) spawn_cars (traffic.cpp:143-184) into the lowest free slots; metrics row
        if (warp == 0) {
            const unsigned long long ks = ks_step;
            const int k = static_cast<int>(uniform_span(ks, 0, 4));
            int lanes[3] = {0, 1, 2};
            for (int i = 0; i < (k < 2 ? k : 2); ++i) {
                const int j = i + static_cast<int>(uniform_span(ks, static_cast<unsigned long long>(1 + i),
                                                                static_cast<unsigned long long>(3 - i)));
                const int tmp = lanes[i];
                lanes[i] = lanes[j];
                lanes[j] = tmp;
            }
            int rows[3];
            int nv = 0;
            for (int q = 0; q < (k < 3 ? k : 3); ++q)
                if (R.occ[lanes[q] * L] < 0) rows[nv++] = lanes[q];
            int spawned = 0;
            for (int base = 0; base < C && spawned < nv; base += 32) {
                const int i = base + lane;
                unsigned fm = __ballot_sync(0xffffffffu, i < C && !R.act[i]);
                while (fm && spawned < nv) {
                    const int s = base + __ffs(fm) - 1;
                    fm &= fm - 1;
                    if (lane == 0) {
                        R.act[s] = 1;
                        R.lane[s] = static_cast<uint8_t>(rows[spawned]);
                        R.pos[s] = static_cast<short>(rows[spawned] * L);
                        R.occ[rows[spawned] * L] = static_cast<short>(s);
                    }
                    ++spawned;
                }
            }
            if (lane == 0) {
                const int exited = s_exited;
                s_active += spawned - exited;
                double* row = P.metrics + (static_cast<size_t>(road) * P.steps + (t - 1)) * 4;
                row[0] = static_cast<double>(s_active);
                row[1] = static_cast<double>(spawned);
                row[2] = static_cast<double>(exited);
                row[3] = green ? 1.0 : 0.0;
                s_exited = 0;
            }
        }
        __syncthreads();
    }
}

}  // namespace abmx_trfe

namespace abmx_internal {

size_t traffic_ens_smem(long long length) { return static_cast<size_t>(16) * 3 * static_cast<size_t>(length); }

bool traffic_ens_fits(const abmx_traffic_config& cfg) {
    return cfg.length >= 1 && 3 * cfg.length <= 32767 && traffic_ens_smem(cfg.length) <= 160 * 1024;
}

// run_batch of TrafficModel on the SMEM path; metrics_out host [count][steps][4]
int traffic_ensemble_run(const abmx_traffic_config& cfg, const uint64_t* seeds, int count, long long steps,
                         double* metrics_out, double* kernel_ms) {
    using namespace abmx_trfe;
    const size_t smem = traffic_ens_smem(cfg.length);
    long long gl = llround(static_cast<double>(cfg.period) * cfg.green_fraction);
    EnsP P{};
    P.L = static_cast<int>(cfg.length);
    P.C = 3 * P.L;
    P.period = cfg.period;
    P.green_len = gl < 0 ? 0 : (gl > cfg.period ? cfg.period : gl);
    P.steps = steps;
    std::vector<long long> ph(static_cast<size_t>(count));
    for (int r = 0; r < count; ++r)
        ph[static_cast<size_t>(r)] = static_cast<long long>(static_cast<unsigned long long>(
            (static_cast<unsigned __int128>(draw(split(seeds[r], 5), 0)) * static_cast<unsigned long long>(cfg.period)) >> 64));
    // 64 threads for short roads (more CTAs per SM, cheaper barriers), 128 otherwise
    const int nt = cfg.length <= 256 ? 64 : 128;
    const void* kfn = nt == 64 ? reinterpret_cast<const void*>(k_traffic_ens<64>)
                               : reinterpret_cast<const void*>(k_traffic_ens<128>);
    cudaStream_t s;
    cudaError_t e = cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        set_error(std::string("stream: ") + cudaGetErrorString(e));
        return ABMX_E_CUDA;
    }
    unsigned long long* d_seeds = nullptr;
    long long* d_phase = nullptr;
    double* d_metrics = nullptr;
    const size_t mb = static_cast<size_t>(count) * static_cast<size_t>(steps) * 32;
    int rc = ABMX_OK;
    cudaEvent_t a = nullptr, b = nullptr;
    if ((e = abmx_internal::malloc_async(&d_seeds, static_cast<size_t>(count) * 8, s)) != cudaSuccess ||
        (e = abmx_internal::malloc_async(&d_phase, static_cast<size_t>(count) * 8, s)) != cudaSuccess ||
        (e = abmx_internal::malloc_async(&d_metrics, mb, s)) != cudaSuccess ||
        (e = abmx_internal::raise_dyn_smem(kfn, static_cast<size_t>(smem))) !=
            cudaSuccess) {
        set_error(std::string("traffic ensemble: ") + cudaGetErrorString(e));
        rc = ABMX_E_CUDA;
    } else {
        cudaMemcpyAsync(d_seeds, seeds, static_cast<size_t>(count) * 8, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_phase, ph.data(), ph.size() * 8, cudaMemcpyHostToDevice, s);
        P.seeds = d_seeds;
        P.phase = d_phase;
        P.metrics = d_metrics;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        (void)cudaGetLastError();
        cudaEventRecord(a, s);
        void* args[1] = {&P};
        cudaLaunchKernel(kfn, dim3(static_cast<unsigned>(count)), dim3(static_cast<unsigned>(nt)), args, smem, s);
        cudaEventRecord(b, s);
        count_launch();
        if ((e = cudaGetLastError()) == cudaSuccess && metrics_out)
            e = cudaMemcpyAsync(metrics_out, d_metrics, mb, cudaMemcpyDeviceToHost, s);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s);
        if (e != cudaSuccess) {
            set_error(std::string("traffic ensemble: ") + cudaGetErrorString(e));
            rc = ABMX_E_CUDA;
        } else if (kernel_ms) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, a, b);
            *kernel_ms = ms;
        }
    }
    if (a) cudaEventDestroy(a);
    if (b) cudaEventDestroy(b);
    cudaFreeAsync(d_seeds, s);
    cudaFreeAsync(d_phase, s);
    cudaFreeAsync(d_metrics, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return rc;
}

}  // namespace abmx_internal
