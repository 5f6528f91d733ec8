// ensemble.cu — batched ensemble of independent predation models (run_batch,
// src/batch.cpp:21-101; the paper's vmapped ensemble), one CTA per replica.
//
// A C1-sized replica (100x100 cells, 2 x 1024 slots) is small enough that its whole state
// stays ON CHIP for the entire run: agent columns live in REGISTERS (thread t owns slots
// t*SPT .. t*SPT+SPT-1 of both species for every step), the lattice and the per-cell lists
// live in shared memory, and HBM is touched only for the initial draw, the id column
// (written at births/deaths) and one metrics row per step. A step is three phases and three
// __syncthreads (B1-B3):
//   1 move + push onto packed per-cell lists (u32: sheep head | wolf head)     lifecycle.cpp:87-122
//   B1
//   2 every live agent resolves its own outcome by walking its cell's lists: a sheep's rank
//     among the cell's sheep decides the graze (rank 0) and whether it is eaten (rank < wolves
//     in the cell), a wolf's rank decides whether it eats (rank < sheep): the slot-sorted
//     pairing of predation.cpp:178-239 without a per-cell leader. Then eat / metabolise /
//     starve / reproduce (predation.cpp:241-250) and a scan of four packed 16-bit counters
//     (free/valid x sheep/wolves) whose warp totals are combined inside every warp
//   B2
//   3 compaction of the valid rows, clear of the lists
//   B3
//   4 free slots pull their rank-matched row (spawn_agents, lifecycle.cpp:144-195), metrics;
//     then phase 1 of the next step follows without a barrier.
// Regrow (predation.cpp:252-258) is lazy, as in the large-model engine: a grazed cell stores the
// step at whose end it is ready again (15 bits, renormalised every 8192 steps) and a ring of
// 256 due counters keeps the ready count, so no step sweeps the lattice.
// Per slot a thread keeps only cell, energy and one active bit: a dead slot's cell, energy and id
// are stale until a birth overwrites them (the dump masks them), and age is the birth step,
// stored only when a dump asks for it.
#include <climits>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "abmx_device.cuh"
#include "abmx_internal.h"
#include "ensemble.h"
#include "predation_engine.h"

using namespace abmx_dev;

namespace abmx_ens {

constexpr int kT = 512;
constexpr int kMaxSPT = 8;
constexpr unsigned kEnd = 0xFFFFu;
// grass word per cell (u16): a due step in [0, 0x7FFF], or one of
constexpr unsigned short kReady = 0x8000u;  // ready (full_grass, or regrown)
constexpr unsigned short kNever = 0x8001u;  // grazed with regrow_delay <= 0 (never regrows), or padding
constexpr int kRenorm = 8192;               // due steps older than this are folded into kReady
constexpr int kRecord = 6;                  // per-replica global words per slot index: 2 ids + 2 x 16-byte rows
// shared-memory layout: the fixed-size pieces first, then the cell words, grass words, list links
constexpr int kOffScan = 0;                   // warp totals of the step's scan
constexpr int kOffMisc = 8 * (kT / 32 + 2);   // grazed count, next ids + ready cells, stream keys
constexpr int kOffDue = kOffMisc + 96;        // [256] cells due per step
constexpr int kOffCw = kOffDue + 4 * 256;

__device__ __forceinline__ bool grass_ready(unsigned short gv, int t) {  // at a graze of step t
    return gv == kReady || (gv < 0x8000u && ((static_cast<unsigned>(t) - 1u - gv) & 0x7FFFu) < 0x4000u);
}


struct EnsParams {
    int W, H, C, Cpad;
    unsigned long long wdiv;  // ceil(2^40 / W)
    int N[2], n0[2], stride;
    double gain[2], metab, prob[2], frac;
    int delay;  // regrow_delay (<= 0: a grazed cell never regrows)
    long long steps;
    const unsigned long long* seeds;
    long long* ids;     // [count] records of kRecord * stride words: ids [2][stride], then rows
    double* metrics;    // [count][steps][4]
    // optional final-state dump
    uint8_t* d_active;  // [count][2][stride]
    int* d_cell;
    int* d_age;
    double* d_energy;
    unsigned short* d_g;  // [count][Cpad] grass words
    long long* d_next;  // [count][2]
    int* d_num;         // [count][2]
    struct Row {        // a valid row of the step: the child's energy and cell
        double e;
        unsigned c, pad;
    };
    int smem;  // dynamic shared memory bytes (layout())
};

__device__ __forceinline__ unsigned long long pack4(unsigned a, unsigned b, unsigned c, unsigned d) {
    return (static_cast<unsigned long long>(a) << 48) | (static_cast<unsigned long long>(b) << 32) |
           (static_cast<unsigned long long>(c) << 16) | d;
}
__device__ __forceinline__ unsigned f16(unsigned long long v, int k) {  // k = 0..3 from the top
    return static_cast<unsigned>((v >> (48 - 16 * k)) & 0xFFFFu);
}

// Block exclusive scan of four packed counters (16-bit fields of a u64, field 0 on top) with
// ONE barrier: the warp totals are published, then every warp scans them itself with shuffles
// (kThreads / 32 <= 32 warps). With at most kLane counts per lane and field, a warp's fields stay
// below 256 when kLane <= 4, so the warp-level part runs on 8-bit fields of a u32.
__device__ __forceinline__ unsigned long long widen8(unsigned x) {
    return (static_cast<unsigned long long>(x >> 24) << 48) | (static_cast<unsigned long long>((x >> 16) & 0xFFu) << 32) |
           (static_cast<unsigned long long>((x >> 8) & 0xFFu) << 16) | (x & 0xFFu);
}
template <int kThreads, int kLane>
__device__ __forceinline__ unsigned long long scan_1b(unsigned c0, unsigned c1, unsigned c2, unsigned c3,
                                                      unsigned long long* smem, unsigned long long* block_total) {
    constexpr int kWarps = kThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned long long incl, v;
    if constexpr (kLane <= 4) {
        const unsigned v32 = (c0 << 24) | (c1 << 16) | (c2 << 8) | c3;
        unsigned x = v32;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned n = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += n;
        }
        if (lane == 31) smem[warp] = widen8(x);
        v = 0;
        incl = widen8(x - v32);  // this lane's exclusive offset within the warp
    } else {
        v = pack4(c0, c1, c2, c3);
        incl = warp_incl_scan(v);
        if (lane == 31) smem[warp] = incl;
    }
    __syncthreads();
    unsigned long long w = lane < kWarps ? smem[lane] : 0ULL;
#pragma unroll
    for (int d = 1; d < kWarps; d <<= 1) {
        const unsigned long long n = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= d) w += n;
    }
    *block_total = __shfl_sync(0xffffffffu, w, kWarps - 1);
    const unsigned long long before = __shfl_sync(0xffffffffu, w, warp > 0 ? warp - 1 : 0);
    return (warp > 0 ? before : 0ULL) + incl - v;
}

template <int SPT>
__global__ void __launch_bounds__(kT, SPT <= 2 ? 3 : 1) k_ensemble(EnsParams P) {
    extern __shared__ __align__(16) unsigned char sm[];
    // fixed-size pieces and the cell words at constant offsets (immediates, not registers)
    unsigned long long* scan = reinterpret_cast<unsigned long long*>(sm + kOffScan);
    unsigned* misc = reinterpret_cast<unsigned*>(sm + kOffMisc);  // [1] grazed this step
    long long* ctr = reinterpret_cast<long long*>(sm + kOffMisc + 16);  // next_id[2], n_grass (thread 0)
    unsigned* due_cnt = reinterpret_cast<unsigned*>(sm + kOffDue);  // [256] cells due per step
    unsigned* cw = reinterpret_cast<unsigned*>(sm + kOffCw);
    unsigned short* g = reinterpret_cast<unsigned short*>(sm + kOffCw + 4 * P.Cpad);
    unsigned short* nxt = g + P.Cpad;  // [slot][species]: both species' list links of a slot

    const int r = blockIdx.x, tid = threadIdx.x;
    const unsigned long long seed = P.seeds[r];
    // A replica's global record: its id column, then the valid rows of the step (L1/L2-resident,
    // ordered by B3 like shared memory; keeping them out of SMEM lets three C1 replicas share an
    // SM). One base pointer serves both.
    long long* ids = P.ids + static_cast<size_t>(r) * kRecord * P.stride;
    EnsParams::Row* rows = reinterpret_cast<EnsParams::Row*>(ids + 2 * P.stride);
    auto bit = [](int s, int k) { return 1u << (s * SPT + k); };

    // ---- create_species (predation.cpp:22-33, lifecycle.cpp:53-85)
    unsigned act = 0;  // bit s*SPT+k: slot tid*SPT+k of species s is active
    int cell[2][SPT];
    double E[2][SPT];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const unsigned long long root = split(split(seed, s == 0 ? 20 : 21), 1);
        const unsigned long long kx = split(root, 0), ky = split(root, 1), ke = split(root, 2);
        const long long ehi = 2 * static_cast<long long>(P.gain[s]) + 1;
#pragma unroll
        for (int k = 0; k < SPT; ++k) {
            const int i = tid * SPT + k;
            cell[s][k] = 0;
            E[s][k] = 0.0;
            if (i < P.n0[s]) {
                act |= bit(s, k);
                const long long x = static_cast<long long>(__umul64hi(draw(kx, i), static_cast<unsigned long long>(P.W)));
                const long long y = static_cast<long long>(__umul64hi(draw(ky, i), static_cast<unsigned long long>(P.H)));
                const long long en = 1 + static_cast<long long>(__umul64hi(draw(ke, i), static_cast<unsigned long long>(ehi - 1)));
                cell[s][k] = static_cast<int>(y * P.W + x);
                E[s][k] = static_cast<double>(en);
            }
            if (i < P.N[s]) {
                ids[static_cast<size_t>(s) * P.stride + i] = i < P.n0[s] ? i : 0;
                if (P.d_age) P.d_age[(static_cast<size_t>(r) * 2 + s) * P.stride + i] = 0;  // birth step
            }
        }
    }
    for (int c = tid; c < P.Cpad; c += kT) g[c] = c < P.C ? kReady : kNever;
    for (int k = tid; k < 256; k += kT) due_cnt[k] = 0;
    for (int c = tid; c < P.C; c += kT) cw[c] = 0xFFFFFFFFu;
    if (tid == 0) {
        misc[1] = 0;
        ctr[0] = P.n0[0];  // next ids: thread 0 adds the step's births between B2 and B3
        ctr[1] = P.n0[1];
        ctr[2] = P.C;  // ready cells (full_grass)
    }
    // the four stream keys of a step (move, reproduce x sheep, wolves), derived by warp 0 into
    // SMEM: two splits per lane instead of six, lanes 0/1 the step roots, lanes 0..3 the keys
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(sm + kOffMisc + 48);
    if (tid == 0) {
        keys[4] = split(seed, 3);  // the move and reproduce roots
        keys[5] = split(seed, 4);
    }
    __syncwarp();
    auto derive_keys = [&](int t) {
        const unsigned ln = static_cast<unsigned>(tid) & 31u;
        const unsigned long long a = split(keys[4 + (ln & 1u)], static_cast<unsigned long long>(t));
        const unsigned long long mt = __shfl_sync(0xffffffffu, a, 0), rt = __shfl_sync(0xffffffffu, a, 1);
        const unsigned long long b = split(ln & 2u ? rt : mt, static_cast<unsigned long long>(ln & 1u));
        if (ln < 4) keys[ln] = b;  // mk[0], mk[1], rk[0], rk[1]
    };
    if (tid < 32) derive_keys(1);
    __syncthreads();

    for (int t = 1; t <= P.steps; ++t) {  // steps < 2^31 (run_smem)
        // ---- phase 1: move + push onto the per-cell lists
        const unsigned moved = act;  // the slots whose cell words are cleared in phase 3
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                if (!(act & bit(s, k))) continue;
                const int i = tid * SPT + k;
                const int u = static_cast<int>(draw(keys[s], static_cast<unsigned long long>(i)) >> 61);
                const int c = cell[s][k];
                // c / W by multiply-high: exact for c, W < 2^18 (smem_fits bounds C by 2^18)
                const int y = static_cast<int>((static_cast<unsigned long long>(c) * P.wdiv) >> 40);
                const int x = c - y * P.W;
                int nx = x + move_dx(u), ny = y + move_dy(u);
                nx = nx < 0 ? nx + P.W : (nx >= P.W ? nx - P.W : nx);
                ny = ny < 0 ? ny + P.H : (ny >= P.H ? ny - P.H : ny);
                const int nc = ny * P.W + nx;
                ABMX_ASSERT(nc >= 0 && nc < P.C && i < P.N[s]);
                cell[s][k] = nc;
                unsigned old = cw[nc];
                for (;;) {
                    const unsigned nv = s == 0 ? ((old & 0xFFFF0000u) | static_cast<unsigned>(i))
                                               : ((old & 0x0000FFFFu) | (static_cast<unsigned>(i) << 16));
                    const unsigned prev = atomicCAS(&cw[nc], old, nv);
                    if (prev == old) break;
                    old = prev;
                }
                nxt[2 * i + s] = static_cast<unsigned short>(s == 0 ? (old & 0xFFFFu) : (old >> 16));
            }
        __syncthreads();  // B1: the lists are complete
        // ---- phase 2: graze, pairing, eat / metabolise / starve / reproduce, one packed scan
        unsigned freeb = 0, validb = 0;
        unsigned cnt[2][2] = {{0, 0}, {0, 0}};  // [species][free, valid]
        double child[2][SPT];
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const int i = tid * SPT + k;
                child[s][k] = 0.0;
                bool alive = act & bit(s, k);
                if (alive) {
                    const int c = cell[s][k];
                    const unsigned head = cw[c];
                    const unsigned own = s == 0 ? (head & 0xFFFFu) : (head >> 16);
                    const unsigned other = s == 0 ? (head >> 16) : (head & 0xFFFFu);
                    // the rank matters only to a sheep on ready grass or an agent sharing its cell
                    // with the other species: most agents skip the walk
                    const bool ready = s == 0 && grass_ready(g[c], t);
                    int rank = 0;  // slots of this species in the cell below i
                    if (ready || other != kEnd)
                        for (unsigned v = own; v != kEnd; v = nxt[2 * v + s]) {
                        ABMX_ASSERT(v < static_cast<unsigned>(P.N[s]));
                        rank += v < static_cast<unsigned>(i);
                    }
                    if (ready && rank == 0) {  // the lowest sheep grazes
                        if (P.delay >= 1) {  // ready again at the end of step t + delay - 1
                            const unsigned due = static_cast<unsigned>(t + P.delay - 1) & 0x7FFFu;
                            g[c] = static_cast<unsigned short>(due);
                            atomicAdd(&due_cnt[due & 255u], 1u);
                        } else {
                            g[c] = kNever;
                        }
                        atomicAdd(&misc[1], 1u);
                        E[s][k] = __dadd_rn(E[s][k], P.gain[0]);
                    }
                    int n_other = 0;  // the p-th lowest sheep pairs with the p-th lowest wolf
                    for (unsigned v = other; v != kEnd && n_other <= rank; v = nxt[2 * v + 1 - s]) ++n_other;
                    if (rank < n_other) {
                        if (s == 0)
                            alive = false;  // eaten (predation.cpp:224-238)
                        else
                            E[s][k] = __dadd_rn(E[s][k], P.gain[1]);
                    }
                }
                if (alive) {
                    E[s][k] = __dsub_rn(E[s][k], P.metab);
                    if (E[s][k] <= 0.0) alive = false;
                }
                if (alive && E[s][k] > P.metab &&
                    uniform_double(keys[2 + s], static_cast<unsigned long long>(i)) < P.prob[s]) {
                    const double cE = __dmul_rn(floor(__dmul_rn(__dmul_rn(P.frac, E[s][k]), 1048576.0)), 0x1p-20);
                    E[s][k] = __dsub_rn(E[s][k], cE);
                    child[s][k] = cE;
                    validb |= bit(s, k);
                    ++cnt[s][1];
                }
                if (!alive) act &= ~bit(s, k);  // a dead slot's id reads as 0 (the dump masks it)
                if (!alive && i < P.N[s]) {
                    freeb |= bit(s, k);
                    ++cnt[s][0];
                }
            }
        unsigned long long total;
        const unsigned long long ex =
            scan_1b<kT, SPT>(cnt[0][0], cnt[0][1], cnt[1][0], cnt[1][1], scan, &total);  // B2
        // ---- phase 3: compaction of the valid rows; clear the cell words for the next step
        unsigned run[2][2] = {{f16(ex, 0), f16(ex, 1)}, {f16(ex, 2), f16(ex, 3)}};
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                if (moved & bit(s, k)) cw[cell[s][k]] = 0xFFFFFFFFu;
                if (validb & bit(s, k)) {
                    const unsigned v = run[s][1]++;
                    ABMX_ASSERT(v < static_cast<unsigned>(P.N[s]));
                    rows[s * P.stride + v].e = child[s][k];
                    rows[s * P.stride + v].c = static_cast<unsigned>(cell[s][k]);
                }
            }
        const int F[2] = {static_cast<int>(f16(total, 0)), static_cast<int>(f16(total, 2))};
        const int Q[2] = {static_cast<int>(f16(total, 1)), static_cast<int>(f16(total, 3))};
        if (tid < 32) derive_keys(t + 1);  // phase 2 has read this step's keys (B2)
        if (tid == 0) {  // phase 4 reads ctr[s] - pairs[s] as the first id of the step's births
            ctr[0] += F[0] < Q[0] ? F[0] : Q[0];
            ctr[1] += F[1] < Q[1] ? F[1] : Q[1];
        }
        __syncthreads();  // B3: rows written, cell words cleared
        // ---- phase 4: rank-matched births, regrow, metrics row
        int pairs[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            pairs[s] = F[s] < Q[s] ? F[s] : Q[s];
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                if (!(freeb & bit(s, k))) continue;
                const int f = static_cast<int>(run[s][0]++);
                if (f < pairs[s]) {
                    const int i = tid * SPT + k;
                    ABMX_ASSERT(f < P.N[s] && i < P.N[s] && rows[s * P.stride + f].c < static_cast<unsigned>(P.C));
                    act |= bit(s, k);
                    cell[s][k] = static_cast<int>(rows[s * P.stride + f].c);
                    E[s][k] = rows[s * P.stride + f].e;
                    ids[static_cast<size_t>(s) * P.stride + i] = ctr[s] - pairs[s] + f;
                    if (P.d_age) P.d_age[(static_cast<size_t>(r) * 2 + s) * P.stride + i] = static_cast<int>(t);
                }
            }
        }
        if (t % kRenorm == 0)  // due steps that have passed become kReady before they alias
            for (int c = tid; c < P.C; c += kT) {
                const unsigned short gv = g[c];
                if (gv < 0x8000u && ((static_cast<unsigned>(t) - gv) & 0x7FFFu) < 0x4000u) g[c] = kReady;
            }
        if (tid == 0) {
            // regrow of this step, lazily: - grazed + those due at its end (predation.cpp:252-258)
            const unsigned slot = static_cast<unsigned>(t) & 255u;
            const long long n_grass = ctr[2] + static_cast<long long>(due_cnt[slot]) - static_cast<long long>(misc[1]);
            ctr[2] = n_grass;
            due_cnt[slot] = 0;
            misc[1] = 0;
            double* row = P.metrics + (static_cast<size_t>(r) * P.steps + (t - 1)) * 4;
            row[0] = static_cast<double>(P.N[0] - F[0] + pairs[0]);
            row[1] = static_cast<double>(P.N[1] - F[1] + pairs[1]);
            row[2] = static_cast<double>(n_grass);
            row[3] = static_cast<double>((Q[0] - pairs[0]) + (Q[1] - pairs[1]));
            if (t == P.steps && P.d_num) {
                P.d_num[2 * r] = P.N[0] - F[0] + pairs[0];
                P.d_num[2 * r + 1] = P.N[1] - F[1] + pairs[1];
            }
        }
    }
    if (P.d_active) {  // inactive slots read as zeros; age = steps - birth step
#pragma unroll
        for (int s = 0; s < 2; ++s)
#pragma unroll
            for (int k = 0; k < SPT; ++k) {
                const int i = tid * SPT + k;
                if (i >= P.N[s]) continue;
                const size_t q = (static_cast<size_t>(r) * 2 + s) * P.stride + i;
                const bool a = act & bit(s, k);
                P.d_active[q] = a;
                P.d_cell[q] = a ? cell[s][k] : 0;
                P.d_age[q] = a ? static_cast<int>(P.steps - P.d_age[q]) : 0;
                P.d_energy[q] = a ? E[s][k] : 0.0;
                if (!a) ids[static_cast<size_t>(s) * P.stride + i] = 0;
            }
        for (int c = tid; c < P.Cpad; c += kT) P.d_g[static_cast<size_t>(r) * P.Cpad + c] = g[c];
        if (tid == 0) {
            P.d_next[2 * r] = ctr[0];
            P.d_next[2 * r + 1] = ctr[1];
        }
    }
}

static int layout(const abmx_predation_config& cfg, EnsParams& P) {
    const int N[2] = {cfg.sheep_capacity, cfg.wolf_capacity};
    int off = 0;
    auto take = [&](int bytes, int align) {
        off = (off + align - 1) / align * align;
        const int o = off;
        off += bytes;
        return o;
    };
    take(kOffCw, 16);  // scan, misc (grazed count, next ids + ready cells, stream keys), due counters
    take(4 * P.Cpad, 16);  // cell words
    take(2 * P.Cpad, 16);  // grass words
    take(4 * (N[0] > N[1] ? N[0] : N[1]), 16);  // list links, both species interleaved
    P.smem = (off + 15) / 16 * 16;
    return P.smem;
}

static int spt_for(const abmx_predation_config& cfg) {
    const int n = cfg.sheep_capacity > cfg.wolf_capacity ? cfg.sheep_capacity : cfg.wolf_capacity;
    for (int spt = 1; spt <= kMaxSPT; spt *= 2)
        if (n <= spt * kT) return spt;
    return 0;
}

bool smem_fits(const abmx_predation_config& cfg) {
    if (cfg.width < 1 || cfg.height < 1 || cfg.sheep_capacity < 0 || cfg.wolf_capacity < 0) return false;
    if (cfg.regrow_delay > 254) return false;
    const long long C = static_cast<long long>(cfg.width) * cfg.height;
    if (C > 65536LL * 4) return false;
    if (spt_for(cfg) == 0) return false;
    EnsParams P{};
    P.C = static_cast<int>(C);
    P.Cpad = static_cast<int>((C + 15) / 16 * 16);
    return layout(cfg, P) <= 227 * 1024;
}

#define CKE(x)                                                                        \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            abmx_internal::set_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
            rc = ABMX_E_CUDA;                                                         \
            goto done;                                                                \
        }                                                                             \
    } while (0)

int run_smem(const abmx_predation_config& cfg, const uint64_t* seeds, int count, long long steps,
             double* metrics_out, double* kernel_ms, Dump* dump) {
    if (const int rc = abmx_pred::check_create(cfg)) return rc;
    if (!smem_fits(cfg)) {
        abmx_internal::set_error("configuration does not fit the SMEM-resident ensemble kernel");
        return ABMX_E_DOMAIN;
    }
    if (steps > 0x7FFFFFFFLL) {  // the kernel counts steps in 32 bits, as the batched engine does
        abmx_internal::set_error("steps must be below 2^31");
        return ABMX_E_DOMAIN;
    }
    EnsParams P{};
    P.W = cfg.width;
    P.H = cfg.height;
    P.C = cfg.width * cfg.height;
    P.Cpad = (P.C + 15) / 16 * 16;
    P.wdiv = ((1ULL << 40) + static_cast<unsigned long long>(P.W) - 1) / static_cast<unsigned long long>(P.W);
    P.N[0] = cfg.sheep_capacity;
    P.N[1] = cfg.wolf_capacity;
    P.n0[0] = cfg.n_sheep0;
    P.n0[1] = cfg.n_wolves0;
    P.stride = ((P.N[0] > P.N[1] ? P.N[0] : P.N[1]) + 15) / 16 * 16;
    if (P.stride == 0) P.stride = 16;
    P.gain[0] = cfg.energy_gain_sheep;
    P.gain[1] = cfg.energy_gain_wolf;
    P.metab = cfg.metabolism;
    P.prob[0] = cfg.reproduce_prob_sheep;
    P.prob[1] = cfg.reproduce_prob_wolf;
    P.frac = cfg.reproduce_energy_frac;
    P.delay = cfg.regrow_delay >= 1 ? static_cast<int>(cfg.regrow_delay) : 0;
    P.steps = steps;
    layout(cfg, P);
    const int spt = spt_for(cfg);

    int rc = ABMX_OK;
    cudaStream_t st = nullptr;
    cudaEvent_t ea = nullptr, eb = nullptr;
    void* dseeds = nullptr;
    void* dids = nullptr;
    void* dmet = nullptr;
    void* ddump = nullptr;
    const size_t mbytes = sizeof(double) * 4 * static_cast<size_t>(count) * static_cast<size_t>(steps);
    const size_t ids_n = static_cast<size_t>(count) * 2 * P.stride;
    float ms = 0.f;
    CKE(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CKE(cudaEventCreate(&ea));
    CKE(cudaEventCreate(&eb));
    CKE(abmx_internal::malloc_async(&dseeds, sizeof(unsigned long long) * count, st));
    CKE(abmx_internal::malloc_async(&dids, ids_n * kRecord / 2 * 8, st));
    CKE(abmx_internal::malloc_async(&dmet, mbytes, st));
    CKE(cudaMemcpyAsync(dseeds, seeds, sizeof(unsigned long long) * count, cudaMemcpyHostToDevice, st));
    P.seeds = static_cast<const unsigned long long*>(dseeds);
    P.ids = static_cast<long long*>(dids);
    P.metrics = static_cast<double*>(dmet);
    if (dump) {
        const size_t n = ids_n;
        const size_t bytes = n * (1 + 4 + 4 + 8) + static_cast<size_t>(count) * 2 * P.Cpad + static_cast<size_t>(count) * 2 * (8 + 4) + 64;
        CKE(abmx_internal::malloc_async(&ddump, bytes, st));
        char* b = static_cast<char*>(ddump);
        P.d_energy = reinterpret_cast<double*>(b);
        b += n * 8;
        P.d_next = reinterpret_cast<long long*>(b);
        b += static_cast<size_t>(count) * 2 * 8;
        P.d_cell = reinterpret_cast<int*>(b);
        b += n * 4;
        P.d_age = reinterpret_cast<int*>(b);
        b += n * 4;
        P.d_num = reinterpret_cast<int*>(b);
        b += static_cast<size_t>(count) * 2 * 4;
        P.d_active = reinterpret_cast<uint8_t*>(b);
        b += n;
        P.d_g = reinterpret_cast<unsigned short*>(b);
    }
    {
        void (*kern)(EnsParams) = nullptr;
        switch (spt) {
            case 1: kern = k_ensemble<1>; break;
            case 2: kern = k_ensemble<2>; break;
            case 4: kern = k_ensemble<4>; break;
            default: kern = k_ensemble<8>; break;
        }
        CKE(abmx_internal::raise_dyn_smem(kern, static_cast<size_t>(P.smem)));
        CKE(cudaEventRecord(ea, st));
        (void)cudaGetLastError();
        kern<<<count, kT, P.smem, st>>>(P);
        abmx_internal::count_launch();
        CKE(cudaGetLastError());
        CKE(cudaEventRecord(eb, st));
    }
    if (metrics_out) CKE(cudaMemcpyAsync(metrics_out, dmet, mbytes, cudaMemcpyDeviceToHost, st));
    if (dump) {
        const int r = dump->replica;
        std::vector<uint8_t> a(P.stride);
        std::vector<unsigned short> gg(P.Cpad);
        std::vector<int> c(P.stride), ag(P.stride);
        long long nx[2];
        int nm[2];
        for (int s = 0; s < 2; ++s) {
            const size_t q = (static_cast<size_t>(r) * 2 + s) * P.stride;
            const size_t n = static_cast<size_t>(P.N[s]);
            if (n == 0) continue;
            CKE(cudaMemcpyAsync(a.data(), P.d_active + q, n, cudaMemcpyDeviceToHost, st));
            CKE(cudaMemcpyAsync(c.data(), P.d_cell + q, n * 4, cudaMemcpyDeviceToHost, st));
            CKE(cudaMemcpyAsync(ag.data(), P.d_age + q, n * 4, cudaMemcpyDeviceToHost, st));
            CKE(cudaMemcpyAsync(dump->energy[s], P.d_energy + q, n * 8, cudaMemcpyDeviceToHost, st));
            CKE(cudaMemcpyAsync(dump->ids[s], P.ids + (static_cast<size_t>(r) * kRecord + s) * P.stride, n * 8,
                                cudaMemcpyDeviceToHost, st));
            CKE(cudaStreamSynchronize(st));
            for (size_t i = 0; i < n; ++i) {
                dump->active[s][i] = a[i];
                dump->ages[s][i] = ag[i];
                dump->x[s][i] = c[i] % P.W;
                dump->y[s][i] = c[i] / P.W;
            }
        }
        CKE(cudaMemcpyAsync(nx, P.d_next + 2 * r, 16, cudaMemcpyDeviceToHost, st));
        CKE(cudaMemcpyAsync(nm, P.d_num + 2 * r, 8, cudaMemcpyDeviceToHost, st));
        CKE(cudaMemcpyAsync(gg.data(), P.d_g + static_cast<size_t>(r) * P.Cpad, 2 * static_cast<size_t>(P.Cpad),
                            cudaMemcpyDeviceToHost, st));
        CKE(cudaStreamSynchronize(st));
        for (int s = 0; s < 2; ++s) {
            dump->next_id[s] = nx[s];
            dump->num_active[s] = nm[s];
        }
        const unsigned T = static_cast<unsigned>(steps);
        for (int cc = 0; cc < P.C; ++cc) {  // the reference's (grass_ready, regrow) after step T
            const unsigned short gv = gg[cc];
            const bool ready = gv == kReady || (gv < 0x8000u && ((T - gv) & 0x7FFFu) < 0x4000u);
            dump->grass_ready[cc] = ready;
            dump->regrow[cc] = ready ? 0
                                     : (gv == kNever ? (cfg.regrow_delay <= 0 ? cfg.regrow_delay : 0)
                                                     : static_cast<int64_t>((gv - T) & 0x7FFFu));
        }
    }
    CKE(cudaStreamSynchronize(st));
    CKE(cudaEventElapsedTime(&ms, ea, eb));
    if (kernel_ms) *kernel_ms = ms;
done:
    if (st) {
        if (dseeds) cudaFreeAsync(dseeds, st);
        if (dids) cudaFreeAsync(dids, st);
        if (dmet) cudaFreeAsync(dmet, st);
        if (ddump) cudaFreeAsync(ddump, st);
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
    }
    if (ea) cudaEventDestroy(ea);
    if (eb) cudaEventDestroy(eb);
    return rc;
}

}  // namespace abmx_ens
