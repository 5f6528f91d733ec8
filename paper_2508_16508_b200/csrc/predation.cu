// predation.cu — the predation step (src/models/predation.cpp:167-263) on sm_100a for R
// replicas at once, device-resident SoA state, bit-exact with the reference.
//
// A step is TWO kernels (three on crowded grids), captured once in a CUDA graph:
//   k_move    (a) births of the previous step: the k-th free slot (ascending) receives the
//                 k-th valid parent row (rank-match, lifecycle.cpp:144-195), ranks from one
//                 block scan of the active mask + the per-tile counts published by k_update;
//             (b) step_agents with the move transition (predation.cpp:35-49,
//                 lifecycle.cpp:87-122), then every live agent pushes itself onto its new
//                 cell's list (atomicExch) and sheep post their slot to the cell's
//                 lowest-slot word (atomicMax, fire-and-forget).
//   [k_cells] crowded grids only (capacity > cells): sort-based k-th wolf <-> k-th sheep
//             pairing per wolf cell (predation.cpp:197-239) -> flags.
//   k_update  graze (lowest sheep slot of a ready cell), predation (sparse grids: each agent
//             of a wolf-and-sheep cell walks the cell's two short lists for its slot rank),
//             metabolise, starve, reproduce (predation.cpp:178-250); valid parent rows are
//             compacted tile-locally and every tile publishes its (free, valid) counts.
// The births of the last step are applied by k_finalize (k_move without the move) whenever
// the host needs the state (export, metrics, end of a run).
//
// HBM layout (per species, per replica, stride Npad): active u8, cell i32 (= y*W + x),
// age i32, energy f64, id i64; the agent type is implied by the species. Per cell one uint4
// (list heads, lowest sheep slot, grass due epoch — see "per-cell words").
#include <atomic>
#include <chrono>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/abmx_cuda.h"
#include "abmx_device.cuh"
#include "abmx_internal.h"
#include "predation_engine.h"

using namespace abmx_dev;

namespace abmx_pred {

// neighbour order of the move draw (predation.cpp:13-15): move_dx / move_dy, abmx_device.cuh

// Checked builds (-DABMX_CHECKED, tools/build_variant.sh checked "-DABMX_CHECKED"): every index
// into the slot columns, the cell words and the list links is bounds-checked on the device; the
// first failing check id is kept in g_check_fail (abmx_predation_check_status). compute-sanitizer
// is closed on this GPU pool, so this is the out-of-bounds net of tools/sanitize_smoke.py.
#ifdef ABMX_CHECKED
__device__ unsigned g_check_fail;
#define ABMX_CHECK(cond, id)                                         \
    do {                                                             \
        if (!(cond)) atomicCAS(&abmx_pred::g_check_fail, 0u, (id));  \
    } while (0)
#else
#define ABMX_CHECK(cond, id) ((void)0)
#endif

__device__ __forceinline__ size_t sidx(const Params& P, int s, int r, int i) {
    ABMX_CHECK(r >= 0 && r < P.R && i >= 0 && i + kS <= P.Npad[s], 1u);
    return static_cast<size_t>(r) * P.Npad[s] + i;
}
__device__ __forceinline__ size_t cidx(const Params& P, int r, int c) {
    ABMX_CHECK(r >= 0 && r < P.R && c >= 0 && c < P.C, 2u);
    return static_cast<size_t>(r) * P.Cpad + c;
}
// exact fixed-point image of an energy on the 2^-20 grid (predation.hpp:60-63)
__device__ __forceinline__ long long to_fx(double e) {
    return __double2ll_rn(__dmul_rn(e, 1048576.0));
}

// kS-wide vector accesses of one thread's consecutive slots (kS = 8: 8 B of u8, 32 B of i32,
// 64 B of f64 per thread and column)
__device__ __forceinline__ void loadk_u8(const uint8_t* p, uint8_t (&v)[kS]) {
    static_assert(kS == 2 || kS == 4 || kS == 8, "2, 4 or 8 slots per thread");
    unsigned long long w;
    if constexpr (kS == 8) {
        w = *reinterpret_cast<const unsigned long long*>(p);
    } else if constexpr (kS == 4) {
        w = *reinterpret_cast<const uint32_t*>(p);
    } else {
        w = *reinterpret_cast<const unsigned short*>(p);
    }
#pragma unroll
    for (int k = 0; k < kS; ++k) v[k] = static_cast<uint8_t>(w >> (8 * k));
}
__device__ __forceinline__ void storek_u8(uint8_t* p, const uint8_t (&v)[kS]) {
    unsigned long long w = 0;
#pragma unroll
    for (int k = 0; k < kS; ++k) w |= static_cast<unsigned long long>(v[k]) << (8 * k);
    if constexpr (kS == 8) {
        *reinterpret_cast<unsigned long long*>(p) = w;
    } else if constexpr (kS == 4) {
        *reinterpret_cast<uint32_t*>(p) = static_cast<uint32_t>(w);
    } else {
        *reinterpret_cast<unsigned short*>(p) = static_cast<unsigned short>(w);
    }
}
__device__ __forceinline__ void loadk_f64(const double* p, double (&v)[kS]) {
#pragma unroll
    for (int q = 0; q < kS / 2; ++q) {
        const double2 d = reinterpret_cast<const double2*>(p)[q];
        v[2 * q] = d.x;
        v[2 * q + 1] = d.y;
    }
}
__device__ __forceinline__ void storek_f64(double* p, const double (&v)[kS]) {
#pragma unroll
    for (int q = 0; q < kS / 2; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
}
__device__ __forceinline__ void loadk_i32(const int* p, int (&v)[kS]) {
    if constexpr (kS == 2) {
        const int2 a = *reinterpret_cast<const int2*>(p);
        v[0] = a.x;
        v[1] = a.y;
    } else {
#pragma unroll
        for (int q = 0; q < kS / 4; ++q) {
            const int4 a = reinterpret_cast<const int4*>(p)[q];
            v[4 * q] = a.x;
            v[4 * q + 1] = a.y;
            v[4 * q + 2] = a.z;
            v[4 * q + 3] = a.w;
        }
    }
}
__device__ __forceinline__ void storek_i32(int* p, const int (&v)[kS]) {
    if constexpr (kS == 2) {
        *reinterpret_cast<int2*>(p) = make_int2(v[0], v[1]);
    } else {
#pragma unroll
        for (int q = 0; q < kS / 4; ++q)
            reinterpret_cast<int4*>(p)[q] = make_int4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
}

template <class T>
__device__ __forceinline__ T block_sum(T v, T* smem) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) smem[threadIdx.x >> 5] = v;
    __syncthreads();
    T t = 0;
    if (threadIdx.x == 0)
        for (int w = 0; w < kT / 32; ++w) t += smem[w];
    return t;  // valid in thread 0
}

// ============================================================== per-cell words
// One uint4 per cell, all four words in the same 32-byte sector:
//   .x sheep list head {epoch8:8 | slot:24}      (atomicExch; the list links through next[0])
//   .y wolf  list head {epoch8:8 | slot:24}      (atomicExch; links through next[1])
//   .z lowest sheep slot {tag:8 | ~slot:24}      (atomicMax, fire-and-forget), tag = epoch%128 + 1
//   .w grass "due" epoch: the cell is ready at the graze of step e iff due < e (lazy regrow:
//      grazing at epoch e with delay D >= 1 stores due = e + D - 1, reproducing the countdown
//      regrow[c] = D, -1 per step, ready at 0 of predation.cpp:188-190,252-258 without a
//      per-step sweep; kFrozen marks a cell grazed with D <= 0, never ready again).
// x/y/z are current iff their tag equals this step's; the host clears x/y/z (not w) every
// kEpochClear (= 128) steps, so tags never alias and the .z tag of the current step is the
// largest alive (a max-reduction keeps it).
// Phase timeline (ABMX_PRED_TRACE builds only): thread 0 of each CTA stamps %globaltimer.
#ifdef ABMX_PRED_TRACE
__device__ __forceinline__ void trace_stamp(const Params& P, int kernel, int point) {
    if (threadIdx.x == 0 && P.trace) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.trace[(static_cast<size_t>(kernel) * gridDim.x + blockIdx.x) * 8 + point] = t;
        if (point == 0) {
            unsigned sm;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
            P.trace[(static_cast<size_t>(kernel) * gridDim.x + blockIdx.x) * 8 + 7] = sm;
        }
    }
}
#define TRACE(k, p) trace_stamp(P, k, p)
#else
#define TRACE(k, p) ((void)0)
#endif

__device__ __forceinline__ unsigned epoch8(unsigned long long epoch) {
    return static_cast<unsigned>(epoch % 255ULL) + 1u;  // 1..255, never the cleared 0
}
__device__ __forceinline__ unsigned min_tag(unsigned long long epoch) {
    return static_cast<unsigned>(epoch % kEpochClear) + 1u;  // 1..128, grows within a clear window
}
constexpr unsigned kNil = 0xFFFFFFu;        // end of list
constexpr unsigned kFrozen = 0xFFFFFFFFu;   // grazed with regrow_delay <= 0: never ready

// blockIdx -> (species, replica, tile): sheep tiles first.
__device__ __forceinline__ void tile_of(const Params& P, unsigned b, int& s, int& r, int& tile) {
    const unsigned sheep_ctas = static_cast<unsigned>(P.R * P.tiles[0]);
    if (b < sheep_ctas) {
        s = 0;
        r = b / P.tiles[0];
        tile = b % P.tiles[0];
    } else {
        s = 1;
        const unsigned u = b - sheep_ctas;
        r = u / P.tiles[1];
        tile = u % P.tiles[1];
    }
}

// largest t with prefix(t) <= k over the chosen packed counter (hi31 = free, lo31 = valid)
__device__ __forceinline__ int find_tile(const unsigned long long* pre, int tiles, unsigned k, bool free_rank) {
    int lo = 0, hi = tiles - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        const unsigned v = free_rank ? hi31(pre[mid]) : lo31(pre[mid]);
        if (v <= k)
            lo = mid;
        else
            hi = mid - 1;
    }
    return lo;
}

// Bookkeeping of step P.birth_epoch for (replica r, species s) once its totals F (free slots)
// and Q (valid parent rows) are known: counters (double-buffered by parity), the ledger, the
// metrics row (predation.cpp:281-287) and, for sheep, the lazy-regrow grass count. Run either
// by tile 0 of k_move / k_finalize (P.book) or by k_book (the per-call step graph).
// With add_dropped the births_dropped column accumulates atomically (run rows start zeroed);
// k_book writes the whole row itself instead, so the per-call graph needs no memset.
__device__ void book_step(const Params& P, int s, int r, int F, int Q, bool add_dropped = true) {
    const int pb = static_cast<int>(P.birth_epoch & 1);
    const int N = P.N[s];
    const int pairs = F < Q ? F : Q;
    SpeciesRep* sr = &P.rep[static_cast<size_t>(r) * 2 + s];
    Events* ev = P.ev + static_cast<size_t>(pb) * P.R + r;
    sr->next_id[pb ^ 1] = sr->next_id[pb] + pairs;
    sr->num_active[pb ^ 1] = N - F + pairs;
    sr->pairs = pairs;
    sr->Q = Q;
    atomicAdd(&ev->births[s], static_cast<unsigned long long>(pairs));
    atomicAdd(&ev->dropped[s], static_cast<unsigned long long>(Q - pairs));
    long long* row = P.metrics + (static_cast<size_t>(r) * P.metrics_stride + P.birth_row) * 4;
    row[s] = N - F + pairs;
    if (add_dropped && Q - pairs) atomicAdd(reinterpret_cast<unsigned long long*>(&row[3]), static_cast<unsigned long long>(Q - pairs));
    if (s == 0) {  // ready cells after that step's (lazy) regrow: - grazed + those due
        unsigned* due = &P.due_count[static_cast<size_t>(r) * P.due_ring + P.birth_epoch % P.due_ring];
        const long long ng = P.n_grass[r] - static_cast<long long>(ev->grass_eaten) + *due;
        *due = 0;
        P.n_grass[r] = ng;
        row[2] = ng;
    }
}

// ============================================================== k_move / k_finalize
// kMove = false: k_finalize (births + counters only).
template <bool kMove>
__device__ void move_phase(const Params& P, unsigned b, unsigned nb, unsigned long long* s_pre) {
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ long long s_red[kT / 32];
    __shared__ unsigned s_base;
    const unsigned long long epoch = P.epoch;
    if (kMove) TRACE(0, 0);
    int s, r, tile;
    tile_of(P, b, s, r, tile);
    const int N = P.N[s];
    const int i0 = tile * kTile + threadIdx.x * kS;
    const size_t base = sidx(P, s, r, i0);
    const size_t rb = static_cast<size_t>(r) * P.Npad[s];
    if (kMove) {  // zero this step's event accumulators (its parity; births use the other)
        Events* ev = P.ev + static_cast<size_t>(epoch & 1) * P.R;
        for (unsigned rr = b * kT + threadIdx.x; rr < static_cast<unsigned>(P.R); rr += nb * kT)
            memset(&ev[rr], 0, sizeof(Events));
    }
    // dense species: issue the column loads together with the mask load
    uint8_t act[kS] = {};
    int cell[kS] = {}, age[kS] = {};
    const bool live = i0 < N;
    if (live) {
        if (kMove && s == 0) {
            loadk_i32(P.cell[s] + base, cell);
            loadk_i32(P.age[s] + base, age);
        }
        loadk_u8(P.active[s] + base, act);
    }

    if (kMove) {  // zero the group counters this step's k_update accumulates into
        unsigned long long* gz = P.group + static_cast<size_t>(epoch & 1) * 2 * P.R * P.groups;
        for (unsigned q = b * kT + threadIdx.x; q < 2u * P.R * P.groups; q += nb * kT) gz[q] = 0ULL;
    }

    // ---------------- (a) births of step P.birth_epoch (rank-match, lifecycle.cpp:144-195)
    bool born[kS] = {};
    bool born_any = false;
    bool full = false;
    if (P.pending) {
        // Births fill the LOWEST free slots, so only the first tiles holding free slots receive
        // any. The 32-tile group totals bound the free slots before this tile from below: if
        // that bound already covers every pair (and no row is dropped), skip the full scan.
        __shared__ unsigned long long s_gt[2];
        if (threadIdx.x < 32) {
            const unsigned long long* gp =
                P.group + (static_cast<size_t>(P.birth_epoch & 1) * 2 * P.R + static_cast<size_t>(s) * P.R + r) * P.groups;
            const int gme = tile / kGroup;
            unsigned long long tot = 0, bef = 0;
            for (int g = threadIdx.x; g < P.groups; g += 32) {
                const unsigned long long v = gp[g];
                tot += v;
                if (g < gme) bef += v;
            }
            tot = warp_sum(tot);
            bef = warp_sum(bef);
            if (threadIdx.x == 0) {
                s_gt[0] = tot;
                s_gt[1] = bef;
            }
        }
        __syncthreads();
        const unsigned F = hi31(s_gt[0]), Q = lo31(s_gt[0]);
        const unsigned pairs = F < Q ? F : Q;
        full = tile == 0 || Q > F || hi31(s_gt[1]) < pairs;
    }
    if (full) {
        const int tiles = P.tiles[s];
        const unsigned long long* tc = P.status + (static_cast<size_t>(s) * P.R + r) * P.status_stride;
        unsigned long long carry = 0;  // exclusive prefix of the tile counts -> s_pre
        for (int t0 = 0; t0 < tiles; t0 += kT) {
            const int t = t0 + threadIdx.x;
            const unsigned long long v = t < tiles ? tc[t] : 0ULL;
            unsigned long long tot;
            const unsigned long long ex = block_excl_scan<kT>(v, s_scan, &tot);
            if (t < tiles) s_pre[t] = carry + ex;
            carry += tot;
            __syncthreads();
        }
        const int F = static_cast<int>(hi31(carry)), Q = static_cast<int>(lo31(carry));
        const int pairs = F < Q ? F : Q;
        const int pb = static_cast<int>(P.birth_epoch & 1);
        SpeciesRep* sr = &P.rep[static_cast<size_t>(r) * 2 + s];
        const long long base_id = sr->next_id[pb];
        // free slots of this tile in slot order: block scan of the free counts
        bool fr[kS];
        unsigned nf = 0;
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            fr[k] = live && !act[k] && i0 + k < N;
            nf += fr[k];
        }
        unsigned long long tot_f;
        const unsigned long long off = block_excl_scan<kT>(nf, s_scan, &tot_f);
        unsigned rank = hi31(s_pre[tile]) + static_cast<unsigned>(off);
        int vrow[kS];
        unsigned brank[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (fr[k]) {
                if (static_cast<int>(rank) < pairs) {
                    const int vt = find_tile(s_pre, tiles, rank, false);
                    vrow[k] = vt * kTile + static_cast<int>(rank - lo31(s_pre[vt]));
                    ABMX_CHECK(vrow[k] >= 0 && vrow[k] < P.Npad[s] && static_cast<int>(rank) < P.Npad[s], 3u);
                    brank[k] = rank;
                    born[k] = true;
                }
                ++rank;
            }
        int bc[kS];
        double be[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (born[k]) {
                bc[k] = P.rowcell[s][rb + vrow[k]];
                be[k] = P.rowE[s][rb + vrow[k]];
            }
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (born[k]) {
                act[k] = 1;
                cell[k] = bc[k];
                age[k] = 0;
                P.energy[s][base + k] = be[k];
                P.id[s][base + k] = base_id + brank[k];
                P.birth_child[s][rb + brank[k]] = i0 + k;
                born_any = true;
            }
        // energy of this tile's valid rows beyond the pairs (dropped births, predation.cpp:121-135)
        const int qt = static_cast<int>(lo31(tc[tile])), q0 = static_cast<int>(lo31(s_pre[tile]));
        long long fx = 0;
        if (q0 + qt > pairs)
            for (int l = threadIdx.x; l < qt; l += kT)
                if (q0 + l >= pairs) fx += to_fx(P.rowE[s][rb + static_cast<size_t>(tile) * kTile + l]);
        const long long fx_tot = block_sum<long long>(fx, s_red);
        Events* ev = P.ev + static_cast<size_t>(pb) * P.R + r;
        if (threadIdx.x == 0) {
            if (fx_tot) atomicAdd(reinterpret_cast<unsigned long long*>(&ev->e_dropped_fx[s]), static_cast<unsigned long long>(fx_tot));
            if (tile == 0 && P.book) book_step(P, s, r, F, Q);
        }
        if (!kMove && born_any) {
            storek_u8(P.active[s] + base, act);
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (born[k]) {
                    P.cell[s][base + k] = cell[k];
                    P.age[s][base + k] = 0;
                }
        }
    }
    if (!kMove) return;
    TRACE(0, 1);

    // ---------------- (b) move + bin
    const unsigned e8 = epoch8(epoch), tag = min_tag(epoch);
    const unsigned long long key = split(split(split(P.seeds[r], 3), static_cast<unsigned long long>(P.t)), s);
    bool any = false;
    for (int k = 0; k < kS; ++k) any |= act[k] != 0;
    bool first[kS] = {};
    if (live && any) {
        if (s == 1) {  // sparse species: columns only where something lives (newborns keep theirs)
            int c2[kS], a2[kS];
            loadk_i32(P.cell[s] + base, c2);
            loadk_i32(P.age[s] + base, a2);
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (!born[k]) {
                    cell[k] = c2[k];
                    age[k] = a2[k];
                }
        }
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            if (!act[k]) continue;
            const int u = static_cast<int>(draw(key, static_cast<unsigned long long>(i0 + k)) >> 61);
            const int c = cell[k];
            const int y = c / P.W, x = c - y * P.W;
            int nx = x + move_dx(u), ny = y + move_dy(u);
            nx = nx < 0 ? nx + P.W : (nx >= P.W ? nx - P.W : nx);
            ny = ny < 0 ? ny + P.H : (ny >= P.H ? ny - P.H : ny);
            cell[k] = ny * P.W + nx;
            age[k] += 1;
        }
        unsigned* cw = reinterpret_cast<unsigned*>(P.cw);
        unsigned old[kS];
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) old[k] = atomicExch(&cw[4 * cidx(P, r, cell[k]) + s], (e8 << 24) | static_cast<unsigned>(i0 + k));
        if (s == 0) {
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (act[k]) atomicMax(&cw[4 * cidx(P, r, cell[k]) + 2], (tag << 24) | (kNil - static_cast<unsigned>(i0 + k)));
        }
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (act[k]) {
                const bool cur = (old[k] >> 24) == e8;
                P.next[s][base + k] = cur ? static_cast<int>(old[k] & kNil) : -1;
                first[k] = P.crowded && s == 1 && !cur;
            }
        TRACE(0, 2);
        storek_i32(P.cell[s] + base, cell);
        storek_i32(P.age[s] + base, age);
        if (born_any) storek_u8(P.active[s] + base, act);
    }
    TRACE(0, 3);
    if (live && P.needs_blend) {  // step_agents masks placeholder state back to defaults
#pragma unroll
        for (int k = 0; k < kS; ++k)
            if (!act[k] && i0 + k < N) {
                P.cell[s][base + k] = 0;
                P.energy[s][base + k] = 0.0;
            }
    }
    if (P.crowded && s == 1) {  // block-aggregated append of the cells this thread's wolves opened
        unsigned nfirst = 0;
        for (int k = 0; k < kS; ++k) nfirst += first[k];
        unsigned long long total;
        const unsigned long long off = block_excl_scan<kT>(nfirst, s_scan, &total);
        if (threadIdx.x == 0 && total) s_base = atomicAdd(&P.ctl->occ, static_cast<unsigned>(total));
        __syncthreads();
        if (nfirst) {
            unsigned pos = s_base + static_cast<unsigned>(off);
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (first[k]) {
                    ABMX_CHECK(pos < static_cast<unsigned>(P.R) * static_cast<unsigned>(P.Npad[1]), 8u);
                    P.occ[pos++] = (static_cast<unsigned long long>(r) << 32) | static_cast<uint32_t>(cell[k]);
                }
        }
    }
}

// ============================================================== k_cells (crowded grids)
__device__ void insertion_sort(int* a, int n) {
    for (int i = 1; i < n; ++i) {
        const int v = a[i];
        int j = i - 1;
        while (j >= 0 && a[j] > v) {
            a[j + 1] = a[j];
            --j;
        }
        a[j + 1] = v;
    }
}
__device__ void heap_sort(int* a, int n) {
    auto sift = [&](int root, int end) {
        for (;;) {
            int child = 2 * root + 1;
            if (child >= end) return;
            if (child + 1 < end && a[child + 1] > a[child]) ++child;
            if (a[root] >= a[child]) return;
            const int tmp = a[root];
            a[root] = a[child];
            a[child] = tmp;
            root = child;
        }
    };
    for (int i = n / 2 - 1; i >= 0; --i) sift(i, n);
    for (int end = n - 1; end > 0; --end) {
        const int tmp = a[0];
        a[0] = a[end];
        a[end] = tmp;
        sift(0, end);
    }
}

constexpr int kSmallList = 8;

// One thread per cell holding >= 1 wolf: sort both lists by slot (registers, or a heap sort
// in the scratch pool for long lists) and flag the k-th wolf / k-th sheep pairs
// (predation.cpp:197-239). On crowded grids the pull pairing of k_update would walk long lists.
__device__ unsigned long long wolf_cell(const Params& P, unsigned long long ent, unsigned e8) {
    const int r = static_cast<int>(ent >> 32), c = static_cast<int>(static_cast<uint32_t>(ent));
    const uint2 word = *reinterpret_cast<const uint2*>(&P.cw[cidx(P, r, c)]);
    if ((word.x >> 24) != e8) return 0;  // no sheep in this cell
    const size_t sb = static_cast<size_t>(r) * P.Npad[0], wb = static_cast<size_t>(r) * P.Npad[1];
    const int w0 = static_cast<int>(word.y & kNil), s0 = static_cast<int>(word.x & kNil);
    int wl[kSmallList], sl[kSmallList];
    int lw = 0, ls = 0;
    for (int w = w0, v = s0; w >= 0 || v >= 0;) {
        ABMX_CHECK(w < P.Npad[1] && v < P.Npad[0], 6u);
        const int nw = w >= 0 ? P.next[1][wb + w] : -1;
        const int nv = v >= 0 ? P.next[0][sb + v] : -1;
        if (w >= 0) {
            if (lw < kSmallList) wl[lw] = w;
            ++lw;
        }
        if (v >= 0) {
            if (ls < kSmallList) sl[ls] = v;
            ++ls;
        }
        w = nw;
        v = nv;
    }
    const int pairs = lw < ls ? lw : ls;
    if (lw <= kSmallList && ls <= kSmallList) {
        insertion_sort(wl, lw);
        insertion_sort(sl, ls);
        for (int q = 0; q < pairs; ++q) {
            P.flag[0][sb + sl[q]] = 1;  // eaten
            P.flag[1][wb + wl[q]] = 1;  // ate
        }
    } else {
        // every agent sits in exactly one cell list, so the pool (R * (Npad0 + Npad1) entries)
        // cannot overflow
        const unsigned off = atomicAdd(&P.ctl->pool_top, static_cast<unsigned>(lw + ls));
        ABMX_CHECK(static_cast<long long>(off) + lw + ls <= P.pool_size, 7u);
        int* pw = P.pool + off;
        int* ps = pw + lw;
        int q = 0;
        for (int w = w0; w >= 0; w = P.next[1][wb + w]) pw[q++] = w;
        q = 0;
        for (int v = s0; v >= 0; v = P.next[0][sb + v]) ps[q++] = v;
        heap_sort(pw, lw);
        heap_sort(ps, ls);
        for (q = 0; q < pairs; ++q) {
            P.flag[0][sb + ps[q]] = 1;
            P.flag[1][wb + pw[q]] = 1;
        }
    }
    return static_cast<unsigned long long>(pairs);
}

__global__ void __launch_bounds__(kT) k_cells(Params P) {
    const unsigned e8 = epoch8(P.epoch);
    const unsigned nw = *reinterpret_cast<volatile unsigned*>(&P.ctl->occ);
    const unsigned stride = gridDim.x * kT;
    for (unsigned q = blockIdx.x * kT + threadIdx.x; q - threadIdx.x < nw; q += stride) {
        unsigned long long eaten = 0;
        int rw = -1;
        if (q < nw) {
            const unsigned long long ent = P.occ[q];
            rw = static_cast<int>(ent >> 32);
            eaten = wolf_cell(P, ent, e8);
        }
        const unsigned grp = __match_any_sync(0xffffffffu, rw);
        const unsigned long long tot = __reduce_add_sync(grp, static_cast<unsigned>(eaten));
        if (rw >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1 && tot)
            atomicAdd(&P.ev[static_cast<size_t>(P.epoch & 1) * P.R + rw].sheep_eaten, tot);
    }
}

// ============================================================== k_update
// Rank of `me` among a cell list's slots, and the list's length (short lists on sparse grids).
__device__ __forceinline__ void list_rank(const int* next, int head, int me, int& rank, int& len) {
    rank = 0;
    len = 0;
    for (int v = head; v >= 0; v = next[v]) {
        rank += v < me;
        ++len;
    }
}

__device__ void update_phase(const Params& P, unsigned b) {
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ unsigned long long s_cnt[kT / 32];
    __shared__ long long s_fx[kT / 32];
    __shared__ unsigned s_eat[kT / 32];
    const unsigned long long epoch = P.epoch;
    const int p = static_cast<int>(epoch & 1);
    const unsigned tag = min_tag(epoch), e8 = epoch8(epoch), ep = static_cast<unsigned>(epoch);
    TRACE(1, 0);
    int s, r, tile;
    tile_of(P, b, s, r, tile);
    if (b == 0 && threadIdx.x == 0) {  // the move (and pairing) of this step are complete
        P.ctl->occ = 0;
        P.ctl->pool_top = 0;
    }
    const unsigned long long key = split(split(split(P.seeds[r], 4), static_cast<unsigned long long>(P.t)), s);
    const int N = P.N[s];
    const int i0 = tile * kTile + threadIdx.x * kS;
    const size_t base = sidx(P, s, r, i0);
    const size_t sb = static_cast<size_t>(r) * P.Npad[0], wb = static_cast<size_t>(r) * P.Npad[1];
    const double gain = P.gain[s], metab = P.metab, prob = P.prob[s], frac = P.frac;

    uint8_t act[kS] = {};
    double E[kS] = {}, child[kS] = {};
    int cell[kS] = {};
    bool valid[kS] = {}, freek[kS] = {};
    unsigned n_graze = 0, n_metab = 0, n_death = 0, n_eaten = 0;
    long long fx_removed = 0;
    if (i0 < N) {
        uint8_t flg[kS] = {};
        if (s == 0) {  // dense species: issue the column loads with the mask
            loadk_f64(P.energy[s] + base, E);
            loadk_i32(P.cell[s] + base, cell);
        }
        loadk_u8(P.active[s] + base, act);
        if (P.crowded) loadk_u8(P.flag[s] + base, flg);
        bool any = false;
    for (int k = 0; k < kS; ++k) any |= act[k] != 0;
        if (s == 1 && any) {
            loadk_f64(P.energy[s] + base, E);
            loadk_i32(P.cell[s] + base, cell);
        }
        bool anyflg = false;
        for (int k = 0; k < kS; ++k) anyflg |= flg[k] != 0;
        if (P.crowded && anyflg) {
            const uint8_t z[kS] = {};
            storek_u8(P.flag[s] + base, z);
        }
        if (any) {
            // the cell word of every live agent (list heads, lowest sheep slot, grass due)
            uint4 cw[kS];
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (act[k]) cw[k] = P.cw[cidx(P, r, cell[k])];
            TRACE(1, 1);
            if (s == 0) {  // graze: lowest sheep slot of a ready cell (predation.cpp:178-195)
#pragma unroll
                for (int k = 0; k < kS; ++k)
                    if (act[k] && cw[k].z == ((tag << 24) | (kNil - static_cast<unsigned>(i0 + k))) && cw[k].w < ep) {
                        P.cw[cidx(P, r, cell[k])].w = P.delay >= 1 ? ep + static_cast<unsigned>(P.delay) - 1u : kFrozen;
                        E[k] = __dadd_rn(E[k], gain);
                        ++n_graze;
                    }
            }
            if (!P.crowded) {
                // predation (predation.cpp:197-239): in a cell holding wolves and sheep the k-th
                // wolf by slot takes the k-th sheep by slot. Each agent ranks itself in its own
                // cell list and counts the other species' list; the up to 2*kS walks of a thread
                // advance in lockstep, so their dependent hops overlap (latency = longest list,
                // not the sum of all walks).
                const int* nmine = s == 0 ? P.next[0] + sb : P.next[1] + wb;
                const int* noth = s == 0 ? P.next[1] + wb : P.next[0] + sb;
                int cm[kS], co[kS], rank[kS], lo[kS];
                bool walk = false;
#pragma unroll
                for (int k = 0; k < kS; ++k) {
                    cm[k] = -1;
                    co[k] = -1;
                    rank[k] = 0;
                    lo[k] = 0;
                    if (!act[k] || (cw[k].x >> 24) != e8 || (cw[k].y >> 24) != e8) continue;
                    const int hs = static_cast<int>(cw[k].x & kNil), hw = static_cast<int>(cw[k].y & kNil);
                    cm[k] = s == 0 ? hs : hw;
                    co[k] = s == 0 ? hw : hs;
                    walk = true;
                }
                while (walk) {
                    int nm[kS], no[kS];
#pragma unroll
                    for (int k = 0; k < kS; ++k) {  // all hops of this round issued together
                        ABMX_CHECK(cm[k] < P.Npad[s] && co[k] < P.Npad[s ^ 1], 4u);
                        nm[k] = cm[k] >= 0 ? nmine[cm[k]] : -1;
                        no[k] = co[k] >= 0 ? noth[co[k]] : -1;
                    }
                    walk = false;
#pragma unroll
                    for (int k = 0; k < kS; ++k) {
                        if (cm[k] >= 0) rank[k] += cm[k] < i0 + k;
                        if (co[k] >= 0) ++lo[k];
                        cm[k] = nm[k];
                        co[k] = no[k];
                        walk |= (cm[k] >= 0) | (co[k] >= 0);
                    }
                }
#pragma unroll
                for (int k = 0; k < kS; ++k) flg[k] = flg[k] || rank[k] < lo[k];
            }
        }
        TRACE(1, 2);
        bool died_any = false;
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            const int i = i0 + k;
            bool alive = act[k] != 0;
            if (alive && flg[k]) {
                if (s == 0) {  // eaten by a wolf this step (predation.cpp:224-238)
                    fx_removed += to_fx(E[k]);
                    ++n_death;
                    ++n_eaten;
                    alive = false;
                } else {
                    E[k] = __dadd_rn(E[k], gain);  // the wolf ate (predation.cpp:236)
                }
            }
            if (alive) {
                E[k] = __dsub_rn(E[k], metab);  // metabolize (predation.cpp:51-60)
                ++n_metab;
                if (E[k] <= 0.0) {  // die_if_starved (predation.cpp:62-74)
                    fx_removed += to_fx(E[k]);
                    ++n_death;
                    alive = false;
                }
            }
            if (alive && E[k] > metab && uniform_double(key, static_cast<unsigned long long>(i)) < prob) {
                // reproduce (predation.cpp:96-113): child = floor(frac*E / 2^-20) * 2^-20
                const double c = __dmul_rn(floor(__dmul_rn(__dmul_rn(frac, E[k]), 1048576.0)), 0x1p-20);
                E[k] = __dsub_rn(E[k], c);
                child[k] = c;
                valid[k] = true;
            }
            if (act[k] && !alive) {
                act[k] = 0;
                E[k] = 0.0;
                died_any = true;
            }
            freek[k] = !alive && i < N;
        }
        if (any) storek_f64(P.energy[s] + base, E);
        if (died_any) {
            storek_u8(P.active[s] + base, act);
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (!act[k] && i0 + k < N) {
                    P.cell[s][base + k] = 0;
                    P.age[s][base + k] = 0;
                    P.id[s][base + k] = 0;
                }
        }
    }
    unsigned nf = 0, nv = 0;
#pragma unroll
    for (int k = 0; k < kS; ++k) {
        nf += freek[k];
        nv += valid[k];
    }
    TRACE(1, 3);
    unsigned long long tile_total;
    const unsigned long long excl = block_excl_scan<kT>(pack2(nf, nv), s_scan, &tile_total);
    // tile-local compaction of the valid parent rows (slot order); k_move concatenates tiles
    int vr = static_cast<int>(lo31(excl));
    const size_t tb = static_cast<size_t>(r) * P.Npad[s] + static_cast<size_t>(tile) * kTile;
#pragma unroll
    for (int k = 0; k < kS; ++k)
        if (valid[k]) {
            ABMX_CHECK(vr >= 0 && vr < kTile, 5u);
            P.row_at[s][tb + vr] = i0 + k;
            P.rowcell[s][tb + vr] = cell[k];
            P.rowE[s][tb + vr] = child[k];
            ++vr;
        }
    // one pass of reductions: (graze, metab, death) packed 21 bits each, eaten, energy
    unsigned long long cnt = (static_cast<unsigned long long>(n_graze) << 42) |
                             (static_cast<unsigned long long>(n_metab) << 21) | n_death;
    long long fxr = fx_removed;
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        cnt += __shfl_xor_sync(0xffffffffu, cnt, d);
        fxr += __shfl_xor_sync(0xffffffffu, fxr, d);
        n_eaten += __shfl_xor_sync(0xffffffffu, n_eaten, d);
    }
    if ((threadIdx.x & 31) == 0) {
        s_cnt[threadIdx.x >> 5] = cnt;
        s_fx[threadIdx.x >> 5] = fxr;
        s_eat[threadIdx.x >> 5] = n_eaten;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long c = 0, eaten = 0;
        long long x_sum = 0;
        for (int w = 0; w < kT / 32; ++w) {
            c += s_cnt[w];
            x_sum += s_fx[w];
            eaten += s_eat[w];
        }
        const unsigned long long g_sum = c >> 42, m_sum = (c >> 21) & 0x1FFFFF, d_sum = c & 0x1FFFFF;
        Events* ev = P.ev + static_cast<size_t>(p) * P.R + r;
        P.status[(static_cast<size_t>(s) * P.R + r) * P.status_stride + tile] = tile_total;
        if (tile_total)  // packed (free, valid): both fields add without carry (each < 2^31)
            atomicAdd(&P.group[(static_cast<size_t>(p) * 2 * P.R + static_cast<size_t>(s) * P.R + r) * P.groups +
                               tile / kGroup],
                      tile_total);
        if (g_sum) {
            atomicAdd(&ev->grass_eaten, g_sum);
            if (P.delay >= 1)  // every cell grazed this step comes due at the same epoch
                atomicAdd(&P.due_count[static_cast<size_t>(r) * P.due_ring +
                                       (epoch + static_cast<unsigned long long>(P.delay) - 1) % P.due_ring],
                          static_cast<unsigned>(g_sum));
        }
        if (m_sum) atomicAdd(&ev->metabolized[s], m_sum);
        if (d_sum) atomicAdd(&ev->deaths[s], d_sum);
        if (eaten && !P.crowded) atomicAdd(&ev->sheep_eaten, eaten);
        if (x_sum) atomicAdd(reinterpret_cast<unsigned long long*>(&ev->e_removed_fx[s]), static_cast<unsigned long long>(x_sum));
    }
    TRACE(1, 4);
}

// ============================================================== kernels
__global__ void __launch_bounds__(kT, kMinB) k_move(Params P) {
    extern __shared__ unsigned long long s_pre[];
    move_phase<true>(P, blockIdx.x, gridDim.x, s_pre);
}
__global__ void __launch_bounds__(kT) k_finalize(Params P) {
    extern __shared__ unsigned long long s_pre[];
    move_phase<false>(P, blockIdx.x, gridDim.x, s_pre);
}
__global__ void __launch_bounds__(kT, kMinB) k_update(Params P) { update_phase(P, blockIdx.x); }

// k_book: one CTA per replica, both species: totals of the tile counts -> book_step, the
// births_dropped column (both species) written directly, then the finished metrics row goes
// straight to mapped host memory (collect_metrics needs no copy).
__global__ void __launch_bounds__(kT) k_book(Params P) {
    // book_step for both species (its bookkeeping, inlined), with every input thread 0 needs from
    // the step's kernels loaded first and both species' tile totals in one round of loads and one
    // reduction: k_book sits on the per-call step's critical path, before the host sees the row
    __shared__ unsigned long long s_red[2][kT / 32];
    const int r = blockIdx.x;
    const int pb = static_cast<int>(P.birth_epoch & 1);
    Events* ev = P.ev + static_cast<size_t>(pb) * P.R + r;
    unsigned* due = &P.due_count[static_cast<size_t>(r) * P.due_ring + P.birth_epoch % P.due_ring];
    long long nid[2] = {0, 0}, ng0 = 0;
    unsigned long long eaten = 0;
    unsigned duev = 0;
    if (threadIdx.x == 0) {
        nid[0] = P.rep[static_cast<size_t>(r) * 2].next_id[pb];
        nid[1] = P.rep[static_cast<size_t>(r) * 2 + 1].next_id[pb];
        ng0 = P.n_grass[r];
        eaten = ev->grass_eaten;
        duev = *due;
    }
    unsigned long long v[2] = {0, 0};
#pragma unroll
    for (int s = 0; s < 2; ++s) {
        const unsigned long long* tc = P.status + (static_cast<size_t>(s) * P.R + r) * P.status_stride;
        for (int t = threadIdx.x; t < P.tiles[s]; t += kT) v[s] += tc[t];
    }
#pragma unroll
    for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) v[s] += __shfl_xor_sync(0xffffffffu, v[s], d);
    if ((threadIdx.x & 31) == 0) {
        s_red[0][threadIdx.x >> 5] = v[0];
        s_red[1][threadIdx.x >> 5] = v[1];
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    long long row[4];
    long long dropped = 0;
#pragma unroll
    for (int s = 0; s < 2; ++s) {  // book_step (above) for species s
        unsigned long long tot = 0;
        for (int w = 0; w < kT / 32; ++w) tot += s_red[s][w];
        const int F = static_cast<int>(hi31(tot)), Q = static_cast<int>(lo31(tot));
        const int N = P.N[s];
        const int pairs = F < Q ? F : Q;
        SpeciesRep* sr = &P.rep[static_cast<size_t>(r) * 2 + s];
        sr->next_id[pb ^ 1] = nid[s] + pairs;
        sr->num_active[pb ^ 1] = N - F + pairs;
        sr->pairs = pairs;
        sr->Q = Q;
        atomicAdd(&ev->births[s], static_cast<unsigned long long>(pairs));
        atomicAdd(&ev->dropped[s], static_cast<unsigned long long>(Q - pairs));
        row[s] = N - F + pairs;
        dropped += Q - pairs;
    }
    const long long ng = ng0 - static_cast<long long>(eaten) + duev;  // ready cells after the lazy regrow
    *due = 0;
    P.n_grass[r] = ng;
    row[2] = ng;
    row[3] = dropped;
    long long* mrow = P.metrics + (static_cast<size_t>(r) * P.metrics_stride + P.birth_row) * 4;
#pragma unroll
    for (int q = 0; q < 4; ++q) mrow[q] = row[q];
    if (P.host_row) {
        long long* h = P.host_row + static_cast<size_t>(r) * 4;
#pragma unroll
        for (int q = 0; q < 4; ++q) h[q] = row[q];
        // publish: the last of the R rows of this call bumps the mapped sequence word, so
        // the host can poll it instead of waiting for the stream to drain. One replica is
        // its own last row: one system fence, no counter round trip.
        __threadfence_system();
        if (P.R == 1) {
            *reinterpret_cast<volatile long long*>(P.host_seq) = static_cast<long long>(P.book_seq);
        } else {
            const unsigned long long done = atomicAdd(P.book_count, 1ULL) + 1ULL;
            if (done == P.book_seq * static_cast<unsigned long long>(P.R)) {
                __threadfence_system();
                *reinterpret_cast<volatile long long*>(P.host_seq) = static_cast<long long>(P.book_seq);
            }
        }
    }
}

// ============================================================== init (create_agents)
// predation.cpp:22-33 + lifecycle.cpp:53-85: x, y, energy drawn for ALL slots from
// seed.split(20|21).split(CreateField=1).split(ordinal); slots >= n0 reset to placeholders.
__global__ void k_init_species(Params P, int s, int n0) {
    const size_t total = static_cast<size_t>(P.R) * P.Npad[s];
    const long long ehi = 2 * static_cast<long long>(P.gain[s]) + 1;
    for (size_t q = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = static_cast<int>(q / P.Npad[s]);
        const int i = static_cast<int>(q % P.Npad[s]);
        const bool live = i < n0;
        int c = 0;
        double e = 0.0;
        if (live) {
            const unsigned long long root = split(split(P.seeds[r], s == 0 ? 20 : 21), 1);
            const long long x = static_cast<long long>(__umul64hi(draw(split(root, 0), i), static_cast<unsigned long long>(P.W)));
            const long long y = static_cast<long long>(__umul64hi(draw(split(root, 1), i), static_cast<unsigned long long>(P.H)));
            const long long en = 1 + static_cast<long long>(__umul64hi(draw(split(root, 2), i), static_cast<unsigned long long>(ehi - 1)));
            c = static_cast<int>(y * P.W + x);
            e = static_cast<double>(en);
        }
        P.active[s][q] = live;
        P.cell[s][q] = c;
        P.age[s][q] = 0;
        P.energy[s][q] = e;
        P.id[s][q] = live ? i : 0;
        P.flag[s][q] = 0;
    }
}

__global__ void k_init_cells(Params P) {
    const size_t total = static_cast<size_t>(P.R) * P.Cpad;
    for (size_t q = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < total;
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const long long c = static_cast<long long>(q % P.Cpad);
        P.cw[q] = make_uint4(0u, 0u, 0u, c < P.C ? 0u : kFrozen);  // full grass; padding frozen
    }
}

// Every kEpochClear steps: reset the tagged words (list heads, lowest slot), keep the due word.
__global__ void k_clear_cells(uint4* cw, size_t n) {
    for (size_t q = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < n;
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        cw[q].x = 0u;
        cw[q].y = 0u;
        cw[q].z = 0u;
    }
}

// L2 flush between timed steps: overwrite a buffer larger than the 126 MB L2, then read a
// second one so L2 is left holding CLEAN lines (otherwise the timed step would pay for
// writing back the flush buffer's dirty lines, traffic that is not part of the workload).
__global__ void k_flush(uint4* p, size_t n) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = make_uint4(static_cast<unsigned>(i), 0u, 0u, 0u);
}
__global__ void k_flush_read(const uint4* p, size_t n, unsigned* sink) {
    unsigned acc = 0;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const uint4 v = p[i];
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9E3779B9u) *sink = acc;  // practically never; keeps the loads alive
}

}  // namespace abmx_pred

// ====================================================================== host engine
namespace abmx_pred {

static const char* kKernelNames[kNumKernels] = {"k_move", "k_cells", "k_update"};
static void* const kKernelFns[kNumKernels] = {reinterpret_cast<void*>(k_move), reinterpret_cast<void*>(k_cells),
                                              reinterpret_cast<void*>(k_update)};

const char* kernel_name(int k) { return (k >= 0 && k < kNumKernels) ? kKernelNames[k] : ""; }

#define CK(x)                                                                        \
    do {                                                                             \
        cudaError_t e_ = (x);                                                        \
        if (e_ != cudaSuccess) {                                                     \
            abmx_internal::set_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
            return ABMX_E_CUDA;                                                      \
        }                                                                            \
    } while (0)

Engine::~Engine() {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    if (graph) cudaGraphDestroy(graph);
    if (step_exec) cudaGraphExecDestroy(step_exec);
    if (h_metrics_pinned) cudaFreeHost(h_metrics_pinned);
    if (d_book_count) cudaFree(d_book_count);
    if (step_graph) cudaGraphDestroy(step_graph);
    for (void* p : allocs) cudaFree(p);
    if (d_run_metrics) cudaFree(d_run_metrics);
    if (flush_buf) cudaFree(flush_buf);
    if (d_trace) cudaFree(d_trace);
    if (stream) cudaStreamDestroy(stream);
}

int Engine::alloc(void** p, size_t bytes) {
    cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
    if (e != cudaSuccess) {
        abmx_internal::set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
        return ABMX_E_CUDA;
    }
    allocs.push_back(*p);
    device_bytes += static_cast<long long>(bytes);
    return ABMX_OK;
}

// init_predation's errors, in its order (predation.cpp:154-164): the initial counts, then per
// species create_agents (lifecycle.cpp:53-85) -- a negative capacity, then the draws of
// x in [0, W), y in [0, H) and energy in [1, 2*trunc(gain) + 1) for EVERY slot, which throw
// DomainError on an empty range (rng.cpp:30-36) whenever the species has any slot.
int check_create(const abmx_predation_config& c) {
    if (c.n_sheep0 > c.sheep_capacity || c.n_wolves0 > c.wolf_capacity) {
        abmx_internal::set_error("initial counts exceed capacities");  // predation.cpp:155-156
        return ABMX_E_CAPACITY;
    }
    const long long cap[2] = {c.sheep_capacity, c.wolf_capacity}, n0[2] = {c.n_sheep0, c.n_wolves0};
    const double gain[2] = {c.energy_gain_sheep, c.energy_gain_wolf};
    for (int s = 0; s < 2; ++s) {
        if (cap[s] < 0 || n0[s] < 0) {
            abmx_internal::set_error("negative capacity");  // lifecycle.cpp:55-58
            return ABMX_E_CAPACITY;
        }
        if (cap[s] == 0) continue;
        if (c.width < 1 || c.height < 1 || !(gain[s] >= 1.0 && gain[s] < 9.2e18)) {
            abmx_internal::set_error("uniform_int: empty range");  // 2*trunc(gain)+1 <= 1, or W/H <= 0
            return ABMX_E_DOMAIN;
        }
    }
    if (c.width < 1 || c.height < 1) {  // an engine limit (the reference builds an empty grid)
        abmx_internal::set_error("width and height must be >= 1");
        return ABMX_E_DOMAIN;
    }
    return ABMX_OK;
}

int Engine::create(const abmx_predation_config& c, const uint64_t* seeds, int R_) {
    cfg = c;
    R = R_;
    if (R < 1) {
        abmx_internal::set_error("replicas must be >= 1");
        return ABMX_E_DOMAIN;
    }
    if (const int rc = check_create(c)) return rc;
    if (c.sheep_capacity > 0xFFFFFE || c.wolf_capacity > 0xFFFFFE) {
        abmx_internal::set_error("capacity per species above 16,777,214 (24-bit cell-list slots)");
        return ABMX_E_CAPACITY;
    }
    if (c.regrow_delay > (1 << 24)) {
        abmx_internal::set_error("regrow_delay > 2^24 is not supported (due-epoch ring size)");
        return ABMX_E_DOMAIN;
    }
    const long long C = static_cast<long long>(c.width) * c.height;
    if (C > (1LL << 31) - 1) {
        abmx_internal::set_error("grid too large (cells must fit int32)");
        return ABMX_E_DOMAIN;
    }
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    Params& P = params;
    memset(&P, 0, sizeof P);
    P.R = R;
    P.W = c.width;
    P.H = c.height;
    P.C = C;
    P.Cpad = static_cast<int>((C + 15) / 16 * 16);
    const int N[2] = {c.sheep_capacity, c.wolf_capacity};
    for (int s = 0; s < 2; ++s) {
        P.N[s] = N[s];
        P.Npad[s] = (N[s] + kTile - 1) / kTile * kTile;  // whole tiles per replica
        if (P.Npad[s] == 0) P.Npad[s] = kTile;
        P.tiles[s] = P.Npad[s] / kTile;
    }
    P.gain[0] = c.energy_gain_sheep;
    P.gain[1] = c.energy_gain_wolf;
    P.metab = c.metabolism;
    P.prob[0] = c.reproduce_prob_sheep;
    P.prob[1] = c.reproduce_prob_wolf;
    P.frac = c.reproduce_energy_frac;
    P.delay = c.regrow_delay >= 1 ? static_cast<int>(c.regrow_delay) : 0;
    P.due_ring = 256;  // must exceed the longest pending countdown (regrow_delay)
    while (P.due_ring <= P.delay) P.due_ring *= 2;
    // crowded grid (more slots than cells): the per-agent list walks of the pull pairing
    // could become long, so pairing runs sort-based in k_cells instead
    P.crowded = (static_cast<long long>(N[0]) + N[1]) > C ? 1 : 0;
    {
        const long long wolves = static_cast<long long>(R) * N[1];
        long long k2 = (wolves + kT - 1) / kT;
        if (k2 > abmx_internal::num_sms() * 8LL) k2 = abmx_internal::num_sms() * 8LL;
        P.k2_ctas = static_cast<int>(k2 > 0 ? k2 : 1);
    }
    P.status_stride = P.tiles[0] > P.tiles[1] ? P.tiles[0] : P.tiles[1];

    int rc;
#define AL(ptr, bytes)                                                 \
    if ((rc = alloc(reinterpret_cast<void**>(&(ptr)), (bytes))) != 0) \
        return rc;
    for (int s = 0; s < 2; ++s) {
        const size_t n = static_cast<size_t>(R) * P.Npad[s];
        AL(P.active[s], n);
        AL(P.cell[s], n * 4);
        AL(P.age[s], n * 4);
        AL(P.energy[s], n * 8);
        AL(P.id[s], n * 8);
        AL(P.next[s], n * 4);
        AL(P.flag[s], n);
        AL(P.row_at[s], n * 4);
        AL(P.rowcell[s], n * 4);
        AL(P.rowE[s], n * 8);
        AL(P.birth_child[s], n * 4);
    }
    AL(P.occ, static_cast<size_t>(R) * P.Npad[1] * 8);
    AL(P.n_grass, sizeof(long long) * R);
    AL(P.due_count, sizeof(unsigned) * P.due_ring * R);
    AL(P.cw, static_cast<size_t>(R) * P.Cpad * 16);
    AL(P.status, static_cast<size_t>(2) * R * P.status_stride * 8);
    P.groups = (P.status_stride + kGroup - 1) / kGroup;
    AL(P.group, static_cast<size_t>(2) * 2 * R * P.groups * 8);
    P.pool_size = static_cast<long long>(R) * (P.Npad[0] + P.Npad[1]);
    AL(P.pool, static_cast<size_t>(P.pool_size) * 4);
    AL(P.ctl, sizeof(Ctl));
    AL(P.rep, sizeof(SpeciesRep) * 2 * R);
    AL(P.ev, sizeof(Events) * 2 * R);
    AL(d_seeds, sizeof(unsigned long long) * R);
    AL(d_metrics_step, sizeof(long long) * 4 * R);
#undef AL
    P.seeds = d_seeds;
    CK(cudaMemcpyAsync(d_seeds, seeds, sizeof(unsigned long long) * R, cudaMemcpyHostToDevice, stream));
    for (int s = 0; s < 2; ++s) CK(cudaMemsetAsync(P.next[s], 0xFF, static_cast<size_t>(R) * P.Npad[s] * 4, stream));
    CK(cudaMemsetAsync(P.due_count, 0, sizeof(unsigned) * P.due_ring * R, stream));
    CK(cudaMemsetAsync(P.status, 0, static_cast<size_t>(2) * R * P.status_stride * 8, stream));
    CK(cudaMemsetAsync(P.group, 0, static_cast<size_t>(2) * 2 * R * P.groups * 8, stream));
    CK(cudaMemsetAsync(P.ev, 0, sizeof(Events) * 2 * R, stream));
    CK(cudaMemsetAsync(P.ctl, 0, sizeof(Ctl), stream));
    {
        std::vector<long long> ng(static_cast<size_t>(R), C);
        CK(cudaMemcpyAsync(P.n_grass, ng.data(), sizeof(long long) * R, cudaMemcpyHostToDevice, stream));
        std::vector<SpeciesRep> rep(static_cast<size_t>(2) * R);
        for (int r = 0; r < R; ++r) {
            rep[2 * r + 0] = SpeciesRep{{c.n_sheep0, c.n_sheep0}, {c.n_sheep0, c.n_sheep0}, 0, 0};
            rep[2 * r + 1] = SpeciesRep{{c.n_wolves0, c.n_wolves0}, {c.n_wolves0, c.n_wolves0}, 0, 0};
        }
        CK(cudaMemcpyAsync(P.rep, rep.data(), sizeof(SpeciesRep) * rep.size(), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));  // the host vectors must be consumed
    }
    move_smem = static_cast<size_t>(P.status_stride + 1) * 8;
    CK(abmx_internal::raise_dyn_smem(k_move, move_smem));
    CK(abmx_internal::raise_dyn_smem(k_finalize, move_smem));
    P.epoch = 1;
    P.t = 1;
    P.metrics = d_metrics_step;
    P.metrics_stride = 1;
    P.run_step = 0;
    P.pending = 0;
    P.book = 1;
    const int g = abmx_internal::num_sms() * 8;
    (void)cudaGetLastError();
    k_init_species<<<g, 256, 0, stream>>>(P, 0, c.n_sheep0);
    k_init_species<<<g, 256, 0, stream>>>(P, 1, c.n_wolves0);
    k_init_cells<<<g, 256, 0, stream>>>(P);
    abmx_internal::count_launch(3);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(d_metrics_step, 0, sizeof(long long) * 4 * R, stream));
    // R metrics rows + the sequence word k_book publishes after them
    CK(cudaHostAlloc(reinterpret_cast<void**>(&h_metrics_pinned), sizeof(long long) * (4 * R + 1), cudaHostAllocMapped));
    memset(h_metrics_pinned, 0, sizeof(long long) * (4 * R + 1));
    CK(cudaMalloc(&d_book_count, 8));
    CK(cudaMemset(d_book_count, 0, 8));
    CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&h_metrics_dev), h_metrics_pinned, 0));
    return ABMX_OK;
}

unsigned Engine::grid(int k) const {
    const Params& P = params;
    if (k == 1) return static_cast<unsigned>(P.k2_ctas);
    return static_cast<unsigned>(P.R * (P.tiles[0] + P.tiles[1]));
}
size_t Engine::smem(int k) const { return k == 0 ? move_smem : 0; }
bool Engine::launched(int k) const { return k != 1 || params.crowded; }

int Engine::build_graph() {
    CK(cudaGraphCreate(&graph, 0));
    void* args[1] = {&params};
    cudaGraphNode_t prev = nullptr;
    for (int k = 0; k < kNumKernels; ++k) {
        if (!launched(k)) continue;
        cudaKernelNodeParams kp{};
        kp.func = kKernelFns[k];
        kp.gridDim = dim3(grid(k));
        kp.blockDim = dim3(kT);
        kp.sharedMemBytes = static_cast<unsigned>(smem(k));
        kp.kernelParams = args;
        CK(cudaGraphAddKernelNode(&nodes[k], graph, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
        prev = nodes[k];
    }
    CK(cudaGraphInstantiate(&graph_exec, graph, 0));
    return ABMX_OK;
}

// One step's kernels. With `ev` (2 events per kernel) every kernel is bracketed by CUDA events
// and launched directly; otherwise the graph is launched with refreshed node parameters.
int Engine::enqueue_step(cudaEvent_t* ev) {
    params.epoch = host_epoch;
    if (host_epoch % kEpochClear == 0)  // epoch tags must not alias stale words
        k_clear_cells<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(params.cw, static_cast<size_t>(R) * params.Cpad);
    void* args[1] = {&params};
    if (ev) {
        for (int k = 0; k < kNumKernels; ++k) {
            if (!launched(k)) continue;
            CK(cudaEventRecord(ev[2 * k], stream));
            CK(cudaLaunchKernel(kKernelFns[k], dim3(grid(k)), dim3(kT), args, smem(k), stream));
            CK(cudaEventRecord(ev[2 * k + 1], stream));
            abmx_internal::count_launch(1);
        }
    } else {
        if (!graph_exec) {
            int rc = build_graph();
            if (rc) return rc;
        }
        for (int k = 0; k < kNumKernels; ++k) {
            if (!launched(k)) continue;
            cudaKernelNodeParams kp{};
            kp.func = kKernelFns[k];
            kp.gridDim = dim3(grid(k));
            kp.blockDim = dim3(kT);
            kp.sharedMemBytes = static_cast<unsigned>(smem(k));
            kp.kernelParams = args;
            CK(cudaGraphExecKernelNodeSetParams(graph_exec, nodes[k], &kp));
            abmx_internal::count_launch(1);
        }
        CK(cudaGraphLaunch(graph_exec, stream));
    }
    // this step's births stay pending until the next k_move (or k_finalize) applies them
    params.needs_blend = 0;
    params.pending = 1;
    params.book = 1;
    params.birth_epoch = host_epoch;
    params.birth_row = params.run_step;
    params.t += 1;
    params.run_step += 1;
    ++host_epoch;
    return ABMX_OK;
}

int Engine::finalize() {
    if (!params.pending) return ABMX_OK;
    void* args[1] = {&params};
    (void)cudaGetLastError();
    CK(cudaLaunchKernel(reinterpret_cast<void*>(k_finalize), dim3(grid(0)), dim3(kT), args, move_smem, stream));
    abmx_internal::count_launch(1);
    params.pending = 0;
    params.book = 1;
    return ABMX_OK;
}

// checked builds: the first failing device bounds check (0 = none); -1 in normal builds
int check_status() {
#ifdef ABMX_CHECKED
    unsigned v = 0;
    if (cudaMemcpyFromSymbol(&v, g_check_fail, sizeof v) != cudaSuccess) return -2;
    return static_cast<int>(v);
#else
    return -1;
#endif
}

int Engine::set_t(long long t) {
    params.t = t;
    return ABMX_OK;
}

int Engine::set_metrics_target(long long* d_metrics, unsigned stride) {
    if (params.pending && params.book) {  // a pending, unbooked row belongs to the previous target
        int rc = finalize();
        if (rc) return rc;
    }
    params.metrics = d_metrics;
    params.metrics_stride = stride;
    params.run_step = 0;
    host_row_valid = false;
    return ABMX_OK;
}

int Engine::launch_steps(long long steps) {
    (void)cudaGetLastError();  // drop stale non-sticky errors of unrelated runtime calls
    for (long long q = 0; q < steps; ++q) {
        int rc = enqueue_step(nullptr);
        if (rc) return rc;
    }
    CK(cudaGetLastError());
    return ABMX_OK;
}

// PredationModel::step(t) as ONE graph launch: the step's kernels, then k_book writes the whole
// metrics row (and its mapped host copy) and the counters; the births stay pending (booked) and
// are applied by the next k_move, or by k_finalize before any state read.
int Engine::step(long long t) {
    int rc = set_metrics_target(d_metrics_step, 1);  // also applies any births still pending
    if (rc) return rc;
    set_t(t);
    (void)cudaGetLastError();
    params.epoch = host_epoch;
    if (host_epoch % kEpochClear == 0)
        k_clear_cells<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(params.cw, static_cast<size_t>(R) * params.Cpad);
    Params fin = params;  // k_book: the bookkeeping of this very step
    fin.birth_epoch = host_epoch;
    fin.birth_row = params.run_step;
    fin.host_row = h_metrics_dev;
    fin.host_seq = h_metrics_dev + 4 * static_cast<size_t>(R);
    fin.book_count = d_book_count;
    fin.book_seq = ++step_seq;
    void* args[1] = {&params};
    void* fargs[1] = {&fin};
    auto kparams = [&](int k, void** a) {
        cudaKernelNodeParams kp{};
        kp.func = k < kNumKernels ? kKernelFns[k] : reinterpret_cast<void*>(k_book);
        kp.gridDim = dim3(k < kNumKernels ? grid(k) : static_cast<unsigned>(R));
        kp.blockDim = dim3(kT);
        kp.sharedMemBytes = static_cast<unsigned>(k < kNumKernels ? smem(k) : 0);
        kp.kernelParams = a;
        return kp;
    };
    if (!step_exec) {
        CK(cudaGraphCreate(&step_graph, 0));
        cudaGraphNode_t prev = nullptr;
        for (int k = 0; k <= kNumKernels; ++k) {
            if (k < kNumKernels && !launched(k)) continue;
            const cudaKernelNodeParams kp = kparams(k, k < kNumKernels ? args : fargs);
            CK(cudaGraphAddKernelNode(&step_nodes[k], step_graph, prev ? &prev : nullptr, prev ? 1 : 0, &kp));
            prev = step_nodes[k];
        }
        CK(cudaGraphInstantiate(&step_exec, step_graph, 0));
    }
    for (int k = 0; k <= kNumKernels; ++k) {
        if (k < kNumKernels && !launched(k)) continue;
        const cudaKernelNodeParams kp = kparams(k, k < kNumKernels ? args : fargs);
        CK(cudaGraphExecKernelNodeSetParams(step_exec, step_nodes[k], &kp));
        abmx_internal::count_launch(1);
    }
    CK(cudaGraphLaunch(step_exec, stream));
    params.needs_blend = 0;
    params.pending = 1;  // births still to apply ...
    params.book = 0;     // ... but already booked
    params.birth_epoch = host_epoch;
    params.birth_row = params.run_step;
    params.t += 1;
    params.run_step += 1;
    ++host_epoch;
    last_run_steps = 0;
    host_row_valid = true;
    CK(cudaGetLastError());
    return ABMX_OK;
}

int Engine::reserve_run(long long steps) {
    const size_t mbytes = sizeof(long long) * 4 * static_cast<size_t>(R) * static_cast<size_t>(steps);
    if (mbytes > run_metrics_bytes) {
        CK(cudaStreamSynchronize(stream));
        if (d_run_metrics) cudaFree(d_run_metrics);
        d_run_metrics = nullptr;
        run_metrics_bytes = 0;
        CK(cudaMalloc(&d_run_metrics, mbytes));
        run_metrics_bytes = mbytes;
    }
    return ABMX_OK;
}

int Engine::prepare_run(long long t0, long long steps) {
    if (steps > 0x7FFFFFFFLL) {
        abmx_internal::set_error("too many steps in one run");
        return ABMX_E_DOMAIN;
    }
    const size_t mbytes = sizeof(long long) * 4 * static_cast<size_t>(R) * static_cast<size_t>(steps);
    int rc = finalize();
    if (rc) return rc;
    rc = reserve_run(steps);
    if (rc) return rc;
    CK(cudaMemsetAsync(d_run_metrics, 0, mbytes, stream));
    rc = set_metrics_target(d_run_metrics, static_cast<unsigned>(steps));
    if (rc) return rc;
    set_t(t0);
    return ABMX_OK;
}

int Engine::run_async(long long t0, long long steps) {
    if (steps <= 0) return ABMX_OK;
    int rc = prepare_run(t0, steps);
    if (rc) return rc;
    rc = launch_steps(steps);
    if (rc) return rc;
    rc = finalize();
    last_run_steps = steps;
    return rc;
}

int Engine::fetch_run_metrics(double* out) {
    int rc = finalize();
    if (rc) return rc;
    const size_t n = static_cast<size_t>(R) * static_cast<size_t>(last_run_steps) * 4;
    std::vector<long long> h(n);
    if (n) CK(cudaMemcpyAsync(h.data(), d_run_metrics, n * sizeof(long long), cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    for (size_t i = 0; i < n; ++i) out[i] = static_cast<double>(h[i]);
    return ABMX_OK;
}

int Engine::last_metrics(long long* out) {
    if (params.pending && params.book) {  // the last row is filled by the births pass
        int rc = finalize();
        if (rc) return rc;
    }
    if (last_run_steps == 0) {
        if (host_row_valid) {  // k_book of the last step() wrote the row to mapped memory
            // poll the mapped sequence word k_book publishes after the rows (cheaper than the
            // stream-completion path); a missing word (a fault) falls back to the stream sync,
            // which reports the error
            const volatile long long* seq = h_metrics_pinned + 4 * static_cast<size_t>(R);
            const auto t0 = std::chrono::steady_clock::now();
            bool seen = false;
            for (unsigned spin = 0;; ++spin) {
                if (*seq == static_cast<long long>(step_seq)) {
                    seen = true;
                    break;
                }
                if ((spin & 1023u) == 1023u &&
                    std::chrono::steady_clock::now() - t0 > std::chrono::milliseconds(200))
                    break;
            }
            if (!seen) CK(cudaStreamSynchronize(stream));
            std::atomic_thread_fence(std::memory_order_acquire);
            memcpy(out, h_metrics_pinned, sizeof(long long) * 4 * R);
            return ABMX_OK;
        }
        CK(cudaMemcpyAsync(out, d_metrics_step, sizeof(long long) * 4 * R, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
        return ABMX_OK;
    }
    for (int r = 0; r < R; ++r) {
        CK(cudaMemcpyAsync(out + static_cast<size_t>(r) * 4,
                           d_run_metrics + (static_cast<size_t>(r) * last_run_steps + last_run_steps - 1) * 4,
                           sizeof(long long) * 4, cudaMemcpyDeviceToHost, stream));
    }
    CK(cudaStreamSynchronize(stream));
    return ABMX_OK;
}

int Engine::last_events(abmx_predation_events* out) {
    int rc = finalize();
    if (rc) return rc;
    const int p = static_cast<int>((host_epoch - 1) & 1);
    std::vector<Events> h(static_cast<size_t>(R));
    CK(cudaMemcpyAsync(h.data(), params.ev + static_cast<size_t>(p) * R, sizeof(Events) * R, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    for (int r = 0; r < R; ++r) {
        const Events& e = h[r];
        abmx_predation_events& o = out[r];
        o.grass_eaten = static_cast<int64_t>(e.grass_eaten);
        o.sheep_eaten_by_wolves = static_cast<int64_t>(e.sheep_eaten);
        abmx_species_events* sp[2] = {&o.sheep, &o.wolves};
        for (int s = 0; s < 2; ++s) {
            sp[s]->metabolized = static_cast<int64_t>(e.metabolized[s]);
            sp[s]->deaths = static_cast<int64_t>(e.deaths[s]);
            sp[s]->births = static_cast<int64_t>(e.births[s]);
            sp[s]->births_dropped = static_cast<int64_t>(e.dropped[s]);
            sp[s]->energy_removed_deaths = static_cast<double>(e.e_removed_fx[s]) * 0x1p-20;
            sp[s]->energy_dropped_births = static_cast<double>(e.e_dropped_fx[s]) * 0x1p-20;
        }
    }
    return ABMX_OK;
}

int Engine::export_species(int r, int s, uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages,
                           int64_t* x, int64_t* y, double* energy, int32_t* num_active, int64_t* next_id) {
    int rc = finalize();
    if (rc) return rc;
    const Params& P = params;
    const size_t n = static_cast<size_t>(P.N[s]);
    const size_t off = static_cast<size_t>(r) * P.Npad[s];
    std::vector<int> cell(n), age(n);
    SpeciesRep sr;
    if (n) {
        CK(cudaMemcpyAsync(active, P.active[s] + off, n, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(ids, P.id[s] + off, n * 8, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(energy, P.energy[s] + off, n * 8, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(cell.data(), P.cell[s] + off, n * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(age.data(), P.age[s] + off, n * 4, cudaMemcpyDeviceToHost, stream));
    }
    CK(cudaMemcpyAsync(&sr, P.rep + static_cast<size_t>(r) * 2 + s, sizeof sr, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    for (size_t i = 0; i < n; ++i) {
        types[i] = s;
        ages[i] = age[i];
        x[i] = cell[i] % P.W;
        y[i] = cell[i] / P.W;
    }
    const int q = static_cast<int>(host_epoch & 1);  // slot the next step will read
    *num_active = sr.num_active[q];
    *next_id = sr.next_id[q];
    return ABMX_OK;
}

int Engine::import_species(int r, int s, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                           const int64_t* x, const int64_t* y, const double* energy, int32_t num_active,
                           int64_t next_id) {
    int rc = finalize();
    if (rc) return rc;
    const Params& P = params;
    const size_t n = static_cast<size_t>(P.N[s]);
    std::vector<uint8_t> act(n);
    std::vector<int> cell(n), age(n);
    int32_t pop = 0;
    for (size_t i = 0; i < n; ++i) {
        act[i] = active[i] ? 1 : 0;
        pop += act[i];
        if (ages[i] < INT32_MIN || ages[i] > INT32_MAX) {
            abmx_internal::set_error("age outside the int32 device layout");
            return ABMX_E_DOMAIN;
        }
        age[i] = static_cast<int>(ages[i]);
        if (x[i] < 0 || x[i] >= P.W || y[i] < 0 || y[i] >= P.H) {
            abmx_internal::set_error(act[i] ? "active agent outside the lattice"
                                            : "placeholder coordinates outside the lattice");
            return ABMX_E_DOMAIN;
        }
        cell[i] = static_cast<int>(y[i] * P.W + x[i]);
    }
    if (pop != num_active) {
        abmx_internal::set_error("num_active must equal popcount(active)");
        return ABMX_E_CAPACITY;
    }
    const size_t off = static_cast<size_t>(r) * P.Npad[s];
    CK(cudaStreamSynchronize(stream));
    if (n) {
        CK(cudaMemcpy(P.active[s] + off, act.data(), n, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(P.id[s] + off, ids, n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(P.energy[s] + off, energy, n * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(P.cell[s] + off, cell.data(), n * 4, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(P.age[s] + off, age.data(), n * 4, cudaMemcpyHostToDevice));
    }
    SpeciesRep sr;
    CK(cudaMemcpy(&sr, P.rep + static_cast<size_t>(r) * 2 + s, sizeof sr, cudaMemcpyDeviceToHost));
    const int q = static_cast<int>(host_epoch & 1);
    sr.num_active[q] = num_active;
    sr.next_id[q] = next_id;
    CK(cudaMemcpy(P.rep + static_cast<size_t>(r) * 2 + s, &sr, sizeof sr, cudaMemcpyHostToDevice));
    params.needs_blend = 1;
    return ABMX_OK;
}

// Lazy regrow (see the cell words): at the end of the last completed step E, a cell is ready
// iff due <= E, and its reference counter is regrow = due - E (predation.cpp:252-258).
int Engine::export_world(int r, uint8_t* ready, int64_t* regrow) {
    int rc = finalize();
    if (rc) return rc;
    const Params& P = params;
    const size_t C = static_cast<size_t>(P.C);
    std::vector<uint4> w(C);
    CK(cudaMemcpyAsync(w.data(), P.cw + static_cast<size_t>(r) * P.Cpad, C * sizeof(uint4), cudaMemcpyDeviceToHost,
                       stream));
    CK(cudaStreamSynchronize(stream));
    const unsigned long long E = host_epoch - 1;
    for (size_t c = 0; c < C; ++c) {
        const unsigned due = w[c].w;
        if (due == 0xFFFFFFFFu) {  // grazed with regrow_delay <= 0: regrow holds the delay
            ready[c] = 0;
            regrow[c] = cfg.regrow_delay;
        } else {
            ready[c] = due <= E;
            regrow[c] = due <= E ? 0 : static_cast<int64_t>(due - E);
        }
    }
    return ABMX_OK;
}

int Engine::import_world(int r, const uint8_t* ready, const int64_t* regrow) {
    int rc = finalize();
    if (rc) return rc;
    Params& P = params;
    const size_t C = static_cast<size_t>(P.C);
    const unsigned long long E = host_epoch - 1;
    std::vector<unsigned> due(C);
    std::vector<unsigned> ring(static_cast<size_t>(P.due_ring), 0u);
    long long n_ready = 0;
    for (size_t c = 0; c < C; ++c) {
        if (ready[c]) {
            if (regrow[c] != 0) {
                abmx_internal::set_error("grass_ready cell with a nonzero regrow counter");
                return ABMX_E_DOMAIN;
            }
            due[c] = 0;
            ++n_ready;
        } else if (regrow[c] <= 0) {
            due[c] = 0xFFFFFFFFu;  // not ready and never regrowing (predation.cpp:254 guard)
        } else if (regrow[c] < P.due_ring) {
            due[c] = static_cast<unsigned>(E + static_cast<unsigned long long>(regrow[c]));
            ++ring[due[c] % static_cast<unsigned>(P.due_ring)];
        } else {
            abmx_internal::set_error("regrow counter exceeds the due-epoch ring of this model");
            return ABMX_E_DOMAIN;
        }
    }
    std::vector<uint4> w(C);
    CK(cudaStreamSynchronize(stream));
    CK(cudaMemcpy(w.data(), P.cw + static_cast<size_t>(r) * P.Cpad, C * sizeof(uint4), cudaMemcpyDeviceToHost));
    for (size_t c = 0; c < C; ++c) w[c].w = due[c];
    CK(cudaMemcpy(P.cw + static_cast<size_t>(r) * P.Cpad, w.data(), C * sizeof(uint4), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(P.due_count + static_cast<size_t>(r) * P.due_ring, ring.data(), ring.size() * sizeof(unsigned),
                  cudaMemcpyHostToDevice));
    CK(cudaMemcpy(P.n_grass + r, &n_ready, sizeof(long long), cudaMemcpyHostToDevice));
    return ABMX_OK;
}

// (parent slot, child slot) of the last step's births: the k-th valid row (tile-local rows
// concatenated in tile order) and the child slot recorded when the birth was applied.
int Engine::birth_pairs(int r, int s, int32_t* parent, int32_t* child, int32_t cap) {
    int rc = finalize();
    if (rc) return rc;
    const Params& P = params;
    SpeciesRep sr;
    const int tiles = P.tiles[s];
    std::vector<unsigned long long> tc(static_cast<size_t>(tiles));
    CK(cudaMemcpyAsync(&sr, P.rep + static_cast<size_t>(r) * 2 + s, sizeof sr, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(tc.data(), P.status + (static_cast<size_t>(s) * P.R + r) * P.status_stride,
                       tiles * sizeof(unsigned long long), cudaMemcpyDeviceToHost, stream));
    const size_t off = static_cast<size_t>(r) * P.Npad[s];
    std::vector<int> rows(static_cast<size_t>(P.Npad[s])), kids(static_cast<size_t>(P.Npad[s]));
    CK(cudaMemcpyAsync(rows.data(), P.row_at[s] + off, rows.size() * 4, cudaMemcpyDeviceToHost, stream));
    CK(cudaMemcpyAsync(kids.data(), P.birth_child[s] + off, kids.size() * 4, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    int k = 0;
    for (int t = 0; t < tiles && k < sr.pairs; ++t) {
        const int nv = static_cast<int>(abmx_dev::lo31(tc[t]));
        for (int j = 0; j < nv && k < sr.pairs; ++j, ++k)
            if (k < cap) parent[k] = rows[static_cast<size_t>(t) * kTile + j];
    }
    for (k = 0; k < sr.pairs && k < cap; ++k) child[k] = kids[static_cast<size_t>(k)];
    return sr.pairs;
}

int Engine::bench(long long t0, long long steps, size_t flush_bytes, bool per_kernel, double* step_ms) {
    if (steps <= 0) return ABMX_OK;
    int rc = prepare_run(t0, steps);
    if (rc) return rc;
    if (flush_bytes > flush_cap) {
        if (flush_buf) cudaFree(flush_buf);
        CK(cudaMalloc(&flush_buf, 2 * flush_bytes + 64));
        CK(cudaMemset(flush_buf, 0, 2 * flush_bytes + 64));
        flush_cap = flush_bytes;
    }
    // per-kernel mode records 2 events around every kernel of every step and synchronises only
    // at the end, so host launch latency never lands inside a kernel's bracket
    const size_t per_step = per_kernel ? 2 * kNumKernels : 2;
    std::vector<cudaEvent_t> ev(per_step * static_cast<size_t>(steps));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    if (!per_kernel && !graph_exec) {
        rc = build_graph();
        if (rc) return rc;
    }
    (void)cudaGetLastError();
    for (long long q = 0; q < steps; ++q) {
        if (flush_bytes) {
            uint4* fb = static_cast<uint4*>(flush_buf);
            k_flush<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(fb, flush_bytes / 16);
            k_flush_read<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(
                fb + flush_bytes / 16, flush_bytes / 16, reinterpret_cast<unsigned*>(fb + flush_bytes / 8));
        }
        cudaEvent_t* e = &ev[per_step * static_cast<size_t>(q)];
        if (per_kernel) {
            rc = enqueue_step(e);
        } else {
            CK(cudaEventRecord(e[0], stream));
            rc = enqueue_step(nullptr);
            // the last step's births are applied by k_finalize (the next step's k_move applies
            // them otherwise): inside the last step's bracket, so every timed step is complete
            if (!rc && q == steps - 1) rc = finalize();
            CK(cudaEventRecord(e[1], stream));
        }
        if (rc) return rc;
    }
    rc = finalize();  // per-kernel mode: the last step's births (kernel times only)
    if (rc) return rc;
    CK(cudaStreamSynchronize(stream));
    for (long long q = 0; q < steps; ++q) {
        cudaEvent_t* e = &ev[per_step * static_cast<size_t>(q)];
        float ms = 0.f;
        if (per_kernel) {
            double tot = 0.0;
            for (int k = 0; k < kNumKernels; ++k) {
                if (!launched(k)) continue;
                CK(cudaEventElapsedTime(&ms, e[2 * k], e[2 * k + 1]));
                kernel_ms[k] += ms;
                kernel_launches[k] += 1;
                tot += ms;
            }
            step_ms[q] = tot;
        } else {
            CK(cudaEventElapsedTime(&ms, e[0], e[1]));
            step_ms[q] = ms;
        }
    }
    for (auto& e : ev) cudaEventDestroy(e);
    last_run_steps = steps;
    return ABMX_OK;
}

}  // namespace abmx_pred
