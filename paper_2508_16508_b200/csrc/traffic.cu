// traffic.cu — the three-lane traffic model (src/models/traffic.cpp:47-238) on sm_100a for R
// roads at once, device-resident state, bit-exact with the reference.
//
// A step is two kernels (one in a multi-step run, which folds each step's spawn into the next
// step's k_accept):
//   k_accept   per column, all three lanes: each car's proposal (traffic.cpp:47-80: forward /
//              forward-left / forward-right drawn from seed.split(6).split(t).draw(slot); exit
//              column: exit iff green, no draw) and the conflict winner of its target
//              (traffic.cpp:95-124: same lane > from the left lane > from the right lane). Every
//              bidder for a cell of column c+1 sits in column c, so the winner needs no global
//              bids. Then the acceptance fixed point (traffic.cpp:124-138): a winner enters once
//              its target is empty or its occupant moves out; the acceptance bits of column c
//              are a function of those of column c+1, F_c : {0,1}^3 -> {0,1}^3 (three 3-bit lane
//              modes), and the fixed point is the suffix composition F_c ∘ ... ∘ F_{L-1}
//              (F_{L-1} is constant: exits), a single-pass scan with decoupled lookback from the
//              road's end. Then, in the same kernel, the apply: accepted moves (set_agents_mask,
//              the mover writes its target's occupancy), exits (remove_agents -> reset_slot,
//              published as the step's exit record) and vacated cells (cleared unless a winner
//              enters: decided from the cell's own acceptance and the bids of the column to its
//              left, re-proposed by the thread as a halo).
//   k_spawn    per road: spawn_cars (traffic.cpp:143-184): k = uniform_int(0, 0, 4), partial lane
//              shuffle, entry cells that are free, rank-match into the lowest free slots (a
//              free-slot bitmap with a summary level and a low-water word, merged with the
//              step's exits), fresh ids.
//
// Layout per road r (capacity 3L slots, 3L cells): active u8, pos i32 (= lane*Lp + cell), ids i64,
// ages i64; occupancy i32 (slot or -1) per cell; free-slot bitmap u32 [Wb] + summary u32 [Ws];
// exit records int4 [2] (by epoch parity).
#include <climits>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/abmx_cuda.h"
#include "abmx_device.cuh"
#include "abmx_internal.h"

using namespace abmx_dev;

namespace abmx_trf {

// CTA sizes are template parameters chosen per road length at create(): slot kernels use
// NT threads x kS slots per CTA, k_accept NA threads x kCI columns per CTA (short roads get small
// CTAs, long roads large ones so the decoupled lookback crosses few tiles).
constexpr int kS = 4;
constexpr int kCI = 4;  // columns per thread in k_accept: one int4 of occupants per lane
#ifndef ABMX_TRF_NA_MAX
#define ABMX_TRF_NA_MAX 1024
#endif
constexpr int kAcceptMaxNT = ABMX_TRF_NA_MAX;  // k_accept CTA size for long roads
#ifndef ABMX_TRF_POLL_NS
#define ABMX_TRF_POLL_NS 0
#endif
constexpr unsigned kSlotMask = (1u << 28) - 1;
constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagPre = 2ULL << 62;
constexpr int kNumKernels = 2;
// A tile's lookback word sits alone in a 128-byte line: packed, the ~90 words of C4's road were
// 6 lines, and the first poll of every tile (32 lanes x 86 tiles at once) queued ~2.5 us at
// their L2 slices (traced: one poll load, ~2.7 us walk).
constexpr int kStatusStride = 16;  // k_accept (with the apply), k_spawn

enum : int { kStay = -1, kExit = -2 };

struct TParams {
    // per step
    unsigned long long epoch;
    long long t;
    double* metrics;  // [R][metrics_stride][4]
    unsigned run_step, metrics_stride;
    // constants
    int R, L, Lp, C, Cpad, Npad, tiles, ctiles;  // C = 3L slots; cells lane*Lp + cell
    int tile_slots, tile_cols;                  // slots per slot-kernel CTA, columns per k_accept CTA
    long long period, green_len;
    const long long* phase;
    const unsigned long long* seeds;
    uint8_t* active;
    int* pos;
    long long* ids;
    long long* ages;
    int* occ;
    unsigned long long* cstatus;  // [R][ctiles][kStatusStride] lookback words, one per 128-byte line
    unsigned* ticket;             // [2]
    int spawn_pending;            // 1: k_accept's column-0 tile first runs the PREVIOUS step's
    long long spawn_t;            //    spawn (step spawn_t, metrics row spawn_row), which a
    unsigned spawn_row;           //    multi-step run folds into the next step (no k_spawn launch)
    int accept_ticketless;        // 1: every k_accept CTA is co-resident (one wave), so the
                                  // lookback needs no ticket order: tile = blockIdx.x
    unsigned* fbits;              // [R][Wb] free-slot bitmap (bit set: slot free), slots < C
    unsigned* fsum;               // [R][Ws] summary: bit w & 31 of word w >> 5 set iff fbits[w] != 0
    int Wb, Ws;
    int4* exits;                  // [R][2] {count, slot x3} exits of the step of epoch parity [e & 1]
    long long* cnt;               // [R][8] num_active, next_id, spawned_total, exited_total, spawned,
                                  // exited, green, low-water bitmap word (every word below is 0)
};

__device__ __forceinline__ bool green_at(const TParams& P, int r, long long t) {  // SignalSchedule::green
    const long long m = ((t + P.phase[r]) % P.period + P.period) % P.period;
    return m < P.green_len;
}
__device__ __forceinline__ bool green_of(const TParams& P, int r) { return green_at(P, r, P.t); }
__device__ __forceinline__ unsigned long long propose_key(const TParams& P, int r) {
    return split(split(P.seeds[r], 6), static_cast<unsigned long long>(P.t));  // TrafficPropose
}
// the TARGET LANE of car `slot` at (lane, cell), or kStay / kExit (traffic.cpp:57-79): the
// target cell is always (lane', cell + 1), so k_accept keeps lanes and never divides by the
// lane stride
__device__ __forceinline__ int proposal_lane(const TParams& P, int slot, int lane, int cell, bool green,
                                            unsigned long long key) {
    if (cell == P.L - 1) return green ? kExit : kStay;
    const int n = 1 + (lane > 0) + (lane < 2);
    const int pick = static_cast<int>(uniform_span(key, static_cast<unsigned long long>(slot), static_cast<unsigned long long>(n)));
    return pick == 0 ? lane : (pick == 1 ? (lane > 0 ? lane - 1 : lane + 1) : lane + 1);
}
// a[k % 3][k / 3] for a runtime k < 12, by selects (a per-thread array indexed at run time would
// live in local memory)
__device__ __forceinline__ int pick12(const int (&a)[3][4], int k) {
    int v = a[0][0];
#pragma unroll
    for (int kk = 1; kk < 12; ++kk) v = k == kk ? a[kk % 3][kk / 3] : v;
    return v;
}
__device__ __forceinline__ unsigned long long bid_word(unsigned long long epoch, int prio, int slot) {
    return (epoch << 32) | (0xFFFFFFFFu - ((static_cast<unsigned>(prio) << 28) | static_cast<unsigned>(slot)));
}
// winner of a cell's bid word this epoch: slot, prio; false if no bid this epoch
__device__ __forceinline__ bool bid_winner(unsigned long long w, unsigned long long epoch, int& slot, int& prio) {
    if ((w >> 32) != (epoch & 0xFFFFFFFFULL)) return false;
    const unsigned v = 0xFFFFFFFFu - static_cast<unsigned>(w);
    slot = static_cast<int>(v & kSlotMask);
    prio = static_cast<int>(v >> 28);
    return true;
}

// ---------------------------------------------------------------- k_accept
// A column map sends each output lane to a constant or to ONE input lane, so it is stored as
// three 3-bit modes (lane l: 0 never, 1 always, 2 + k: iff input bit k) — 9 bits — and maps
// compose lane by lane: (f ∘ g)_l = f_l < 2 ? f_l : g_{f_l - 2}.
constexpr unsigned kIdentityFn = 2u | (3u << 3) | (4u << 6);
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
__device__ __forceinline__ unsigned apply_fn(unsigned f, unsigned v) {  // f(v), v = 3 bits
    unsigned out = 0;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        const unsigned m = mode_of(f, l);
        out |= (m < 2 ? m : (v >> (m - 2)) & 1u) << l;
    }
    return out;
}

__device__ void spawn_road(const TParams& P, int r, long long t, unsigned row, unsigned long long ep,
                           int lane);  // (below)

#ifdef ABMX_TRF_TRACE  // per-CTA %globaltimer stamps of k_accept (thread 0): start, occupants
                       // used, targets used, block scan, lookback, end
__device__ unsigned long long g_trf_trace[4096][10];
__device__ unsigned g_trf_polls[4096][2];  // lane 0's poll loads and walk rounds
__device__ unsigned long long g_trf_warp[32][4];  // the last tile: per warp, lane 0: occupants, targets, maps
#define TRF_WSTAMP(k)                                                                   \
    if ((threadIdx.x & 31) == 0 && blockIdx.x == gridDim.x - 1) {                      \
        unsigned long long t_;                                                          \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                          \
        g_trf_warp[threadIdx.x >> 5][k] = t_;                                           \
    }
#define TRF_STAMP(k)                                                           \
    if (threadIdx.x == 0) {                                                    \
        unsigned long long t_;                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
        if (blockIdx.x < 4096) g_trf_trace[blockIdx.x][k] = t_;                \
    }
#else
#define TRF_STAMP(k)
#define TRF_WSTAMP(k)
#endif

template <int NA>
__global__ void __launch_bounds__(NA) k_accept(TParams P) {
    __shared__ unsigned s_tile;
    __shared__ unsigned s_warp[NA / 32];
    __shared__ unsigned s_vin;
    __shared__ unsigned long long s_key;
    __shared__ int s_green;
    TRF_STAMP(0);
    // tiles of one road depend on their right neighbours: ticket order guarantees progress
    if (threadIdx.x == 0) {
        s_tile = P.ctiles > 1 && !P.accept_ticketless ? atomicAdd(&P.ticket[P.epoch & 1], 1u) : blockIdx.x;
        const int r0 = static_cast<int>(s_tile / P.ctiles);  // the road's light and propose key, once
        s_green = green_of(P, r0);                            // per CTA (64-bit modulo, two splits)
        s_key = propose_key(P, r0);
    }
    __syncthreads();
    const unsigned g = s_tile;
    const int r = static_cast<int>(g / P.ctiles), tau = static_cast<int>(g % P.ctiles);
    if (blockIdx.x == 0 && threadIdx.x == 0 && P.ctiles > 1 && !P.accept_ticketless)
        P.ticket[(P.epoch + 1) & 1] = 0u;  // the next step's tickets (this step uses epoch & 1)
    if (P.spawn_pending && tau == P.ctiles - 1) {  // the tile holding column 0: the previous
        if (threadIdx.x < 32)                       // step's spawn first (its entrance cells)
            spawn_road(P, r, P.spawn_t, P.spawn_row, P.epoch - 1, static_cast<int>(threadIdx.x));
        __syncthreads();
    }
    // tile 0 holds the road's last columns; columns L..Lp-1 are empty padding (-1)
    const int hi = P.Lp - tau * NA * kCI;
    const bool green = s_green != 0;
    const unsigned long long key = s_key;
    const size_t cb = static_cast<size_t>(r) * P.Cpad;
    // columns per thread: kCI, except in a road-entry tile (the partial last one) whose span fits
    // 2 or 1 column per thread. Cars enter at column 0, so early in a run every car of a long
    // road sits in that tile's first few warps: thinner columns spread their proposals over
    // 2-4x the threads (the traced critical path of C4). Columns c_lo + q, q >= cpt,
    // belong to the previous thread: empty here, identity maps.
    const int cpt = tau == P.ctiles - 1 && hi <= NA * 2 ? (hi <= NA ? 1 : 2) : kCI;
    const int c_lo = hi - (static_cast<int>(threadIdx.x) + 1) * cpt;  // multiple of cpt
    // occupants of this thread's columns x 3 lanes (column c_lo + q)
    int o[3][kCI];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        int4 v4 = make_int4(-1, -1, -1, -1);
        if (c_lo >= 0) {
            const int* p = &P.occ[cb + l * P.Lp + c_lo];
            if (cpt == kCI) {
                v4 = *reinterpret_cast<const int4*>(p);
            } else {
                v4.x = p[0];
                if (cpt > 1) v4.y = p[1];
            }
        }
        o[l][0] = v4.x;
        o[l][1] = v4.y;
        o[l][2] = v4.z;
        o[l][3] = v4.w;
    }
    // proposals (no memory). Every bidder for a cell of column c+1 sits in column c, which this
    // thread holds in all three lanes, so the conflict winner (same lane > from the left > from
    // the right, traffic.cpp:95-124) is decided here without bid words; then the targets'
    // occupants, one batched round of independent loads
    int X[3][kCI];  // target lane (the target cell is (X, c + 1)), kStay or kExit
#pragma unroll
    for (int l = 0; l < 3; ++l)
#pragma unroll
        for (int q = 0; q < kCI; ++q)
            X[l][q] = o[l][q] >= 0 ? proposal_lane(P, o[l][q], l, c_lo + q, green, key) : kStay;
    TRF_STAMP(1);
    TRF_WSTAMP(0);
    // occupants of column c_lo + cpt (every target of this thread's last column): the previous
    // thread's first column (a shuffle; across warps and tiles a load), so no target occupant
    // needs a dependent load: the other targets are this thread's own occupants
    int nx[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        nx[l] = __shfl_up_sync(0xffffffffu, o[l][0], 1);
        if ((threadIdx.x & 31) == 0) nx[l] = c_lo >= 0 && c_lo + cpt < P.Lp ? P.occ[cb + l * P.Lp + c_lo + cpt] : -1;
    }
    int ox[3][kCI];  // occupant of the target if this car won it, else kStay - 1 (lost / no move)
#pragma unroll
    for (int q = 0; q < kCI; ++q)
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            bool won = X[l][q] >= 0;
            if (won) {
                const int tl = X[l][q];
                const int pr = l == tl ? 0 : (l == tl - 1 ? 1 : 2);
#pragma unroll
                for (int l2 = 0; l2 < 3; ++l2)
                    if (l2 != l && X[l2][q] == X[l][q] && (l2 == tl ? 0 : (l2 == tl - 1 ? 1 : 2)) < pr) won = false;
            }
            if (won) {
                const int tl = X[l][q];
                ox[l][q] = q + 1 < cpt ? (tl == 0 ? o[0][q + 1 < kCI ? q + 1 : 0] : (tl == 1 ? o[1][q + 1 < kCI ? q + 1 : 0] : o[2][q + 1 < kCI ? q + 1 : 0]))
                                       : (tl == 0 ? nx[0] : (tl == 1 ? nx[1] : nx[2]));
            } else {
                ox[l][q] = kStay - 1;
            }
        }
    // the halo: occupants of column c_lo - 1, read now, before any thread or tile of this step
    // writes occupancy (lane + 1's column c_lo + 3 of its int4; across warps and tiles a load)
    int oh[3];
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        oh[l] = __shfl_down_sync(0xffffffffu, cpt == kCI ? o[l][kCI - 1] : (cpt == 2 ? o[l][1] : o[l][0]), 1);
        if ((threadIdx.x & 31) == 31) oh[l] = c_lo > 0 ? P.occ[cb + l * P.Lp + c_lo - 1] : -1;
    }
    // bit 3q + l of into (q >= 1; q = 0 after the scan, from the halo): a car of column
    // c_lo + q - 1 won the bid for (l, c_lo + q)
    unsigned into = 0;
#pragma unroll
    for (int q = 1; q < kCI; ++q)
#pragma unroll
        for (int l = 0; l < 3; ++l)
            if (ox[l][q - 1] != kStay - 1) into |= 1u << (3 * q + X[l][q - 1]);
    unsigned F[kCI];
    unsigned occm = 0;
    TRF_STAMP(2);
    TRF_WSTAMP(1);
    unsigned T = kIdentityFn;
#pragma unroll
    for (int j = 0; j < kCI; ++j) {  // j = 0 is the rightmost column of this thread
        const int q = kCI - 1 - j;
        unsigned f = kIdentityFn;
        if (c_lo + q >= 0 && q < cpt) {
            f = 0;
#pragma unroll
            for (int l = 0; l < 3; ++l) {
                // mode: 0 never, 1 always, 2 + tl iff the occupant of (tl, c+1) moves out
                unsigned m = 0;
                if (o[l][q] >= 0) {
                    occm |= 1u << (3 * j + l);
                    if (X[l][q] == kExit)
                        m = 1;
                    else if (ox[l][q] != kStay - 1)
                        m = ox[l][q] < 0 ? 1u : 2u + static_cast<unsigned>(X[l][q]);
                }
                f |= m << (3 * l);
            }
        }
        F[j] = f;
        T = compose(f, T);
    }
    // the proposals, packed for the apply (3 bits per (l, q): target lane + 2, kStay + 2, kExit
    // + 2): the unpacked array would stay live across the scan and lookback (register pressure)
    unsigned long long xp = 0;
#pragma unroll
    for (int q = 0; q < kCI; ++q)
#pragma unroll
        for (int l = 0; l < 3; ++l) xp |= static_cast<unsigned long long>(X[l][q] + 2) << (3 * (3 * q + l));
    TRF_STAMP(6);
    TRF_WSTAMP(2);
    // block scan over threads (thread 0 = rightmost): I_t = T_t ∘ I_{t-1}
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    unsigned I = T;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned o = __shfl_up_sync(0xffffffffu, I, d);
        if (lane >= d) I = compose(I, o);
    }
    if (lane == 31) s_warp[warp] = I;
    __syncthreads();
    TRF_STAMP(7);
    if (warp == 0) {
        unsigned wv = lane < NA / 32 ? s_warp[lane] : kIdentityFn;
#pragma unroll
        for (int d = 1; d < NA / 32; d <<= 1) {
            const unsigned o = __shfl_up_sync(0xffffffffu, wv, d);
            if (lane >= d) wv = compose(wv, o);
        }
        if (lane < NA / 32) s_warp[lane] = wv;  // inclusive warp prefixes
    }
    __syncthreads();
    const unsigned wex = warp > 0 ? s_warp[warp - 1] : kIdentityFn;
    const unsigned up = __shfl_up_sync(0xffffffffu, I, 1);
    const unsigned E = lane > 0 ? compose(up, wex) : wex;  // exclusive prefix of this thread
    TRF_STAMP(3);
    if (warp == 0) {  // decoupled lookback, 32 predecessors per round
        const unsigned A = s_warp[NA / 32 - 1];  // tile aggregate
        unsigned long long* st = P.cstatus + static_cast<size_t>(r) * P.ctiles * kStatusStride;
        const unsigned long long tag = (P.epoch & 0x3FFFFFFFULL) << 32;
        unsigned vin = 0;
        if (tau > 0) {
            if (lane == 0) st_word(&st[tau * kStatusStride], kFlagAgg | tag | A);
            unsigned accf = kIdentityFn;  // composition of the aggregates passed so far
#ifdef ABMX_TRF_TRACE
            unsigned n_polls = 0, n_rounds = 0;
#endif
            for (int base = tau - 1;; base -= 32) {
#ifdef ABMX_TRF_TRACE
                ++n_rounds;
#endif
                const int j = base - lane;  // lane 0 = nearest predecessor
                unsigned long long w = 0;
                unsigned fl = j >= 0 ? 0u : 2u;  // beyond the road's first tile: never reached
                for (;;) {  // all lanes stay in the loop until every predecessor has published
                    if (fl == 0) {
#ifdef ABMX_TRF_TRACE
                        ++n_polls;
#endif
                        w = ld_word(&st[j * kStatusStride]);
                        fl = ((w & (0x3FFFFFFFULL << 32)) == tag) ? static_cast<unsigned>(w >> 62) : 0u;
                    }
                    // done once every lane up to the nearest published prefix has its word
                    // (the lanes beyond it are not needed), or every lane has one
                    const unsigned zero = __ballot_sync(0xffffffffu, fl == 0);
                    const unsigned pre2 = __ballot_sync(0xffffffffu, fl == 2);
                    if (!zero || (pre2 && !(zero & ((pre2 & (0u - pre2)) - 1u)))) break;
#if ABMX_TRF_POLL_NS > 0
                    __nanosleep(ABMX_TRF_POLL_NS);  // back off: every tile's warp polls the same few lines
#endif
                }
                // every lane up to the first prefix holds an aggregate (1) or that prefix (2);
                // the lanes BEFORE the first prefix contribute their aggregates, the first prefix
                // ends the walk (lanes beyond it may still be unpublished: not read)
                const unsigned pre = __ballot_sync(0xffffffffu, fl == 2);
                const int first = pre ? __ffs(pre) - 1 : 32;
                unsigned f = lane < first ? static_cast<unsigned>(w & 0x1FFu) : kIdentityFn;
                // ordered reduction: result = f_0 ∘ f_1 ∘ ... (lane 0 nearest)
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    const unsigned o = __shfl_down_sync(0xffffffffu, f, d);
                    if (lane + d < 32) f = compose(f, o);
                }
                accf = compose(accf, __shfl_sync(0xffffffffu, f, 0));
                if (first < 32) {
                    const unsigned pv = static_cast<unsigned>(__shfl_sync(0xffffffffu, w, first) & 7u);
                    vin = apply_fn(accf, pv);
                    break;
                }
            }
#ifdef ABMX_TRF_TRACE
            if (lane == 0 && blockIdx.x < 4096) {
                g_trf_polls[blockIdx.x][0] = n_polls;
                g_trf_polls[blockIdx.x][1] = n_rounds;
            }
#endif
        }
        TRF_STAMP(8);
        if (lane == 0) {
            st_word(&st[tau * kStatusStride], kFlagPre | tag | apply_fn(A, vin));
            s_vin = vin;
        }
        TRF_STAMP(9);
    }
    __syncthreads();  // every thread's occupancy loads are done: the writes below may start
    TRF_STAMP(4);
    // acceptance bits: bit 3q + l of accm = the occupant of (l, c_lo + q) moves (or exits)
    unsigned v = apply_fn(E, s_vin), accm = 0;
#pragma unroll
    for (int j = 0; j < kCI; ++j) {
        v = apply_fn(F[j], v);
        accm |= (v & ((occm >> (3 * j)) & 7u)) << (3 * (kCI - 1 - j));
    }
    // An accepted occupant's cell is vacated unless a winner of the bid for it enters: that
    // winner is accepted exactly when the cell's occupant leaves (or the cell is empty), so no
    // other thread's acceptance is needed. For column c_lo the bidders sit in column c_lo - 1
    // (the halo: the next thread's or tile's), re-proposed here. The code from here on is kept
    // small and rolled: it runs once per thread, usually for no car at all, and after the
    // bench's L2 flush every instruction line of it is fetched cold (traced: 19.6 KB of
    // unrolled tail cost every tile ~4.7 us, warm 1.3 us).
    if (accm & 7u) {  // column c_lo has a leaving car: its halo bids decide the vacate
        int xh0 = kStay, xh1 = kStay, xh2 = kStay;
#pragma unroll 1
        for (int l = 0; l < 3; ++l) {
            const int ohl = l == 0 ? oh[0] : (l == 1 ? oh[1] : oh[2]);
            const int x = ohl >= 0 ? proposal_lane(P, ohl, l, c_lo - 1, green, key) : kStay;
            if (l == 0)
                xh0 = x;
            else if (l == 1)
                xh1 = x;
            else
                xh2 = x;
        }
        const int xh[3] = {xh0, xh1, xh2};
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            if (xh[l] < 0) continue;
            const int tl = xh[l];
            const int pr = l == tl ? 0 : (l == tl - 1 ? 1 : 2);
            bool won = true;
#pragma unroll
            for (int l2 = 0; l2 < 3; ++l2)
                if (l2 != l && xh[l2] == xh[l] && (l2 == tl ? 0 : (l2 == tl - 1 ? 1 : 2)) < pr) won = false;
            if (won) into |= 1u << tl;
        }
    }
    // apply (traffic.cpp:186-238): accepted moves (set_agents_mask: lane / cell <- target, the
    // mover writes its target's occupancy), exits (remove_agents -> reset_slot), vacated cells
    const size_t sb = static_cast<size_t>(r) * P.Npad;
    int4 ex = make_int4(0, -1, -1, -1);
#pragma unroll 1
    for (unsigned mm = accm; mm; mm &= mm - 1) {
        const int k = __ffs(static_cast<int>(mm)) - 1, q = k / 3, l = k - 3 * q;
        const int i = pick12(o, k), tl = static_cast<int>((xp >> (3 * k)) & 7u) - 2;
        ABMX_ASSERT(i >= 0 && i < P.C && (tl == kExit || (tl >= 0 && tl < 3)));
        if (tl == kExit) {  // reset_slot (agent_set.cpp:45-58)
            P.active[sb + i] = 0;
            P.ids[sb + i] = 0;
            P.ages[sb + i] = 0;
            P.pos[sb + i] = 0;
            if (ex.x == 0)
                ex.y = i;
            else if (ex.x == 1)
                ex.z = i;
            else
                ex.w = i;
            ++ex.x;
        } else {
            const int x = tl * P.Lp + c_lo + q + 1;
            P.pos[sb + i] = x;
            P.occ[cb + x] = i;
        }
        if (!((into >> k) & 1u)) P.occ[cb + l * P.Lp + c_lo + q] = -1;
    }
    // the exit column's thread publishes the step's exits (read by this step's spawn)
    if (c_lo <= P.L - 1 && P.L - 1 < c_lo + cpt) P.exits[static_cast<size_t>(r) * 2 + (P.epoch & 1)] = ex;
    TRF_STAMP(5);
}

// ---------------------------------------------------------------- k_spawn
// spawn_cars of step t on road r (traffic.cpp:143-184), one warp (lane = 0..31); metrics row
// `row`; ep = the step's epoch (its exit record). The lowest free slots come from the road's
// free-slot bitmap, searched from the low-water word cnt[7] (every word below it is full), merged
// with the step's exits (which become free only now, after the step's moves).
__device__ void spawn_road(const TParams& P, int r, long long t, unsigned row, unsigned long long ep, int lane) {
    const size_t sb = static_cast<size_t>(r) * P.Npad, cb = static_cast<size_t>(r) * P.Cpad;
    long long* cn = P.cnt + static_cast<size_t>(r) * 8;
    unsigned* fb = P.fbits + static_cast<size_t>(r) * P.Wb;
    unsigned* fs = P.fsum + static_cast<size_t>(r) * P.Ws;
    // every load that does not depend on the draws, issued together: the seed, the three
    // entrance cells, the exit record, the counters
    const unsigned long long seed = P.seeds[r];
    const int occ_in[3] = {P.occ[cb], P.occ[cb + P.Lp], P.occ[cb + 2 * static_cast<size_t>(P.Lp)]};
    const int4 ex = P.exits[static_cast<size_t>(r) * 2 + (ep & 1)];
    const long long nid = cn[1], c0 = cn[0], c2 = cn[2], c3 = cn[3];
    const int lw = static_cast<int>(cn[7]);
    const bool g = green_at(P, r, t);
    // rows: k attempts, partial shuffle, free entry cells. Lane lists are 2-bit fields of one
    // word (static register indexing: a per-thread array with runtime indices lives in local memory)
    unsigned rowsw = 0;  // row q (entry lane) in bits 2q..2q+1
    int nvalid = 0;
    {
        const unsigned long long key = split(split(seed, 7), static_cast<unsigned long long>(t));
        const int k = static_cast<int>(uniform_span(key, 0, 4));
        unsigned lanesw = 0u | (1u << 2) | (2u << 4);  // lanes[i] in bits 2i..2i+1
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            if (i >= k) break;
            const int j = i + static_cast<int>(uniform_span(key, static_cast<unsigned long long>(1 + i),
                                                            static_cast<unsigned long long>(3 - i)));
            const unsigned li = (lanesw >> (2 * i)) & 3u, lj = (lanesw >> (2 * j)) & 3u;
            lanesw = (lanesw & ~(3u << (2 * i)) & ~(3u << (2 * j))) | (lj << (2 * i)) | (li << (2 * j));
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            if (q >= k) break;
            const unsigned ln = (lanesw >> (2 * q)) & 3u;
            if ((ln == 0 ? occ_in[0] : (ln == 1 ? occ_in[1] : occ_in[2])) < 0) {
                rowsw |= ln << (2 * nvalid);
                ++nvalid;
            }
        }
    }
    // the lowest nvalid free slots of the bitmap (warp-uniform), windows of 32 words aligned to
    // summary words; an empty window jumps ahead through the summary. Absent entries: INT_MAX.
    int f0 = INT_MAX, f1 = INT_MAX, f2 = INT_MAX;
    unsigned fw0 = 0u, fw1 = 0u, fw2 = 0u;  // each found slot's bitmap word as loaded
    int nfb = 0;
    for (int w0 = lw & ~31; nfb < nvalid && w0 < P.Wb;) {
        const unsigned word = w0 + lane < P.Wb ? fb[w0 + lane] : 0u;
        unsigned m = __ballot_sync(0xffffffffu, word != 0u);
        if (!m) {  // the next non-empty summary word after this window
            int next = -1;
            for (int sw0 = (w0 >> 5) + 1; sw0 < P.Ws && next < 0; sw0 += 32) {
                const unsigned sw = sw0 + lane < P.Ws ? fs[sw0 + lane] : 0u;
                const unsigned sm = __ballot_sync(0xffffffffu, sw != 0u);
                if (sm) next = sw0 + __ffs(static_cast<int>(sm)) - 1;
            }
            if (next < 0) break;  // no free slot in the bitmap
            w0 = next << 5;
            continue;
        }
        while (m && nfb < nvalid) {
            const int src = __ffs(static_cast<int>(m)) - 1;
            m &= m - 1;
            const unsigned wd0 = __shfl_sync(0xffffffffu, word, src);
            for (unsigned wd = wd0; wd && nfb < nvalid; wd &= wd - 1) {
                const int sl = ((w0 + src) << 5) + __ffs(static_cast<int>(wd)) - 1;
                if (nfb == 0) {
                    f0 = sl;
                    fw0 = wd0;
                } else if (nfb == 1) {
                    f1 = sl;
                    fw1 = wd0;
                } else {
                    f2 = sl;
                    fw2 = wd0;
                }
                ++nfb;
            }
        }
        w0 += 32;
    }
    if (lane == 0) {
        // the step's exits are free too (sorted here, INT_MAX when absent): the spawned slots are
        // the lowest nvalid of both lists, the q-th lowest taking row q
        const int ne = ex.x;
        int e0 = ne > 0 ? ex.y : INT_MAX, e1 = ne > 1 ? ex.z : INT_MAX, e2 = ne > 2 ? ex.w : INT_MAX;
        auto cswap = [](int& a, int& b) {
            const int lo = a < b ? a : b, hi = a < b ? b : a;
            a = lo;
            b = hi;
        };
        cswap(e0, e1);
        cswap(e1, e2);
        cswap(e0, e1);
        const int fl[3] = {f0, f1, f2}, el[3] = {e0, e1, e2};
        const unsigned fwl[3] = {fw0, fw1, fw2};
        int frank[3], erank[3];  // rank in the union (slots are distinct), >= 6 when absent
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            int rf = k, re = k;
#pragma unroll
            for (int k2 = 0; k2 < 3; ++k2) {
                rf += el[k2] < fl[k];
                re += fl[k2] < el[k];
            }
            frank[k] = fl[k] == INT_MAX ? 6 : rf;
            erank[k] = el[k] == INT_MAX ? 6 : re;
        }
        const int spawned = nvalid < nfb + ne ? nvalid : nfb + ne;
        // bitmap: exits not taken become free, slots taken from it leave it; a summary bit is
        // cleared when its word empties. Every word below the first found one was full, and the
        // kept exits may lie lower: the new low-water word
        int lw_new = nfb > 0 ? (f0 >> 5) : lw;
#pragma unroll
        for (int u = 0; u < 3; ++u) {
            if (el[u] == INT_MAX || erank[u] < spawned) continue;
            const int w = el[u] >> 5;
            atomicOr(&fb[w], 1u << (el[u] & 31));
            atomicOr(&fs[w >> 5], 1u << (w & 31));
            lw_new = w < lw_new ? w : lw_new;
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            if (frank[k] >= spawned) continue;
            const int w = fl[k] >> 5;
            atomicAnd(&fb[w], ~(1u << (fl[k] & 31)));
            unsigned fin = fwl[k];  // the word after this spawn
#pragma unroll
            for (int k2 = 0; k2 < 3; ++k2)
                if (frank[k2] < spawned && (fl[k2] >> 5) == w) fin &= ~(1u << (fl[k2] & 31));
#pragma unroll
            for (int u = 0; u < 3; ++u)
                if (el[u] != INT_MAX && erank[u] >= spawned && (el[u] >> 5) == w) fin |= 1u << (el[u] & 31);
            if (fin == 0u) atomicAnd(&fs[w >> 5], ~(1u << (w & 31)));
            ABMX_ASSERT(w < P.Wb && (fwl[k] >> (fl[k] & 31)) & 1u);
        }
        // the new cars: the q-th lowest slot takes row q (entry lane), id next_id + q
#pragma unroll
        for (int k = 0; k < 6; ++k) {
            const int rk = k < 3 ? frank[k] : erank[k - 3];
            if (rk >= spawned) continue;
            const int sl = k < 3 ? fl[k] : el[k - 3];
            const int ln = static_cast<int>((rowsw >> (2 * rk)) & 3u);
            ABMX_ASSERT(sl >= 0 && sl < P.C && ln < 3);
            P.active[sb + sl] = 1;
            P.pos[sb + sl] = ln * P.Lp;
            P.ids[sb + sl] = nid + rk;
            P.ages[sb + sl] = 0;
            P.occ[cb + ln * P.Lp] = sl;
        }
        const int exited = ne;
        const long long n_cars = c0 + spawned - exited;
        cn[0] = n_cars;
        cn[1] = nid + spawned;
        cn[2] = c2 + spawned;
        cn[3] = c3 + exited;
        cn[4] = spawned;
        cn[5] = exited;
        cn[6] = g ? 1 : 0;
        cn[7] = lw_new;
        double* mrow = P.metrics + (static_cast<size_t>(r) * P.metrics_stride + row) * 4;
        mrow[0] = static_cast<double>(n_cars);
        mrow[1] = static_cast<double>(spawned);
        mrow[2] = static_cast<double>(exited);
        mrow[3] = g ? 1.0 : 0.0;
    }
}

__global__ void k_spawn(TParams P) { spawn_road(P, blockIdx.x, P.t, P.run_step, P.epoch, threadIdx.x); }

// the bench's L2 flush: after the memset of a buffer larger than L2, read it back so L2 holds
// clean lines (as the predation bench): the timed step pays no write-backs of the flush buffer
__global__ void k_flush_read_t(const uint4* p, size_t n, unsigned* sink) {
    unsigned a = 0;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        a += p[i].x;
    if (a == 0x12345678u) *sink = a;
}

// ---------------------------------------------------------------- resolve_conflicts (explicit)
// General proposals (any in-road target): acceptance is the least fixed point of
// acc(w) = winner(w) && (target empty || acc(occupant)), solved by pointer jumping;
// state >= 0: pointer to the slot whose acceptance decides; -1 accepted; -2 rejected.
__global__ void k_res_bid(const uint8_t* active, const int* lane, const int* target, int n, int L,
                          unsigned long long* bid) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !active[i] || target[i] < 0) return;
    const int tl = target[i] / L;
    const int prio = lane[i] == tl ? 0 : (lane[i] == tl - 1 ? 1 : 2);
    atomicMax(&bid[target[i]], bid_word(1ULL, prio, i));
}
__global__ void k_res_init(const uint8_t* active, const int* target, const int* occ, const unsigned long long* bid,
                           int n, int* st) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    int s = -2;
    if (active[i]) {
        if (target[i] == kExit) {
            s = -1;
        } else if (target[i] >= 0) {
            int ws, wp;
            if (bid_winner(bid[target[i]], 1ULL, ws, wp) && ws == i) s = occ[target[i]] < 0 ? -1 : occ[target[i]];
        }
    }
    st[i] = s;
}
__global__ void k_res_jump(const int* st, int* out, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int s = st[i];
    out[i] = s >= 0 ? st[s] : s;
}
__global__ void k_res_out(const int* st, int n, uint8_t* acc) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) acc[i] = st[i] == -1 ? 1 : 0;
}

// ---------------------------------------------------------------- init / flush
__global__ void k_init(TParams P) {
    const size_t ns = static_cast<size_t>(P.R) * P.Npad, nc = static_cast<size_t>(P.R) * P.Cpad;
    for (size_t q = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < (ns > nc ? ns : nc);
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (q < ns) {
            P.active[q] = 0;
            P.pos[q] = 0;
            P.ids[q] = 0;
            P.ages[q] = 0;
        }
        if (q < nc) P.occ[q] = -1;
    }
    const size_t nw = static_cast<size_t>(P.R) * P.Wb, nsw = static_cast<size_t>(P.R) * P.Ws;
    for (size_t q = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < (nw > nsw ? nw : nsw);
         q += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (q < nw) {  // every slot < C free
            const long long s0 = static_cast<long long>(q % P.Wb) * 32;
            const long long nfree = P.C - s0 < 0 ? 0 : (P.C - s0 > 32 ? 32 : P.C - s0);
            P.fbits[q] = nfree >= 32 ? 0xFFFFFFFFu : ((1u << nfree) - 1u);
        }
        if (q < nsw) {
            const long long w0 = static_cast<long long>(q % P.Ws) * 32;  // words w0.. of this summary word
            const long long nonempty_words = (P.C + 31) / 32 - w0;       // words holding a slot < C
            const long long k = nonempty_words < 0 ? 0 : (nonempty_words > 32 ? 32 : nonempty_words);
            P.fsum[q] = k >= 32 ? 0xFFFFFFFFu : ((1u << k) - 1u);
        }
        if (q < static_cast<size_t>(P.R) * 2) P.exits[q] = make_int4(0, -1, -1, -1);
    }
}

}  // namespace abmx_trf

// ====================================================================== host engine
using namespace abmx_trf;

#define CKT(x)                                                                        \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            abmx_internal::set_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
            return ABMX_E_CUDA;                                                       \
        }                                                                             \
    } while (0)

struct abmx_traffic {
    abmx_traffic_config cfg{};
    int R = 0;
    TParams P{};
    cudaStream_t stream = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t nodes[kNumKernels] = {};
    std::vector<void*> allocs;
    double* d_metrics_step = nullptr;  // [R][1][4]
    double* d_run_metrics = nullptr;
    size_t run_metrics_bytes = 0;
    long long last_run_steps = 0;
    unsigned long long host_epoch = 1;
    double kernel_ms[kNumKernels] = {};
    long long kernel_launches[kNumKernels] = {};
    void* flush_buf = nullptr;
    size_t flush_cap = 0;
    long long* h_cnt = nullptr;  // pinned copy of the counters

    ~abmx_traffic() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (exec2) cudaGraphExecDestroy(exec2);
        if (graph2) cudaGraphDestroy(graph2);
        for (void* p : allocs) cudaFree(p);
        if (d_run_metrics) cudaFree(d_run_metrics);
        if (flush_buf) cudaFree(flush_buf);
        if (h_cnt) cudaFreeHost(h_cnt);
        if (stream) cudaStreamDestroy(stream);
    }
    int alloc(void** p, size_t bytes) {
        cudaError_t e = cudaMalloc(p, bytes ? bytes : 16);
        if (e != cudaSuccess) {
            abmx_internal::set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
            return ABMX_E_CUDA;
        }
        allocs.push_back(*p);
        return ABMX_OK;
    }
    unsigned grid(int k) const {  // k: 0 k_accept, 1 k_spawn
        return static_cast<unsigned>(k == 0 ? R * P.ctiles : R);
    }
    int nt = 256, na = 1024;  // CTA sizes of the slot kernels and of k_accept
    void* fns[kNumKernels] = {};
    unsigned block(int k) const {
        return k == 1 ? 32u : static_cast<unsigned>(na);
    }
    void* fn(int k) const { return fns[k]; }
    void pick_kernels() {
        // slot kernels: the smallest CTA covering a road (32..256 threads x 4 slots)
        nt = 32;
        while (nt < 256 && nt * kS < P.C) nt *= 2;
        // k_accept: the smallest CTA covering a road's columns, else 1024 threads (few tiles)
        na = 32;
        while (na < kAcceptMaxNT && na * kCI < P.Lp) na *= 2;
        switch (na) {
            case 32: fns[0] = reinterpret_cast<void*>(k_accept<32>); break;
            case 64: fns[0] = reinterpret_cast<void*>(k_accept<64>); break;
            case 128: fns[0] = reinterpret_cast<void*>(k_accept<128>); break;
            case 256: fns[0] = reinterpret_cast<void*>(k_accept<256>); break;
            case 512: fns[0] = reinterpret_cast<void*>(k_accept<512>); break;
            default: fns[0] = reinterpret_cast<void*>(k_accept<1024>); break;
        }
        fns[1] = reinterpret_cast<void*>(k_spawn);
    }

    int create(const abmx_traffic_config& c, const uint64_t* seeds, int roads) {
        cfg = c;
        R = roads;
        if (R < 1) {
            abmx_internal::set_error("roads must be >= 1");
            return ABMX_E_DOMAIN;
        }
        if (c.period < 1) {
            abmx_internal::set_error("signal period must be >= 1");  // traffic.cpp:9-10
            return ABMX_E_DOMAIN;
        }
        if (c.length < 1) {
            abmx_internal::set_error("road length must be >= 1");  // traffic.cpp:21-22
            return ABMX_E_DOMAIN;
        }
        if (c.length > (1 << 26)) {
            abmx_internal::set_error("road length above 2^26 cells per lane (28-bit slots)");
            return ABMX_E_CAPACITY;
        }
        CKT(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        memset(&P, 0, sizeof P);
        P.R = R;
        P.L = static_cast<int>(c.length);
        P.C = 3 * P.L;
        P.Lp = (P.L + 3) / 4 * 4;  // lane stride: aligned int4 column groups in k_accept
        P.Cpad = (3 * P.Lp + 15) / 16 * 16;
        pick_kernels();
        P.tile_slots = nt * kS;
        P.tile_cols = na * kCI;
        P.Npad = (P.C + P.tile_slots - 1) / P.tile_slots * P.tile_slots;
        P.tiles = P.Npad / P.tile_slots;
        P.Wb = P.Npad / 32;  // Npad is a multiple of tile_slots >= 128
        P.Ws = (P.Wb + 31) / 32;
        P.ctiles = (P.Lp + P.tile_cols - 1) / P.tile_cols;
        {
            int per_sm = 0;  // k_accept CTAs resident per SM
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fns[0], na, 0) != cudaSuccess) per_sm = 0;
            (void)cudaGetLastError();
            P.accept_ticketless =
                static_cast<long long>(R) * P.ctiles <= static_cast<long long>(per_sm) * abmx_internal::num_sms() ? 1 : 0;
        }
        P.period = c.period;
        long long gl = llround(static_cast<double>(c.period) * c.green_fraction);  // traffic.cpp:11-13
        P.green_len = gl < 0 ? 0 : (gl > c.period ? c.period : gl);
        int rc;
        const size_t ns = static_cast<size_t>(R) * P.Npad, nc = static_cast<size_t>(R) * P.Cpad;
#define ALT(ptr, bytes)                                                 \
    if ((rc = alloc(reinterpret_cast<void**>(&(ptr)), (bytes))) != 0) \
        return rc;
        ALT(P.active, ns);
        ALT(P.pos, ns * 4);
        ALT(P.ids, ns * 8);
        ALT(P.ages, ns * 8);
        ALT(P.occ, nc * 4);
        ALT(P.cstatus, static_cast<size_t>(R) * P.ctiles * 8 * kStatusStride);
        ALT(P.ticket, 16);
        ALT(P.fbits, static_cast<size_t>(R) * P.Wb * 4);
        ALT(P.fsum, static_cast<size_t>(R) * P.Ws * 4);
        ALT(P.exits, static_cast<size_t>(R) * 2 * sizeof(int4));
        ALT(P.cnt, static_cast<size_t>(R) * 8 * 8);
        long long* phase = nullptr;
        unsigned long long* sd = nullptr;
        ALT(phase, static_cast<size_t>(R) * 8);
        ALT(sd, static_cast<size_t>(R) * 8);
        ALT(d_metrics_step, static_cast<size_t>(R) * 4 * 8);
#undef ALT
        P.phase = phase;
        P.seeds = sd;
        std::vector<long long> ph(static_cast<size_t>(R));
        for (int r = 0; r < R; ++r) {  // phase = seed.split(TrafficSignal).uniform_int(0, 0, period)
            const unsigned long long k = abmx_dev::split(seeds[r], 5);
            const unsigned long long d = abmx_dev::draw(k, 0);
            ph[static_cast<size_t>(r)] = static_cast<long long>(
                static_cast<unsigned long long>((static_cast<unsigned __int128>(d) * static_cast<unsigned long long>(c.period)) >> 64));
        }
        CKT(cudaMemcpy(phase, ph.data(), ph.size() * 8, cudaMemcpyHostToDevice));
        CKT(cudaMemcpy(sd, seeds, static_cast<size_t>(R) * 8, cudaMemcpyHostToDevice));
        CKT(cudaMemset(P.cstatus, 0, static_cast<size_t>(R) * P.ctiles * 8 * kStatusStride));
        CKT(cudaMemset(P.ticket, 0, 16));
        CKT(cudaMemset(P.cnt, 0, static_cast<size_t>(R) * 64));
        CKT(cudaMemset(d_metrics_step, 0, static_cast<size_t>(R) * 32));
        CKT(cudaMallocHost(&h_cnt, static_cast<size_t>(R) * 64));
        (void)cudaGetLastError();
        k_init<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(P);
        abmx_internal::count_launch();
        CKT(cudaGetLastError());
        CKT(cudaStreamSynchronize(stream));
        P.metrics = d_metrics_step;
        P.metrics_stride = 1;
        return ABMX_OK;
    }

    // the folded step of a multi-step run: k_accept (+ the previous step's spawn), one kernel
    cudaGraph_t graph2 = nullptr;
    cudaGraphExec_t exec2 = nullptr;
    cudaGraphNode_t nodes2[1] = {};
    int build_graph2() {
        CKT(cudaGraphCreate(&graph2, 0));
        void* args[1] = {&P};
        for (int k = 0; k < 1; ++k) {
            cudaKernelNodeParams kp{};
            kp.func = fn(k);
            kp.gridDim = dim3(grid(k));
            kp.blockDim = dim3(block(k));
            kp.kernelParams = args;
            CKT(cudaGraphAddKernelNode(&nodes2[k], graph2, k ? &nodes2[k - 1] : nullptr, k ? 1 : 0, &kp));
        }
        CKT(cudaGraphInstantiate(&exec2, graph2, 0));
        return ABMX_OK;
    }
    // one step of a multi-step run: the spawn of step q-1 rides in step q's k_accept
    int enqueue_folded(bool pending) {
        P.epoch = host_epoch;
        P.spawn_pending = pending ? 1 : 0;
        P.spawn_t = P.t - 1;
        P.spawn_row = P.run_step - 1;
        if (!exec2) {
            int rc = build_graph2();
            if (rc) return rc;
        }
        void* args[1] = {&P};
        for (int k = 0; k < 1; ++k) {
            cudaKernelNodeParams kp{};
            kp.func = fn(k);
            kp.gridDim = dim3(grid(k));
            kp.blockDim = dim3(block(k));
            kp.kernelParams = args;
            CKT(cudaGraphExecKernelNodeSetParams(exec2, nodes2[k], &kp));
        }
        CKT(cudaGraphLaunch(exec2, stream));
        P.spawn_pending = 0;
        abmx_internal::count_launch(1);
        ++host_epoch;
        ++P.t;
        ++P.run_step;
        return ABMX_OK;
    }
    // the last step's spawn of a folded run
    int spawn_last() {
        TParams Q = P;
        Q.t = P.t - 1;
        Q.run_step = P.run_step - 1;
        Q.epoch = host_epoch - 1;
        void* args[1] = {&Q};
        CKT(cudaLaunchKernel(fn(1), dim3(grid(1)), dim3(block(1)), args, 0, stream));
        abmx_internal::count_launch(1);
        return ABMX_OK;
    }
    int build_graph() {
        CKT(cudaGraphCreate(&graph, 0));
        void* args[1] = {&P};
        for (int k = 0; k < kNumKernels; ++k) {
            cudaKernelNodeParams kp{};
            kp.func = fn(k);
            kp.gridDim = dim3(grid(k));
            kp.blockDim = dim3(block(k));
            kp.kernelParams = args;
            CKT(cudaGraphAddKernelNode(&nodes[k], graph, k ? &nodes[k - 1] : nullptr, k ? 1 : 0, &kp));
        }
        CKT(cudaGraphInstantiate(&exec, graph, 0));
        return ABMX_OK;
    }

    int enqueue(cudaEvent_t* ev) {
        P.epoch = host_epoch;
        void* args[1] = {&P};
        if (ev) {
            for (int k = 0; k < kNumKernels; ++k) {
                CKT(cudaEventRecord(ev[2 * k], stream));
                CKT(cudaLaunchKernel(fn(k), dim3(grid(k)), dim3(block(k)), args, 0, stream));
                CKT(cudaEventRecord(ev[2 * k + 1], stream));
            }
        } else {
            if (!exec) {
                int rc = build_graph();
                if (rc) return rc;
            }
            for (int k = 0; k < kNumKernels; ++k) {
                cudaKernelNodeParams kp{};
                kp.func = fn(k);
                kp.gridDim = dim3(grid(k));
                kp.blockDim = dim3(block(k));
                kp.kernelParams = args;
                CKT(cudaGraphExecKernelNodeSetParams(exec, nodes[k], &kp));
            }
            CKT(cudaGraphLaunch(exec, stream));
        }
        abmx_internal::count_launch(kNumKernels);
        ++host_epoch;
        ++P.t;
        ++P.run_step;
        return ABMX_OK;
    }

    int step(long long t) {
        P.metrics = d_metrics_step;
        P.metrics_stride = 1;
        P.run_step = 0;
        P.t = t;
        (void)cudaGetLastError();
        int rc = enqueue(nullptr);
        if (rc) return rc;
        last_run_steps = 0;
        CKT(cudaGetLastError());
        return ABMX_OK;
    }

    int prepare_run(long long t0, long long steps) {
        const size_t mb = static_cast<size_t>(R) * static_cast<size_t>(steps) * 32;
        if (mb > run_metrics_bytes) {
            CKT(cudaStreamSynchronize(stream));
            if (d_run_metrics) cudaFree(d_run_metrics);
            CKT(cudaMalloc(&d_run_metrics, mb));
            run_metrics_bytes = mb;
        }
        P.metrics = d_run_metrics;
        P.metrics_stride = static_cast<unsigned>(steps);
        P.run_step = 0;
        P.t = t0;
        return ABMX_OK;
    }

    int run(long long t0, long long steps, double* out) {
        if (steps <= 0) return ABMX_OK;
        if (steps > 0x7FFFFFFFLL) {
            abmx_internal::set_error("too many steps in one run");
            return ABMX_E_DOMAIN;
        }
        int rc = prepare_run(t0, steps);
        if (rc) return rc;
        (void)cudaGetLastError();
        for (long long q = 0; q < steps; ++q) {
            rc = enqueue_folded(q > 0);
            if (rc) return rc;
        }
        rc = spawn_last();
        if (rc) return rc;
        last_run_steps = steps;
        if (out) {
            CKT(cudaMemcpyAsync(out, d_run_metrics, static_cast<size_t>(R) * steps * 32, cudaMemcpyDeviceToHost, stream));
            CKT(cudaStreamSynchronize(stream));
        }
        return ABMX_OK;
    }

    int metrics(double* out) {
        if (last_run_steps == 0) {
            CKT(cudaMemcpyAsync(out, d_metrics_step, static_cast<size_t>(R) * 32, cudaMemcpyDeviceToHost, stream));
        } else {
            for (int r = 0; r < R; ++r)
                CKT(cudaMemcpyAsync(out + static_cast<size_t>(r) * 4,
                                    d_run_metrics + (static_cast<size_t>(r) * last_run_steps + last_run_steps - 1) * 4,
                                    32, cudaMemcpyDeviceToHost, stream));
        }
        CKT(cudaStreamSynchronize(stream));
        return ABMX_OK;
    }

    int counters(int r, long long* out8) {
        CKT(cudaMemcpyAsync(h_cnt, P.cnt + static_cast<size_t>(r) * 8, 64, cudaMemcpyDeviceToHost, stream));
        CKT(cudaStreamSynchronize(stream));
        memcpy(out8, h_cnt, 64);
        return ABMX_OK;
    }

    int export_road(int r, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* lane, int64_t* cell,
                    int32_t* occupancy, int64_t* next_id, int32_t* num_active) {
        const size_t n = static_cast<size_t>(P.C);
        const size_t sb = static_cast<size_t>(r) * P.Npad, cb = static_cast<size_t>(r) * P.Cpad;
        std::vector<int> pos(n);
        long long cn[8];
        CKT(cudaMemcpyAsync(active, P.active + sb, n, cudaMemcpyDeviceToHost, stream));
        CKT(cudaMemcpyAsync(ids, P.ids + sb, n * 8, cudaMemcpyDeviceToHost, stream));
        CKT(cudaMemcpyAsync(ages, P.ages + sb, n * 8, cudaMemcpyDeviceToHost, stream));
        CKT(cudaMemcpyAsync(pos.data(), P.pos + sb, n * 4, cudaMemcpyDeviceToHost, stream));
        std::vector<int> occ_dev(static_cast<size_t>(3 * P.Lp));
        if (occupancy) CKT(cudaMemcpyAsync(occ_dev.data(), P.occ + cb, occ_dev.size() * 4, cudaMemcpyDeviceToHost, stream));
        CKT(cudaMemcpyAsync(cn, P.cnt + static_cast<size_t>(r) * 8, 64, cudaMemcpyDeviceToHost, stream));
        CKT(cudaStreamSynchronize(stream));
        for (size_t i = 0; i < n; ++i) {
            lane[i] = pos[i] / P.Lp;
            cell[i] = pos[i] % P.Lp;
        }
        if (occupancy)
            for (int l = 0; l < 3; ++l)
                for (int c = 0; c < P.L; ++c) occupancy[l * P.L + c] = occ_dev[static_cast<size_t>(l * P.Lp + c)];
        if (next_id) *next_id = cn[1];
        if (num_active) *num_active = static_cast<int32_t>(cn[0]);
        return ABMX_OK;
    }

    int import_road(int r, const uint8_t* active, const int64_t* ids, const int64_t* ages, const int64_t* lane,
                    const int64_t* cell, int64_t next_id) {
        const size_t n = static_cast<size_t>(P.C);
        std::vector<uint8_t> act(n);
        std::vector<int> pos(n), occ(static_cast<size_t>(P.Cpad), -1);
        long long na = 0;
        for (size_t i = 0; i < n; ++i) {
            act[i] = active[i] ? 1 : 0;
            if (lane[i] < 0 || lane[i] > 2 || cell[i] < 0 || cell[i] >= P.L) {
                abmx_internal::set_error("car position outside the road");
                return ABMX_E_DOMAIN;
            }
            pos[i] = static_cast<int>(lane[i] * P.Lp + cell[i]);
            if (act[i]) {
                if (occ[static_cast<size_t>(pos[i])] != -1) {
                    abmx_internal::set_error("two cars occupy one road cell");  // traffic.cpp:40-41
                    return ABMX_E_DOMAIN;
                }
                occ[static_cast<size_t>(pos[i])] = static_cast<int>(i);
                ++na;
            }
        }
        const size_t sb = static_cast<size_t>(r) * P.Npad, cb = static_cast<size_t>(r) * P.Cpad;
        CKT(cudaStreamSynchronize(stream));
        CKT(cudaMemcpy(P.active + sb, act.data(), n, cudaMemcpyHostToDevice));
        CKT(cudaMemcpy(P.ids + sb, ids, n * 8, cudaMemcpyHostToDevice));
        CKT(cudaMemcpy(P.ages + sb, ages, n * 8, cudaMemcpyHostToDevice));
        CKT(cudaMemcpy(P.pos + sb, pos.data(), n * 4, cudaMemcpyHostToDevice));
        CKT(cudaMemcpy(P.occ + cb, occ.data(), static_cast<size_t>(P.Cpad) * 4, cudaMemcpyHostToDevice));
        long long cn[8];
        CKT(cudaMemcpy(cn, P.cnt + static_cast<size_t>(r) * 8, 64, cudaMemcpyDeviceToHost));
        cn[0] = na;
        cn[1] = next_id;
        cn[5] = 0;
        cn[7] = 0;  // low-water bitmap word
        CKT(cudaMemcpy(P.cnt + static_cast<size_t>(r) * 8, cn, 64, cudaMemcpyHostToDevice));
        // the road's free-slot bitmap and summary from the imported active flags; no exits pending
        std::vector<unsigned> fbw(static_cast<size_t>(P.Wb), 0u), fsw(static_cast<size_t>(P.Ws), 0u);
        for (size_t i = 0; i < n; ++i)
            if (!act[i]) fbw[i >> 5] |= 1u << (i & 31);
        for (int w = 0; w < P.Wb; ++w)
            if (fbw[static_cast<size_t>(w)]) fsw[static_cast<size_t>(w >> 5)] |= 1u << (w & 31);
        CKT(cudaMemcpy(P.fbits + static_cast<size_t>(r) * P.Wb, fbw.data(), fbw.size() * 4, cudaMemcpyHostToDevice));
        CKT(cudaMemcpy(P.fsum + static_cast<size_t>(r) * P.Ws, fsw.data(), fsw.size() * 4, cudaMemcpyHostToDevice));
        const int4 none[2] = {make_int4(0, -1, -1, -1), make_int4(0, -1, -1, -1)};
        CKT(cudaMemcpy(P.exits + static_cast<size_t>(r) * 2, none, sizeof none, cudaMemcpyHostToDevice));
        return ABMX_OK;
    }

    int bench(long long t0, long long steps, size_t flush_bytes, bool per_kernel, double* step_ms) {
        if (steps <= 0) return ABMX_OK;
        int rc = prepare_run(t0, steps);
        if (rc) return rc;
        if (flush_bytes > flush_cap) {
            if (flush_buf) cudaFree(flush_buf);
            CKT(cudaMalloc(&flush_buf, flush_bytes));
            flush_cap = flush_bytes;
        }
        const size_t per = per_kernel ? 2 * kNumKernels : 2;
        std::vector<cudaEvent_t> ev(per * static_cast<size_t>(steps));
        for (auto& e : ev) CKT(cudaEventCreate(&e));
        (void)cudaGetLastError();
        for (long long q = 0; q < steps; ++q) {
            if (flush_bytes) {
                CKT(cudaMemsetAsync(flush_buf, static_cast<int>(q & 0xFF), flush_bytes, stream));
                k_flush_read_t<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(
                    static_cast<const uint4*>(flush_buf), flush_bytes / 16, reinterpret_cast<unsigned*>(flush_buf));
            }
            cudaEvent_t* e = &ev[per * static_cast<size_t>(q)];
            if (per_kernel) {
                rc = enqueue(e);
            } else {  // the folded run step (the last one also takes its own spawn)
                CKT(cudaEventRecord(e[0], stream));
                rc = enqueue_folded(q > 0);
                if (!rc && q == steps - 1) rc = spawn_last();
                CKT(cudaEventRecord(e[1], stream));
            }
            if (rc) return rc;
        }
        CKT(cudaStreamSynchronize(stream));
        for (long long q = 0; q < steps; ++q) {
            cudaEvent_t* e = &ev[per * static_cast<size_t>(q)];
            float ms = 0.f;
            if (per_kernel) {
                double tot = 0.0;
                for (int k = 0; k < kNumKernels; ++k) {
                    CKT(cudaEventElapsedTime(&ms, e[2 * k], e[2 * k + 1]));
                    kernel_ms[k] += ms;
                    kernel_launches[k] += 1;
                    tot += ms;
                }
                step_ms[q] = tot;
            } else {
                CKT(cudaEventElapsedTime(&ms, e[0], e[1]));
                step_ms[q] = ms;
            }
        }
        for (auto& e : ev) cudaEventDestroy(e);
        last_run_steps = steps;
        return ABMX_OK;
    }
};

#ifdef ABMX_TRF_TRACE
extern "C" int abmx_trf_polls(unsigned* out, int ctas) {
    return cudaMemcpyFromSymbol(out, abmx_trf::g_trf_polls, sizeof(unsigned) * 2 * ctas) == cudaSuccess ? 0 : -1;
}
extern "C" int abmx_trf_warp_trace(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, abmx_trf::g_trf_warp, sizeof(unsigned long long) * 32 * 4) == cudaSuccess ? 0 : -1;
}
extern "C" int abmx_trf_trace(unsigned long long* out, int ctas) {
    return cudaMemcpyFromSymbol(out, abmx_trf::g_trf_trace, sizeof(unsigned long long) * 10 * ctas) == cudaSuccess ? 0 : -1;
}
#endif

namespace {
const char* kTrafficKernels[kNumKernels] = {"k_accept", "k_spawn"};

int resolve_host(int64_t length, const uint8_t* active, const int64_t* lane, const int64_t* cell, const uint8_t* kind,
                 const int64_t* to_lane, const int64_t* to_cell, uint8_t* accepted) {
    if (length < 1) {
        abmx_internal::set_error("road length must be >= 1");
        return ABMX_E_DOMAIN;
    }
    const int L = static_cast<int>(length), n = 3 * L;
    std::vector<uint8_t> act(static_cast<size_t>(n));
    std::vector<int> ln(static_cast<size_t>(n)), tg(static_cast<size_t>(n)), occ(static_cast<size_t>(n), -1);
    for (int i = 0; i < n; ++i) {
        act[i] = active[i] ? 1 : 0;
        ln[i] = static_cast<int>(lane[i]);
        tg[i] = kStay;
        if (!act[i]) continue;
        if (lane[i] < 0 || lane[i] > 2 || cell[i] < 0 || cell[i] >= length) {
            abmx_internal::set_error("car position outside the road");
            return ABMX_E_DOMAIN;
        }
        const int p = static_cast<int>(lane[i] * length + cell[i]);
        if (occ[p] != -1) {
            abmx_internal::set_error("two cars occupy one road cell");
            return ABMX_E_DOMAIN;
        }
        occ[p] = i;
        if (kind[i] == 2) {
            tg[i] = kExit;
        } else if (kind[i] == 1) {
            if (to_lane[i] < 0 || to_lane[i] >= 3 || to_cell[i] < 0 || to_cell[i] >= length) {
                abmx_internal::set_error("move proposal targets a cell outside the road");  // traffic.cpp:104-106
                return ABMX_E_CONTRACT;
            }
            tg[i] = static_cast<int>(to_lane[i] * length + to_cell[i]);
        }
    }
    cudaStream_t s;
    CKT(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    uint8_t *d_act = nullptr, *d_acc = nullptr;
    int *d_lane = nullptr, *d_tg = nullptr, *d_occ = nullptr, *d_a = nullptr, *d_b = nullptr;
    unsigned long long* d_bid = nullptr;
    const size_t N = static_cast<size_t>(n);
    int rc = ABMX_OK;
    auto fail = [&](cudaError_t e) {
        abmx_internal::set_error(std::string("resolve: ") + cudaGetErrorString(e));
        rc = ABMX_E_CUDA;
    };
    cudaError_t e = cudaSuccess;
    if ((e = abmx_internal::malloc_async(&d_act, N, s)) || (e = abmx_internal::malloc_async(&d_acc, N, s)) ||
        (e = abmx_internal::malloc_async(&d_lane, N * 4, s)) || (e = abmx_internal::malloc_async(&d_tg, N * 4, s)) ||
        (e = abmx_internal::malloc_async(&d_occ, N * 4, s)) || (e = abmx_internal::malloc_async(&d_a, N * 4, s)) ||
        (e = abmx_internal::malloc_async(&d_b, N * 4, s)) || (e = abmx_internal::malloc_async(&d_bid, N * 8, s))) {
        fail(e);
    } else {
        cudaMemcpyAsync(d_act, act.data(), N, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_lane, ln.data(), N * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_tg, tg.data(), N * 4, cudaMemcpyHostToDevice, s);
        cudaMemcpyAsync(d_occ, occ.data(), N * 4, cudaMemcpyHostToDevice, s);
        cudaMemsetAsync(d_bid, 0, N * 8, s);
        const int g = (n + 255) / 256;
        k_res_bid<<<g, 256, 0, s>>>(d_act, d_lane, d_tg, n, L, d_bid);
        k_res_init<<<g, 256, 0, s>>>(d_act, d_tg, d_occ, d_bid, n, d_a);
        int rounds = 1;
        while ((1 << rounds) < n + 1) ++rounds;
        for (int q = 0; q <= rounds; ++q) {
            k_res_jump<<<g, 256, 0, s>>>(d_a, d_b, n);
            int* tmp = d_a;
            d_a = d_b;
            d_b = tmp;
        }
        k_res_out<<<g, 256, 0, s>>>(d_a, n, d_acc);
        abmx_internal::count_launch(rounds + 4);
        if ((e = cudaGetLastError()) != cudaSuccess) fail(e);
        cudaMemcpyAsync(accepted, d_acc, N, cudaMemcpyDeviceToHost, s);
        if ((e = cudaStreamSynchronize(s)) != cudaSuccess) fail(e);
    }
    cudaFreeAsync(d_act, s);
    cudaFreeAsync(d_acc, s);
    cudaFreeAsync(d_lane, s);
    cudaFreeAsync(d_tg, s);
    cudaFreeAsync(d_occ, s);
    cudaFreeAsync(d_a, s);
    cudaFreeAsync(d_b, s);
    cudaFreeAsync(d_bid, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    return rc;
}
}  // namespace

#define HANDLE_T(h)                                   \
    if (!(h)) {                                       \
        abmx_internal::set_error("null traffic handle"); \
        return ABMX_E_ARG;                            \
    }

extern "C" {

int abmx_traffic_create(const abmx_traffic_config* cfg, const uint64_t* seeds, int32_t roads, abmx_traffic** out) {
    if (!cfg || !seeds || !out) {
        abmx_internal::set_error("null argument");
        return ABMX_E_ARG;
    }
    auto* h = new abmx_traffic();
    const int rc = h->create(*cfg, seeds, roads);
    if (rc) {
        delete h;
        *out = nullptr;
        return rc;
    }
    *out = h;
    return ABMX_OK;
}
int abmx_traffic_destroy(abmx_traffic* h) {
    delete h;
    return ABMX_OK;
}
int abmx_traffic_step(abmx_traffic* h, int64_t t) {
    HANDLE_T(h);
    return h->step(t);
}
int abmx_traffic_run(abmx_traffic* h, int64_t t0, int64_t steps, double* metrics_out) {
    HANDLE_T(h);
    return h->run(t0, steps, metrics_out);
}
int abmx_traffic_sync(abmx_traffic* h) {
    HANDLE_T(h);
    CKT(cudaStreamSynchronize(h->stream));
    return ABMX_OK;
}
int abmx_traffic_metrics(abmx_traffic* h, double* out) {
    HANDLE_T(h);
    return h->metrics(out);
}
int abmx_traffic_totals(abmx_traffic* h, int32_t road, int64_t* spawned_total, int64_t* exited_total) {
    HANDLE_T(h);
    if (road < 0 || road >= h->R) {
        abmx_internal::set_error("road index out of range");
        return ABMX_E_DOMAIN;
    }
    long long cn[8];
    int rc = h->counters(road, cn);
    if (rc) return rc;
    if (spawned_total) *spawned_total = cn[2];
    if (exited_total) *exited_total = cn[3];
    return ABMX_OK;
}
int abmx_traffic_schedule(abmx_traffic* h, int32_t road, int64_t* period, int64_t* green_len, int64_t* phase) {
    HANDLE_T(h);
    if (road < 0 || road >= h->R) {
        abmx_internal::set_error("road index out of range");
        return ABMX_E_DOMAIN;
    }
    long long ph = 0;
    CKT(cudaMemcpy(&ph, h->P.phase + road, 8, cudaMemcpyDeviceToHost));
    if (period) *period = h->P.period;
    if (green_len) *green_len = h->P.green_len;
    if (phase) *phase = ph;
    return ABMX_OK;
}
int abmx_traffic_export(abmx_traffic* h, int32_t road, uint8_t* active, int64_t* ids, int64_t* ages, int64_t* lane,
                        int64_t* cell, int32_t* occupancy, int64_t* next_id, int32_t* num_active) {
    HANDLE_T(h);
    if (road < 0 || road >= h->R) {
        abmx_internal::set_error("road index out of range");
        return ABMX_E_DOMAIN;
    }
    return h->export_road(road, active, ids, ages, lane, cell, occupancy, next_id, num_active);
}
int abmx_traffic_import(abmx_traffic* h, int32_t road, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                        const int64_t* lane, const int64_t* cell, int64_t next_id) {
    HANDLE_T(h);
    if (road < 0 || road >= h->R) {
        abmx_internal::set_error("road index out of range");
        return ABMX_E_DOMAIN;
    }
    return h->import_road(road, active, ids, ages, lane, cell, next_id);
}
int abmx_traffic_resolve(int64_t length, const uint8_t* active, const int64_t* lane, const int64_t* cell,
                         const uint8_t* kind, const int64_t* to_lane, const int64_t* to_cell, uint8_t* accepted) {
    return resolve_host(length, active, lane, cell, kind, to_lane, to_cell, accepted);
}
int abmx_traffic_bench(abmx_traffic* h, int64_t t0, int64_t steps, int64_t flush_bytes, int32_t per_kernel,
                       double* step_ms) {
    HANDLE_T(h);
    return h->bench(t0, steps, static_cast<size_t>(flush_bytes > 0 ? flush_bytes : 0), per_kernel != 0, step_ms);
}
int32_t abmx_traffic_kernel_count(void) { return kNumKernels; }
const char* abmx_traffic_kernel_name(int32_t k) { return (k >= 0 && k < kNumKernels) ? kTrafficKernels[k] : ""; }
int abmx_traffic_kernel_times(abmx_traffic* h, double* ms, int64_t* launches) {
    HANDLE_T(h);
    for (int k = 0; k < kNumKernels; ++k) {
        if (ms) ms[k] = h->kernel_ms[k];
        if (launches) launches[k] = h->kernel_launches[k];
    }
    return ABMX_OK;
}
int abmx_traffic_run_batch(const abmx_traffic_config* cfg, uint64_t master, int32_t replica_begin, int32_t count,
                           int64_t steps, double* metrics_out, double* kernel_ms) {
    return abmx_traffic_run_batch_path(cfg, master, replica_begin, count, steps, 0, metrics_out, kernel_ms);
}

int abmx_traffic_run_batch_path(const abmx_traffic_config* cfg, uint64_t master, int32_t replica_begin, int32_t count,
                                int64_t steps, int32_t path, double* metrics_out, double* kernel_ms) {
    if (!cfg || count < 0) {
        abmx_internal::set_error("bad run_batch arguments");
        return ABMX_E_ARG;
    }
    if (cfg->period < 1 || cfg->length < 1) {
        abmx_internal::set_error(cfg->period < 1 ? "signal period must be >= 1" : "road length must be >= 1");
        return ABMX_E_DOMAIN;
    }
    if (count == 0 || steps <= 0) return ABMX_OK;
    std::vector<uint64_t> seeds(static_cast<size_t>(count));
    const unsigned long long base = abmx_dev::split(master, 2);  // batch.cpp:12-19
    for (int32_t q = 0; q < count; ++q) seeds[static_cast<size_t>(q)] = abmx_dev::split(base, static_cast<unsigned long long>(replica_begin + q));
    const bool smem_ok = abmx_internal::traffic_ens_fits(*cfg);
    if (path == 1 && !smem_ok) {
        abmx_internal::set_error("road too long for the shared-memory path");
        return ABMX_E_CAPACITY;
    }
    if (path == 1 || (path == 0 && smem_ok))
        return abmx_internal::traffic_ensemble_run(*cfg, seeds.data(), count, steps, metrics_out, kernel_ms);
    abmx_traffic* h = nullptr;
    int rc = abmx_traffic_create(cfg, seeds.data(), count, &h);
    if (rc) return rc;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rc = h->prepare_run(1, steps);  // allocate the run rows outside the timed region
    cudaEventRecord(a, h->stream);
    if (!rc) rc = h->run(1, steps, nullptr);
    cudaEventRecord(b, h->stream);
    if (!rc && metrics_out) {
        cudaError_t e = cudaMemcpyAsync(metrics_out, h->d_run_metrics, static_cast<size_t>(count) * steps * 32,
                                        cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            abmx_internal::set_error(std::string("run_batch: ") + cudaGetErrorString(e));
            rc = ABMX_E_CUDA;
        }
    }
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (kernel_ms) *kernel_ms = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    abmx_traffic_destroy(h);
    return rc;
}

}  // extern "C"
