// agents.cu — device agent sets: the reference's generic lifecycle and subset operations on
// HBM-resident columns.
//
//   remove_agents   lifecycle.cpp:124-142 + reset_slot agent_set.cpp:45-58
//   spawn_agents    lifecycle.cpp:144-195 (rank-match of free slots and valid rows, fresh or
//                   recycled ids, age 0, optional type), copy apply of the row columns
//   set_agents_rm / set_agents_sci   kernels.cpp:116-153 with a column-copy apply: each pair
//                   writes only its own slot from its own row, so RM and SCI coincide
//   set_agents_mask kernels.cpp:155-167 (independent per-slot writes)
//   select_agents   compact_mask kernels.cpp:23-35 (stable partition, trues first)
//   sort_agents     kernels.cpp:52-73: stable LSD radix sort of order-preserving 64-bit keys,
//                   then permute_agents (agent_set.cpp:92-108)
//
// Every pass is an HBM-streaming integer kernel: ticket-ordered single-pass selection with
// decoupled lookback, then a gather/scatter over the selected pairs only. Counts stay in
// device memory, so a whole remove -> spawn cycle is stream-ordered with no host round trip.
#include <cmath>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/abmx_cuda.h"
#include "abmx_device.cuh"
#include "abmx_internal.h"

using namespace abmx_dev;

namespace abmx_agents {

constexpr int kT = 256;
constexpr int kItems = 16;
constexpr int kTile = kT * kItems;
constexpr int kMaxCols = 12;  // columns per launch (more are processed in chunks)

struct Cols {  // kernel-parameter column list: dst[c][slot] <- src[c][row]
    void* dst[kMaxCols];
    const void* src[kMaxCols];
    int sz[kMaxCols];
    int n;
};

struct ScanWs {
    unsigned ticket;
    unsigned pad;
    unsigned long long status[1];  // [tiles]
};

__device__ __forceinline__ unsigned long long load_elem(const void* src, long long j, int sz) {
    if (sz == 8) return static_cast<const unsigned long long*>(src)[j];
    if (sz == 4) return static_cast<const unsigned*>(src)[j];
    return static_cast<const uint8_t*>(src)[j];
}
__device__ __forceinline__ void store_elem(void* dst, long long i, unsigned long long v, int sz) {
    if (sz == 8)
        static_cast<unsigned long long*>(dst)[i] = v;
    else if (sz == 4)
        static_cast<unsigned*>(dst)[i] = static_cast<unsigned>(v);
    else
        static_cast<uint8_t*>(dst)[i] = static_cast<uint8_t>(v);
}
// dst[c][slot] <- src[c][row] for every column with a source: all loads issued before the first
// store (a store may alias a later column's source as far as the compiler knows, so the plain
// per-column copy serialises one random DRAM round trip per column)
__device__ __forceinline__ void copy_cols(const Cols& C, long long slot, long long row) {
    unsigned long long v[kMaxCols];
#pragma unroll
    for (int c = 0; c < kMaxCols; ++c)
        if (c < C.n && C.src[c]) v[c] = load_elem(C.src[c], row, C.sz[c]);
#pragma unroll
    for (int c = 0; c < kMaxCols; ++c)
        if (c < C.n && C.src[c]) store_elem(C.dst[c], slot, v[c], C.sz[c]);
}
__device__ __forceinline__ void zero_elem(void* dst, long long i, int sz) {
    if (sz == 8)
        static_cast<unsigned long long*>(dst)[i] = 0ULL;
    else if (sz == 4)
        static_cast<unsigned*>(dst)[i] = 0u;
    else
        static_cast<uint8_t*>(dst)[i] = 0;
}

__device__ __forceinline__ void load16(const uint8_t* p, size_t base, size_t n, uint8_t (&b)[kItems]) {
    if (p == nullptr) {
#pragma unroll
        for (int k = 0; k < kItems; ++k) b[k] = 0;
        return;
    }
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0 && base + kItems <= n) {
        const uint4 v = *reinterpret_cast<const uint4*>(p + base);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < kItems; ++k) b[k] = static_cast<uint8_t>(w[k >> 2] >> (8 * (k & 3)));
    } else {
#pragma unroll
        for (int k = 0; k < kItems; ++k) b[k] = base + k < n ? p[base + k] : 0;
    }
}

enum SelMode { kSelMask = 0, kSelFree = 1, kSelKill = 2 };

// list[k] = k-th selected index in ascending order; *count = number selected (last tile).
//   kSelMask: mask[i] != 0      kSelFree: active[i] == 0      kSelKill: active[i] && mask[i]
template <int kMode>
__device__ __forceinline__ void select_tile(const uint8_t* __restrict__ mask, const uint8_t* __restrict__ active,
                                            size_t n, int32_t* __restrict__ list, long long* __restrict__ count,
                                            ScanWs* ws, unsigned tiles) {
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_look[kT / 32 + 2];
    if (threadIdx.x == 0) s_tile = atomicAdd(&ws->ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const size_t base = static_cast<size_t>(tile) * kTile + static_cast<size_t>(threadIdx.x) * kItems;
    uint8_t m[kItems], a[kItems];
    load16(kMode == kSelFree ? nullptr : mask, base, n, m);
    load16(kMode == kSelMask ? nullptr : active, base, n, a);
    bool sel[kItems];
    unsigned cnt = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const bool in = base + k < n;
        sel[k] = in && (kMode == kSelMask ? m[k] != 0 : kMode == kSelFree ? a[k] == 0 : (a[k] != 0 && m[k] != 0));
        cnt += sel[k];
    }
    unsigned long long total;
    const unsigned long long excl = block_excl_scan<kT>(cnt, s_scan, &total);
    __syncthreads();
    const unsigned long long pre = block_lookback<kT>(ws->status, static_cast<int>(tile), total, s_look);
    unsigned long long pos = pre + excl;
#pragma unroll
    for (int k = 0; k < kItems; ++k)
        if (sel[k]) list[pos++] = static_cast<int32_t>(base + k);
    if (tile == tiles - 1 && threadIdx.x == 0) *count = static_cast<long long>(pre + total);
}

template <int kMode>
__global__ void __launch_bounds__(kT) k_select(const uint8_t* __restrict__ mask, const uint8_t* __restrict__ active,
                                               size_t n, int32_t* __restrict__ list, long long* __restrict__ count,
                                               ScanWs* ws) {
    select_tile<kMode>(mask, active, n, list, count, ws, gridDim.x);
}

// spawn_agents' two independent selections in one launch: the free slots (blocks [0, ta)) and
// the valid rows (blocks [ta, ta + tb)), each with its own ticket counter and lookback words
__global__ void __launch_bounds__(kT) k_select_spawn(const uint8_t* __restrict__ active, size_t n,
                                                     int32_t* __restrict__ slots, long long* cnt_slots, ScanWs* wa,
                                                     unsigned ta, const uint8_t* __restrict__ valid, size_t m,
                                                     int32_t* __restrict__ rows, long long* cnt_rows, ScanWs* wb) {
    if (blockIdx.x < ta)
        select_tile<kSelFree>(nullptr, active, n, slots, cnt_slots, wa, ta);
    else
        select_tile<kSelMask>(valid, nullptr, m, rows, cnt_rows, wb, gridDim.x - ta);
}

struct Life {  // lifecycle fields of a set (agent_set.hpp:15-77)
    uint8_t* active;
    long long* ids;
    long long* ages;
    long long* types;
    long long* counters;  // [3]: num_active, next_id, retired count
    long long* retired;   // retired-id stack (recycle only)
    int recycle;
};

// The last CTA of a kernel to pass here returns true (all others' writes visible). `done` is a
// zeroed word of the call's scan workspace; null: not the call's last kernel.
__device__ __forceinline__ bool last_cta(unsigned* done) {
    __shared__ unsigned s_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(done, 1u) == gridDim.x - 1 ? 1u : 0u;
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0;
}

// Counters after a spawn (lifecycle.cpp:186-194); out = {spawned, dropped}.
__device__ __forceinline__ void spawn_commit(const long long* p, const long long* q, const Life& L, long long* out) {
    const long long r = min(*p, *q);
    const long long top = L.recycle ? L.counters[2] : 0;
    const long long used = min(top, r);
    L.counters[0] += r;
    L.counters[1] += r - used;
    if (L.recycle) L.counters[2] = top - used;
    if (out) {
        out[0] = r;
        out[1] = *q - r;
    }
}
__device__ __forceinline__ void remove_commit(const long long* count, const Life& L, long long* out) {
    const long long nk = *count;
    L.counters[0] -= nk;
    if (L.recycle) L.counters[2] += nk;
    if (out) *out = nk;
}

// Pair k (k < min(*p, *q)): slot = slots[k] <- row = rows[k]. With `spawn` the slot also
// becomes a fresh agent (lifecycle.cpp:170-185): active, id (recycled LIFO first), age 0, type.
__global__ void __launch_bounds__(kT) k_pair_apply(const int32_t* __restrict__ slots, const int32_t* __restrict__ rows,
                                                   const long long* p, const long long* q, Cols C, int spawn,
                                                   Life L, int set_type, long long agent_type, unsigned* done,
                                                   long long* out) {
    const long long r = min(*p, *q);
    long long top = 0, nid = 0;
    if (spawn) {
        nid = L.counters[1];
        top = L.recycle ? L.counters[2] : 0;
    }
    for (long long k = static_cast<long long>(blockIdx.x) * kT + threadIdx.x; k < r;
         k += static_cast<long long>(gridDim.x) * kT) {
        const int slot = slots[k], row = rows[k];
        copy_cols(C, slot, row);
        if (spawn) {
            L.active[slot] = 1;
            L.ids[slot] = k < top ? L.retired[top - 1 - k] : nid + (k - top);
            L.ages[slot] = 0;
            if (set_type) L.types[slot] = agent_type;
        }
    }
    if (done && last_cta(done) && threadIdx.x == 0) {  // the call's last kernel: commit
        if (spawn)
            spawn_commit(p, q, L, out);
        else if (out) {
            out[0] = r;
            out[1] = *q;
        }
    }
}

__global__ void k_spawn_commit(const long long* p, const long long* q, Life L, long long* out) {
    spawn_commit(p, q, L, out);
}

// {pairs, valid rows} of a set_agents_rm / _sci call
__global__ void k_pair_result(const long long* p, const long long* q, long long* out) {
    const long long r = min(*p, *q);
    out[0] = r;
    out[1] = *q;
}

// remove_agents: killed slot k of the slot-ordered kill list is reset; its id is pushed on
// the retired stack at top + k (the reference pushes in ascending slot order).
__global__ void __launch_bounds__(kT) k_remove_apply(const int32_t* __restrict__ list, const long long* count,
                                                     Cols C, Life L, unsigned* done, Life LC, long long* out) {
    const long long nk = *count;
    const long long top = L.recycle ? L.counters[2] : 0;
    for (long long k = static_cast<long long>(blockIdx.x) * kT + threadIdx.x; k < nk;
         k += static_cast<long long>(gridDim.x) * kT) {
        const int slot = list[k];
        if (L.recycle) L.retired[top + k] = L.ids[slot];
        L.active[slot] = 0;
        L.ids[slot] = 0;
        L.ages[slot] = 0;
        for (int c = 0; c < C.n; ++c) zero_elem(C.dst[c], slot, C.sz[c]);
    }
    if (done && last_cta(done) && threadIdx.x == 0) remove_commit(count, LC, out);  // the call's last kernel
}
__global__ void k_remove_commit(const long long* count, Life L, long long* out) { remove_commit(count, L, out); }

// ---------------------------------------------------------------- fused lifecycle cycle
// remove_agents(kill) then spawn_agents(rows, valid) (lifecycle.cpp:124-195) in TWO kernels:
//   k_life_select  one ticketed single pass over the slot tiles and the row tiles. A slot tile
//                  counts (killed, free-after-removal) packed, looks back once, resets its killed
//                  slots on the spot (the retired push goes to top + killed prefix: slot order)
//                  and lists its free slots; a row tile lists its valid rows.
//   k_life_apply   pair k < min(F, Q): the k-th free slot takes the k-th valid row; ids pop the
//                  retired stack (now top + K deep) LIFO first; the last CTA commits the counters.
struct LifeCounts {  // written by the last slot / row tile
    long long free_, valid, killed;
};

__global__ void __launch_bounds__(kT) k_life_select(const uint8_t* __restrict__ kill, size_t n, int32_t* __restrict__ slots,
                                                    ScanWs* wa, unsigned ta, const uint8_t* __restrict__ valid, size_t m,
                                                    int32_t* __restrict__ rows, ScanWs* wb, Cols C, Life L,
                                                    LifeCounts* cnt) {
    if (blockIdx.x >= ta) {  // row tiles: the valid rows, slot order
        select_tile<kSelMask>(valid, nullptr, m, rows, &cnt->valid, wb, gridDim.x - ta);
        return;
    }
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_look[kT / 32 + 2];
    if (threadIdx.x == 0) s_tile = atomicAdd(&wa->ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const size_t base = static_cast<size_t>(tile) * kTile + static_cast<size_t>(threadIdx.x) * kItems;
    uint8_t kk[kItems], a[kItems];
    load16(kill, base, n, kk);
    load16(L.active, base, n, a);
    bool killed[kItems], fr[kItems];
    unsigned nk = 0, nf = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const bool in = base + k < n;
        killed[k] = in && a[k] != 0 && kk[k] != 0;
        fr[k] = in && (a[k] == 0 || killed[k]);  // free once the removal is done
        nk += killed[k];
        nf += fr[k];
    }
    unsigned long long total;
    const unsigned long long excl = block_excl_scan<kT>(pack2(nk, nf), s_scan, &total);
    __syncthreads();
    const unsigned long long pre = block_lookback<kT>(wa->status, static_cast<int>(tile), total, s_look);
    const long long top = L.recycle ? L.counters[2] : 0;
    long long kpos = static_cast<long long>(hi31(pre)) + hi31(excl);  // killed before this thread
    long long fpos = static_cast<long long>(lo31(pre)) + lo31(excl);      // free before this thread
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
        const size_t slot = base + k;
        if (killed[k]) {  // remove_agents: reset_slot (type kept), push the id
            if (L.recycle) L.retired[top + kpos] = L.ids[slot];
            ++kpos;
            L.active[slot] = 0;
            L.ids[slot] = 0;
            L.ages[slot] = 0;
            for (int c = 0; c < C.n; ++c) zero_elem(C.dst[c], static_cast<long long>(slot), C.sz[c]);
        }
        if (fr[k]) slots[fpos++] = static_cast<int32_t>(slot);
    }
    if (tile == ta - 1 && threadIdx.x == 0) {
        cnt->killed = static_cast<long long>(hi31(pre) + hi31(total));
        cnt->free_ = static_cast<long long>(lo31(pre) + lo31(total));
    }
}

__global__ void __launch_bounds__(kT) k_life_apply(const int32_t* __restrict__ slots, const int32_t* __restrict__ rows,
                                                   const LifeCounts* cnt, Cols C, Life L, int set_type,
                                                   long long agent_type, unsigned* done, long long* out_killed,
                                                   long long* out) {
    const long long K = cnt->killed;
    const long long r = min(cnt->free_, cnt->valid);
    const long long nid = L.counters[1];
    const long long top = (L.recycle ? L.counters[2] : 0) + (L.recycle ? K : 0);  // after the pushes
    for (long long k = static_cast<long long>(blockIdx.x) * kT + threadIdx.x; k < r;
         k += static_cast<long long>(gridDim.x) * kT) {
        const int slot = slots[k], row = rows[k];
        copy_cols(C, slot, row);
        L.active[slot] = 1;
        L.ids[slot] = k < top ? L.retired[top - 1 - k] : nid + (k - top);
        L.ages[slot] = 0;
        if (set_type) L.types[slot] = agent_type;
    }
    if (last_cta(done) && threadIdx.x == 0) {  // counters (lifecycle.cpp:136-141, 186-194)
        const long long used = min(top, r);
        L.counters[0] += r - K;
        L.counters[1] += r - used;
        if (L.recycle) L.counters[2] = top - used;
        if (out_killed) *out_killed = K;
        if (out) {
            out[0] = r;
            out[1] = cnt->valid - r;
        }
    }
}

// The same cycle as ONE cooperative kernel with ONE grid barrier, when every tile CTA is
// co-resident (k_life_coop):
//   count   each CTA (one slot or row tile) counts (killed, free) or valid; a slot tile also
//           writes its tile-local lists (free slots by local rank, and the ids of its killed
//           slots by local kill rank), which need no global information; every CTA publishes
//           its totals and arrives at the barrier (a release increment; thread 0 alone polls)
//   resolve every CTA scans all tile totals into shared memory: K (killed), F (free), Q (valid),
//           r = min(F, Q), its own prefix, and the per-slot-tile prefixes that map a global free
//           rank (or kill rank) to (tile, local rank) by binary search
//   write   slot tiles push their killed ids (retired[top + kill rank]) and reset their killed
//           slots; a killed slot of free rank < r is refilled this cycle, so only the state
//           columns the spawn does not write are zeroed there. Row tiles place their valid rows
//           of rank q < r directly: the q-th free slot from the tile lists, the id popped LIFO
//           (an id pushed this cycle comes from the killed-id lists, not from retired[], which
//           another CTA may still be writing). The reset and the placement write disjoint words.
// Block 0 commits the counters after the barrier (every CTA read the old ones before it).
// One counter barrier replaces the ticket + lookback of k_life_select, the last-CTA handshake of
// k_life_apply, and the second barrier + slot/row pair lists of the previous two-barrier kernel.
#ifdef ABMX_LIFE_TRACE  // per-CTA %globaltimer stamps: start, counted, barrier, written, -, end, resolved
__device__ unsigned long long g_life_trace[4096][8];
#define LIFE_STAMP(k)                                                          \
    if (threadIdx.x == 0) {                                                    \
        unsigned long long t_;                                                 \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
        if (blockIdx.x < 4096) g_life_trace[blockIdx.x][k] = t_;               \
    }
#else
#define LIFE_STAMP(k)
#endif

#ifndef ABMX_BAR_NS
#define ABMX_BAR_NS 100
#endif
constexpr int kCoopMaxTiles = 2048;  // slot + row tiles of one k_life_coop grid (shared prefix array)

struct LifeWs {
    unsigned arrived;           // CTAs past the count phase (zeroed before the launch)
    unsigned pad;
    unsigned long long tot[1];  // [G] pack2(killed, free) (slot tile) or pack2(0, valid) (row tile)
};

__device__ __forceinline__ void grid_barrier(unsigned* ctr, unsigned G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        red_release_add(ctr, 1u);
        while (ld_acquire_u32(ctr) < G) {
#if ABMX_BAR_NS > 0
            __nanosleep(ABMX_BAR_NS);  // back off: every CTA's thread 0 polls this one line
#endif
        }
    }
    __syncthreads();
}

// largest t in [0, cnt) with field(pref[t]) <= q: the tile holding global rank q (empty tiles
// share their successor's prefix and are skipped by taking the last such t)
template <bool kHi>
__device__ __forceinline__ unsigned tile_of_rank(const unsigned long long* pref, unsigned cnt, unsigned long long q) {
    unsigned lo = 0, hi = cnt;  // answer in [lo, hi)
    while (hi - lo > 1) {
        const unsigned mid = (lo + hi) >> 1;
        const unsigned v = kHi ? hi31(pref[mid]) : lo31(pref[mid]);
        if (v <= q)
            lo = mid;
        else
            hi = mid;
    }
    return lo;
}

__global__ void __launch_bounds__(kT) k_life_coop(const uint8_t* __restrict__ kill, size_t n, unsigned ta,
                                                  const uint8_t* __restrict__ valid, size_t m,
                                                  int32_t* __restrict__ free_list, long long* __restrict__ kill_ids,
                                                  LifeWs* ws, Cols Z, unsigned z_refill, Cols A, Life L, int set_type,
                                                  long long agent_type, long long* out_killed, long long* out,
                                                  int32_t* pair_slots, int32_t* pair_rows, int rm) {
    // rm != 0: set_agents_rm / _sci with the copy apply (kernels.cpp:116-153): `kill` is the
    // target mask, the k-th target slot takes the k-th valid row, and nothing else changes (no
    // removal, no lifecycle fields, no counters); out = {pairs, valid rows}
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ unsigned long long s_pref[kCoopMaxTiles + 1];  // exclusive tile prefixes, [G] = total
    __shared__ long long s_cnt[3];
    __shared__ int32_t s_rows[kTile];  // row tile: its valid rows, by local rank
    const unsigned G = gridDim.x, b = blockIdx.x;
    const int tid = threadIdx.x;
    LIFE_STAMP(0);
    const bool slot_tile = b < ta;
    const size_t tile_base = static_cast<size_t>(slot_tile ? b : b - ta) * kTile;
    const size_t base = tile_base + static_cast<size_t>(tid) * kItems;
    // the counters before the cycle (block 0 rewrites them after the barrier), read into shared
    // memory at kernel start: left in registers, the compiler sank the loads past the barrier,
    // a cold DRAM round trip on the critical path
    if (tid == 0) {
        s_cnt[0] = L.counters[0];
        s_cnt[1] = L.counters[1];
        s_cnt[2] = L.recycle ? L.counters[2] : 0;
    }
    // ---- count
    // bit k of m1 / m2: slot tile: killed / free once removed; row tile: - / valid. Bit masks
    // keep the per-slot flags in two registers, so the loops over them stay rolled and visit
    // only the set bits (the unrolled 16-way version was ~3 µs slower in the trace)
    unsigned m1 = 0, m2 = 0;
    unsigned c1 = 0, c2 = 0;
    {
        uint8_t x[kItems], a[kItems];
        load16(slot_tile ? kill : valid, base, slot_tile ? n : m, x);
        load16(slot_tile && !rm ? L.active : nullptr, base, n, a);
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
            const bool in = base + k < (slot_tile ? n : m);
            const bool k1 = !rm && slot_tile && in && a[k] != 0 && x[k] != 0;
            const bool k2 = in && (slot_tile && !rm ? (a[k] == 0 || k1) : x[k] != 0);
            m1 |= static_cast<unsigned>(k1) << k;
            m2 |= static_cast<unsigned>(k2) << k;
            c1 += k1;
            c2 += k2;
        }
    }
    if (L.recycle)  // the killed slots' ids are read below, after the scan: start them now
        for (unsigned mm = m1; mm; mm &= mm - 1) prefetch_l2(L.ids + base + (__ffs(static_cast<int>(mm)) - 1));
    unsigned long long total;
    const unsigned long long excl = block_excl_scan<kT>(pack2(c1, c2), s_scan, &total);
    if (slot_tile) {  // tile-local lists: free slots (killed included; only when rows follow) and
                      // killed ids, in slot order
        unsigned lf = lo31(excl), lk = hi31(excl);
#pragma unroll 1
        for (unsigned mm = G > ta ? m2 : m1; mm; mm &= mm - 1) {
            const unsigned k = static_cast<unsigned>(__ffs(static_cast<int>(mm)) - 1);
            if (G > ta) free_list[tile_base + lf++] = static_cast<int32_t>(base + k);
            if (L.recycle && ((m1 >> k) & 1u)) kill_ids[tile_base + lk++] = L.ids[base + k];
        }
    } else {  // the tile's valid rows in shared memory (placed one per thread after the barrier);
              // their row values start towards L2 now
        unsigned lv = lo31(excl);
#pragma unroll 1
        for (unsigned mm = m2; mm; mm &= mm - 1) {
            const size_t row = base + static_cast<unsigned>(__ffs(static_cast<int>(mm)) - 1);
            s_rows[lv++] = static_cast<int32_t>(row);
            for (int c = 0; c < A.n; ++c)
                if (A.src[c]) prefetch_l2(static_cast<const uint8_t*>(A.src[c]) + row * A.sz[c]);
        }
    }
    if (tid == 0) ws->tot[b] = total;
    LIFE_STAMP(1);
    grid_barrier(&ws->arrived, G);
    LIFE_STAMP(2);
    // ---- resolve: exclusive prefixes over all tiles (slot tiles first: the lo field of a row
    // tile's prefix is F + its valid prefix; F + Q < 2^31 since the grid is co-resident)
    {
        // the totals come in lane-contiguous (coalesced) loads, staged in s_pref: every CTA reads
        // the same few lines, so each load instruction should touch as few of them as possible
        constexpr int kPer = (kCoopMaxTiles + kT - 1) / kT;
        for (unsigned q = tid; q < G; q += kT) s_pref[q] = ws->tot[q];
        __syncthreads();
        unsigned long long v[kPer], sum = 0;
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const unsigned q = static_cast<unsigned>(tid) * kPer + e;
            v[e] = q < G ? s_pref[q] : 0ULL;
            sum += v[e];
        }
        unsigned long long all;
        unsigned long long run = block_excl_scan<kT>(sum, s_scan, &all);
#pragma unroll
        for (int e = 0; e < kPer; ++e) {
            const unsigned q = static_cast<unsigned>(tid) * kPer + e;
            if (q < G) s_pref[q] = run;
            run += v[e];
        }
        if (tid == 0) s_pref[G] = all;
        __syncthreads();
    }
    const unsigned long long at_ta = s_pref[ta];
    const unsigned long long K = hi31(at_ta), F = lo31(at_ta), Q = lo31(s_pref[G]) - F;
    ABMX_ASSERT(G <= static_cast<unsigned>(kCoopMaxTiles) && F <= n && K <= F && Q <= m);
    const long long r = static_cast<long long>(F < Q ? F : Q);
    const long long live0 = s_cnt[0], nid = s_cnt[1], top0 = s_cnt[2];
    const long long top = top0 + (L.recycle ? static_cast<long long>(K) : 0);  // after the pushes
    LIFE_STAMP(6);
    if (b == 0 && tid == 0) {  // counters (lifecycle.cpp:136-141, 186-194)
        const long long used = top < r ? top : r;
        if (!rm) {
            L.counters[0] = live0 - static_cast<long long>(K) + r;
            L.counters[1] = nid + r - used;
            if (L.recycle) L.counters[2] = top - used;
        }
        if (out_killed) *out_killed = static_cast<long long>(K);
        if (out) {
            out[0] = r;
            out[1] = static_cast<long long>(Q) - (rm ? 0 : r);
        }
    }
    // ---- write
    const unsigned long long own = s_pref[b];
    if (slot_tile) {  // remove_agents: reset_slot (type kept), push the id (slot order)
        const long long kpos0 = static_cast<long long>(hi31(own)) + hi31(excl);
        const long long fpos0 = static_cast<long long>(lo31(own)) + lo31(excl);
#pragma unroll 1
        for (unsigned mm = m1; mm; mm &= mm - 1) {
            const unsigned k = static_cast<unsigned>(__ffs(static_cast<int>(mm)) - 1);
            const unsigned below = (1u << k) - 1u;
            const size_t i = base + k;
            const unsigned lk = hi31(excl) + __popc(m1 & below);
            if (L.recycle) L.retired[top0 + kpos0 + __popc(m1 & below)] = kill_ids[tile_base + lk];
            if (fpos0 + __popc(m2 & below) < r) {  // refilled below: zero what the spawn leaves
                for (int c = 0; c < Z.n; ++c)
                    if ((z_refill >> c) & 1u) zero_elem(Z.dst[c], static_cast<long long>(i), Z.sz[c]);
            } else {
                L.active[i] = 0;
                L.ids[i] = 0;
                L.ages[i] = 0;
                for (int c = 0; c < Z.n; ++c) zero_elem(Z.dst[c], static_cast<long long>(i), Z.sz[c]);
            }
        }
    } else {  // spawn_agents: the q-th valid row fills the q-th free slot (tile rows over the threads)
        const long long q0 = static_cast<long long>(lo31(own)) - static_cast<long long>(F);
        const long long cnt = static_cast<long long>(lo31(total)) < r - q0 ? lo31(total) : r - q0;
#pragma unroll 1
        for (long long j = tid; j < cnt; j += kT) {
            const long long q = q0 + j;
            const int row = s_rows[j];
            const unsigned t = tile_of_rank<false>(s_pref, ta, static_cast<unsigned long long>(q));
            ABMX_ASSERT(t < ta && q >= lo31(s_pref[t]) && q < lo31(s_pref[t + 1]) && q < r);
            const int slot = free_list[static_cast<size_t>(t) * kTile + (q - lo31(s_pref[t]))];
            ABMX_ASSERT(slot >= 0 && static_cast<size_t>(slot) < n && static_cast<size_t>(row) < m);
            long long id = nid + (q - top);
            if (!rm && q < top) {
                const long long e = top - 1 - q;  // stack entry popped
                if (e >= top0) {                  // pushed this cycle: killed id of kill rank e - top0
                    const unsigned long long j = static_cast<unsigned long long>(e - top0);
                    const unsigned t2 = tile_of_rank<true>(s_pref, ta, j);
                    ABMX_ASSERT(t2 < ta && j >= hi31(s_pref[t2]) && j < hi31(s_pref[t2 + 1]));
                    id = kill_ids[static_cast<size_t>(t2) * kTile + (j - hi31(s_pref[t2]))];
                } else {
                    id = L.retired[e];
                }
            }
            copy_cols(A, slot, static_cast<long long>(row));
            if (pair_slots) pair_slots[q] = slot;  // spawn_agents' pair lists (abmx_agents_spawn)
            if (pair_rows) pair_rows[q] = row;
            if (rm) continue;
            L.active[slot] = 1;
            L.ids[slot] = id;
            L.ages[slot] = 0;
            if (set_type) L.types[slot] = agent_type;
        }
    }
    LIFE_STAMP(5);
}

// set_agents_mask with per-slot source values: dst[c][i] <- src[c][i] where mask[i].
__global__ void __launch_bounds__(kT) k_mask_apply(const uint8_t* __restrict__ mask, size_t n, Cols C) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * kT + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * kT)
        if (mask[i]) copy_cols(C, static_cast<long long>(i), static_cast<long long>(i));
}

// gather: dst[c][i] <- src[c][perm[i]] (permute_agents, agent_set.cpp:92-108)
__global__ void __launch_bounds__(kT) k_gather(const int32_t* __restrict__ perm, size_t n, Cols C) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * kT + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * kT) {
        const int j = perm[i];
        copy_cols(C, static_cast<long long>(i), j);  // every gather column has a source
    }
}
__global__ void k_check_perm(const int32_t* __restrict__ perm, size_t n, unsigned* bad) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        if (perm[i] < 0 || static_cast<size_t>(perm[i]) >= n) atomicOr(bad, 1u);
}

// ------------------------------------------------------------------ stable radix sort
// Order-preserving key: -0.0 folds onto +0.0 (they compare equal under `<`), negatives are
// bit-inverted, positives get the sign bit; descending inverts the result, so equal keys keep
// slot order either way (std::stable_sort). NaN keys (placeholders only: an active slot with
// a non-finite key is rejected) sort beyond +/-inf by their sign bit.
__global__ void __launch_bounds__(kT) k_sort_keys(const double* __restrict__ key, const uint8_t* __restrict__ active,
                                                  size_t n, int descending, unsigned long long* __restrict__ keys,
                                                  int32_t* __restrict__ vals, unsigned* bad) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * kT + threadIdx.x; i < n; i += static_cast<size_t>(gridDim.x) * kT) {
        double k = key[i];
        if (active[i] && !isfinite(k)) atomicOr(bad, 1u);
        if (k == 0.0) k = 0.0;
        unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(k));
        u = (u >> 63) ? ~u : (u | (1ULL << 63));
        keys[i] = descending ? ~u : u;
        vals[i] = static_cast<int32_t>(i);
    }
}

// per-tile digit histogram, digit-major: hist[d * tiles + tile]
__global__ void __launch_bounds__(kT) k_hist(const unsigned long long* __restrict__ keys, size_t n, int shift,
                                             unsigned* __restrict__ hist, int tiles) {
    __shared__ unsigned h[256];
    h[threadIdx.x] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(blockIdx.x) * kTile;
#pragma unroll 4
    for (int j = 0; j < kItems; ++j) {
        const size_t i = base + static_cast<size_t>(j) * kT + threadIdx.x;
        if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
    }
    __syncthreads();
    hist[static_cast<size_t>(threadIdx.x) * tiles + blockIdx.x] = h[threadIdx.x];
}

// one CTA per digit: exclusive scan of that digit's tile counts; total -> dtot[d]
__global__ void __launch_bounds__(kT) k_digit_scan(unsigned* __restrict__ hist, int tiles, unsigned* __restrict__ dtot) {
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    unsigned* h = hist + static_cast<size_t>(blockIdx.x) * tiles;
    unsigned long long carry = 0;
    for (int t0 = 0; t0 < tiles; t0 += kT) {
        const int t = t0 + threadIdx.x;
        const unsigned v = t < tiles ? h[t] : 0u;
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan<kT>(v, s_scan, &tot);
        if (t < tiles) h[t] = static_cast<unsigned>(carry + ex);
        carry += tot;
        __syncthreads();
    }
    if (threadIdx.x == 0) dtot[blockIdx.x] = static_cast<unsigned>(carry);
}

// Stable scatter of one tile. Keys are visited in kItems rounds of kT consecutive keys
// (round-major = index order); within a round, warps are ordered and lanes ranked by
// __match_any_sync, so equal digits keep their input order.
__global__ void __launch_bounds__(kT) k_scatter(const unsigned long long* __restrict__ kin, const int32_t* __restrict__ vin,
                                                unsigned long long* __restrict__ kout, int32_t* __restrict__ vout,
                                                size_t n, int shift, const unsigned* __restrict__ hist,
                                                const unsigned* __restrict__ dtot, int tiles) {
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ unsigned s_base[256];
    __shared__ unsigned s_w[kT / 32][256];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    {
        unsigned long long tot;
        const unsigned long long ex = block_excl_scan<kT>(dtot[tid], s_scan, &tot);
        s_base[tid] = static_cast<unsigned>(ex) + hist[static_cast<size_t>(tid) * tiles + blockIdx.x];
    }
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) s_w[w][tid] = 0;
    __syncthreads();
    const size_t base = static_cast<size_t>(blockIdx.x) * kTile;
    for (int j = 0; j < kItems; ++j) {
        const size_t i = base + static_cast<size_t>(j) * kT + tid;
        const bool ok = i < n;
        unsigned long long key = 0;
        int32_t val = 0;
        if (ok) {
            key = kin[i];
            val = vin[i];
        }
        const unsigned d = ok ? static_cast<unsigned>((key >> shift) & 255) : 256u;
        const unsigned peers = __match_any_sync(0xffffffffu, d);
        const unsigned rank = __popc(peers & ((1u << lane) - 1u));
        if (ok && rank == 0) s_w[warp][d] = __popc(peers);
        __syncthreads();
        unsigned run = 0;
#pragma unroll
        for (int w = 0; w < kT / 32; ++w) {
            const unsigned c = s_w[w][tid];
            s_w[w][tid] = run;
            run += c;
        }
        __syncthreads();
        if (ok) {
            const unsigned pos = s_base[d] + s_w[warp][d] + rank;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
        s_base[tid] += run;
#pragma unroll
        for (int w = 0; w < kT / 32; ++w) s_w[w][tid] = 0;
        __syncthreads();
    }
}

}  // namespace abmx_agents

// ====================================================================== host side
using namespace abmx_agents;

namespace {

#define CKA(x)                                                                        \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            abmx_internal::set_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
            return ABMX_E_CUDA;                                                       \
        }                                                                             \
    } while (0)

int grid_for(size_t n) {
    const size_t g = (n + kT - 1) / kT;
    const size_t cap = static_cast<size_t>(abmx_internal::num_sms()) * 8;
    return static_cast<int>(g < cap ? (g > 0 ? g : 1) : cap);
}

bool elem_ok(int sz) { return sz == 1 || sz == 4 || sz == 8; }

int check_set(const abmx_agent_set* s) {
    if (!s) {
        abmx_internal::set_error("null agent set");
        return ABMX_E_ARG;
    }
    if (s->capacity < 0) {
        abmx_internal::set_error("negative capacity");  // agent_set.cpp:27-28
        return ABMX_E_CAPACITY;
    }
    if (s->capacity > 0 && (!s->active || !s->ids || !s->ages || !s->types || !s->counters)) {
        abmx_internal::set_error("agent set is missing a lifecycle column");
        return ABMX_E_SCHEMA;
    }
    if (s->recycle_ids && !s->retired) {
        abmx_internal::set_error("recycle_ids needs a retired-id stack of capacity entries");
        return ABMX_E_SCHEMA;
    }
    if (s->n_state < 0 || s->n_extra < 0 || (s->n_state && !s->state) || (s->n_extra && !s->extra)) {
        abmx_internal::set_error("bad column list");
        return ABMX_E_SCHEMA;
    }
    for (int c = 0; c < s->n_state; ++c)
        if (!elem_ok(s->state[c].elem_size) || (s->capacity && !s->state[c].data)) {
            abmx_internal::set_error("state columns need 1, 4 or 8 byte elements");
            return ABMX_E_SCHEMA;
        }
    for (int c = 0; c < s->n_extra; ++c)
        if (!elem_ok(s->extra[c].elem_size) || (s->capacity && !s->extra[c].data)) {
            abmx_internal::set_error("extra columns need 1, 4 or 8 byte elements");
            return ABMX_E_SCHEMA;
        }
    return ABMX_OK;
}

Life life_of(const abmx_agent_set* s) {
    return Life{s->active, reinterpret_cast<long long*>(s->ids), reinterpret_cast<long long*>(s->ages),
                reinterpret_cast<long long*>(s->types), reinterpret_cast<long long*>(s->counters),
                reinterpret_cast<long long*>(s->retired), s->recycle_ids ? 1 : 0};
}

// Scratch for one call, stream-ordered (freed with cudaFreeAsync after the last use).
struct Scratch {
    cudaStream_t st;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : st(s) {}
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, st);
    }
    cudaError_t get(void** p, size_t bytes) {
        cudaError_t e = abmx_internal::malloc_async(p, bytes ? bytes : 16, st);
        if (e == cudaSuccess) ptrs.push_back(*p);
        return e;
    }
};

// slot-ordered selection list + device count
template <int kMode>
int select_list(const uint8_t* mask, const uint8_t* active, size_t n, int32_t* list, long long* count,
                Scratch& sc, unsigned** done = nullptr) {
    cudaStream_t st = sc.st;
    if (done) *done = nullptr;
    if (n == 0) {
        CKA(cudaMemsetAsync(count, 0, sizeof(long long), st));
        return ABMX_OK;
    }
    const size_t tiles = (n + kTile - 1) / kTile;
    void* ws = nullptr;
    const size_t wsb = sizeof(ScanWs) + tiles * sizeof(unsigned long long);
    CKA(sc.get(&ws, wsb));
    CKA(cudaMemsetAsync(ws, 0, wsb, st));
    k_select<kMode><<<static_cast<unsigned>(tiles), kT, 0, st>>>(mask, active, n, list, count,
                                                                 static_cast<ScanWs*>(ws));
    if (done) *done = &static_cast<ScanWs*>(ws)->pad;  // zeroed and unused by k_select
    abmx_internal::count_launch();
    CKA(cudaGetLastError());
    return ABMX_OK;
}

// launch `fn(Cols)` over column chunks of at most kMaxCols
template <class F>
int for_col_chunks(int ncols, F&& fn) {
    for (int c0 = 0; c0 < ncols || (ncols == 0 && c0 == 0); c0 += kMaxCols) {
        const int cn = ncols - c0 < kMaxCols ? ncols - c0 : kMaxCols;
        int rc = fn(c0, cn > 0 ? cn : 0);
        if (rc) return rc;
        if (ncols == 0) break;
    }
    return ABMX_OK;
}

constexpr int kNoCoop = -1000;  // life_coop: the cooperative kernel does not apply

// One cooperative k_life_coop launch for remove (m == 0), spawn (d_kill == nullptr) or both, when
// the set has at most kMaxCols state columns and its ta + tb tiles are co-resident; kNoCoop
// otherwise (the caller takes its multi-kernel path). Arguments are checked by the caller.
static int life_coop(const abmx_agent_set* s, const uint8_t* d_kill, int32_t m, const uint8_t* d_valid,
                     const abmx_column* rows, int32_t set_type, int64_t agent_type, int64_t* d_killed,
                     int64_t* d_result, int32_t* d_slots, int32_t* d_rows, cudaStream_t st, int rm = 0) {
    if (s->capacity == 0 || s->n_state > kMaxCols || (m == 0 && (rm || !d_kill))) return kNoCoop;
    const size_t n = static_cast<size_t>(s->capacity);
    const size_t ta = (n + kTile - 1) / kTile, tb = (static_cast<size_t>(m) + kTile - 1) / kTile;
    Cols Z{};  // removal: zero every state column
    Z.n = s->n_state;
    for (int c = 0; c < s->n_state; ++c) {
        Z.dst[c] = s->state[c].data;
        Z.src[c] = nullptr;
        Z.sz[c] = s->state[c].elem_size;
    }
    Cols A{};  // spawn: copy the row columns given
    A.n = 0;
    for (int c = 0; c < s->n_state; ++c) {
        if (!rows || !rows[c].data) continue;
        A.dst[A.n] = s->state[c].data;
        A.src[A.n] = rows[c].data;
        A.sz[A.n] = s->state[c].elem_size;
        ++A.n;
    }
    const Life L = life_of(s);
    // co-resident k_life_coop CTAs per SM, per device (computed once; racing writers store the
    // same value)
    static std::atomic<int> coop_per_sm[abmx_internal::kMaxDevices] = {};
    int dev = 0;
    CKA(cudaGetDevice(&dev));
    int per_sm = 0;
    if (dev >= 0 && dev < abmx_internal::kMaxDevices) {
        per_sm = coop_per_sm[dev].load(std::memory_order_relaxed);
        if (per_sm == 0) {
            int per = 0;
            CKA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_life_coop, kT, 0));
            per_sm = per > 0 ? per : -1;
            coop_per_sm[dev].store(per_sm, std::memory_order_relaxed);
        }
    }
    const long long coop_cap = per_sm > 0 ? static_cast<long long>(per_sm) * abmx_internal::num_sms() : 0;
    if (static_cast<long long>(ta + tb) > coop_cap || ta + tb > static_cast<size_t>(kCoopMaxTiles)) return kNoCoop;
    {  // one cooperative kernel; scratch: [workspace | free slots per slot tile | killed ids]
        Scratch sc(st);
        const size_t ws_b = (sizeof(LifeWs) + (ta + tb) * sizeof(unsigned long long) + 15) / 16 * 16;
        const size_t lists = ta * kTile;
        void* ws = nullptr;
        CKA(sc.get(&ws, ws_b + lists * 4 + (s->recycle_ids ? lists * 8 : 0)));
        int32_t* free_list = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + ws_b);
        long long* kill_ids = s->recycle_ids ? reinterpret_cast<long long*>(free_list + lists) : nullptr;
        unsigned z_refill = 0;  // state columns a refilled killed slot still zeroes: those without a row column
        for (int c = 0; c < Z.n; ++c) {
            bool written = false;
            for (int e = 0; e < A.n; ++e) written = written || A.dst[e] == Z.dst[c];
            if (!written) z_refill |= 1u << c;
        }
        CKA(cudaMemsetAsync(ws, 0, sizeof(unsigned), st));
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(ta + tb));
        cfg.blockDim = dim3(kT);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        CKA(cudaLaunchKernelEx(&cfg, k_life_coop, d_kill, n, static_cast<unsigned>(ta), d_valid, static_cast<size_t>(m),
                               free_list, kill_ids, static_cast<LifeWs*>(ws), Z, z_refill, A, L, static_cast<int>(set_type),
                               static_cast<long long>(agent_type), reinterpret_cast<long long*>(d_killed),
                               reinterpret_cast<long long*>(d_result), d_slots, d_rows, rm));
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
        return ABMX_OK;
    }
}

// shared pairing core of spawn / set_rm / set_sci
int pair_rows(const abmx_agent_set* s, const uint8_t* d_target, bool spawn, int32_t m, const uint8_t* d_valid,
              const abmx_column* rows, int set_type, int64_t agent_type, int32_t* d_slots, int32_t* d_rows,
              int64_t* d_out, void* stream) {
    int rc = check_set(s);
    if (rc) return rc;
    if (m < 0 || (m > 0 && !d_valid)) {
        abmx_internal::set_error("bad update batch");
        return ABMX_E_ARG;
    }
    if (!spawn && s->capacity > 0 && !d_target) {
        abmx_internal::set_error("null target mask");
        return ABMX_E_ARG;
    }
    for (int c = 0; c < s->n_state; ++c)
        if (rows && rows[c].data && rows[c].elem_size != s->state[c].elem_size) {
            abmx_internal::set_error("row column element size differs from its state column");
            return ABMX_E_SCHEMA;
        }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();
    {  // one cooperative kernel when the tiles fit (pairs k < r listed)
        rc = spawn ? life_coop(s, nullptr, m, d_valid, rows, set_type, agent_type, nullptr, d_out, d_slots, d_rows, st)
                   : life_coop(s, d_target, m, d_valid, rows, 0, 0, nullptr, d_out, d_slots, d_rows, st, 1);
        if (rc != kNoCoop) return rc;
    }
    Scratch sc(st);
    const size_t n = static_cast<size_t>(s->capacity);
    int32_t* slots = d_slots;
    int32_t* rws = d_rows;
    long long* cnt = nullptr;  // [2]: p, q
    CKA(sc.get(reinterpret_cast<void**>(&cnt), 2 * sizeof(long long)));
    if (!slots) CKA(sc.get(reinterpret_cast<void**>(&slots), n * 4));
    if (!rws) CKA(sc.get(reinterpret_cast<void**>(&rws), static_cast<size_t>(m) * 4));
    unsigned* done = nullptr;  // the pad word of the (second) scan's workspace: a zeroed counter
    if (spawn && n > 0 && m > 0) {  // both selections in one launch, one workspace memset
        const size_t ta = (n + kTile - 1) / kTile, tb = (static_cast<size_t>(m) + kTile - 1) / kTile;
        const size_t wa_b = (sizeof(ScanWs) + ta * sizeof(unsigned long long) + 15) / 16 * 16;
        const size_t wb_b = sizeof(ScanWs) + tb * sizeof(unsigned long long);
        void* ws = nullptr;
        CKA(sc.get(&ws, wa_b + wb_b));
        CKA(cudaMemsetAsync(ws, 0, wa_b + wb_b, st));
        ScanWs* wa = static_cast<ScanWs*>(ws);
        ScanWs* wb = reinterpret_cast<ScanWs*>(static_cast<char*>(ws) + wa_b);
        k_select_spawn<<<static_cast<unsigned>(ta + tb), kT, 0, st>>>(s->active, n, slots, cnt, wa,
                                                                       static_cast<unsigned>(ta), d_valid,
                                                                       static_cast<size_t>(m), rws, cnt + 1, wb);
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
        done = &wb->pad;
    } else {
        if (spawn)
            rc = select_list<kSelFree>(nullptr, s->active, n, slots, cnt, sc);
        else
            rc = select_list<kSelMask>(d_target, nullptr, n, slots, cnt, sc);
        if (rc) return rc;
        rc = select_list<kSelMask>(d_valid, nullptr, static_cast<size_t>(m), rws, cnt + 1, sc, &done);
        if (rc) return rc;
    }
    bool committed = false;
    const Life L = life_of(s);
    const size_t pairs_max = n < static_cast<size_t>(m) ? n : static_cast<size_t>(m);
    rc = for_col_chunks(s->n_state, [&](int c0, int cn) {
        Cols C{};
        C.n = 0;
        for (int c = 0; c < cn; ++c) {
            if (!rows || !rows[c0 + c].data) continue;  // the apply leaves this column alone
            C.dst[C.n] = s->state[c0 + c].data;
            C.src[C.n] = rows[c0 + c].data;
            C.sz[C.n] = s->state[c0 + c].elem_size;
            ++C.n;
        }
        const int sp = spawn && c0 == 0;  // lifecycle fields once
        if (C.n == 0 && !sp) return static_cast<int>(ABMX_OK);
        const bool last = c0 + kMaxCols >= s->n_state && done;  // fold the commit into it
        k_pair_apply<<<grid_for(pairs_max), kT, 0, st>>>(slots, rws, cnt, cnt + 1, C, sp, L, set_type, agent_type,
                                                          last ? done : nullptr,
                                                          last ? reinterpret_cast<long long*>(d_out) : nullptr);
        committed = committed || last;
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
        return static_cast<int>(ABMX_OK);
    });
    if (rc) return rc;
    if (committed) return ABMX_OK;
    if (spawn) {
        k_spawn_commit<<<1, 1, 0, st>>>(cnt, cnt + 1, L, reinterpret_cast<long long*>(d_out));
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
    } else if (d_out) {
        // {pairs, valid rows}
        k_pair_result<<<1, 1, 0, st>>>(cnt, cnt + 1, reinterpret_cast<long long*>(d_out));
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
    }
    return ABMX_OK;
}

}  // namespace

extern "C" {

int abmx_agents_remove(const abmx_agent_set* s, const uint8_t* d_kill, int64_t* d_killed, void* stream) {
    int rc = check_set(s);
    if (rc) return rc;
    if (s->capacity > 0 && !d_kill) {
        abmx_internal::set_error("null kill mask");
        return ABMX_E_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();
    rc = life_coop(s, d_kill, 0, nullptr, nullptr, 0, 0, d_killed, nullptr, nullptr, nullptr, st);
    if (rc != kNoCoop) return rc;
    Scratch sc(st);
    const size_t n = static_cast<size_t>(s->capacity);
    int32_t* list = nullptr;
    long long* cnt = nullptr;
    CKA(sc.get(reinterpret_cast<void**>(&list), n * 4));
    CKA(sc.get(reinterpret_cast<void**>(&cnt), sizeof(long long)));
    unsigned* done = nullptr;
    rc = select_list<kSelKill>(d_kill, s->active, n, list, cnt, sc, &done);
    if (rc) return rc;
    const Life L = life_of(s);
    bool committed = false;
    // lifecycle fields with the first chunk; the retired push reads ids before they are zeroed
    rc = for_col_chunks(s->n_state, [&](int c0, int cn) {
        Cols C{};
        C.n = cn;
        for (int c = 0; c < cn; ++c) {
            C.dst[c] = s->state[c0 + c].data;
            C.src[c] = nullptr;
            C.sz[c] = s->state[c0 + c].elem_size;
        }
        const bool last = (c0 + kMaxCols >= s->n_state) && done;  // fold the commit into it
        unsigned* dn = last ? done : nullptr;
        long long* out = last ? reinterpret_cast<long long*>(d_killed) : nullptr;
        if (c0 == 0) {
            k_remove_apply<<<grid_for(n), kT, 0, st>>>(list, cnt, C, L, dn, L, out);
        } else {  // further chunks: state columns only (lifecycle fields already reset)
            Life none = L;
            none.recycle = 0;
            // the lifecycle writes are idempotent, but active was already cleared: reuse the list
            k_remove_apply<<<grid_for(n), kT, 0, st>>>(list, cnt, C, none, dn, L, out);
        }
        committed = committed || last;
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
        return static_cast<int>(ABMX_OK);
    });
    if (rc) return rc;
    if (committed) return ABMX_OK;
    k_remove_commit<<<1, 1, 0, st>>>(cnt, L, reinterpret_cast<long long*>(d_killed));
    abmx_internal::count_launch();
    CKA(cudaGetLastError());
    return ABMX_OK;
}

#ifdef ABMX_LIFE_TRACE
extern "C" int abmx_life_trace(unsigned long long* out, int ctas) {
    return cudaMemcpyFromSymbol(out, abmx_agents::g_life_trace, sizeof(unsigned long long) * 8 * ctas) == cudaSuccess ? 0 : -1;
}
#endif

int abmx_agents_lifecycle(const abmx_agent_set* s, const uint8_t* d_kill, int32_t m, const uint8_t* d_valid,
                          const abmx_column* rows, int32_t set_type, int64_t agent_type, int64_t* d_killed,
                          int64_t* d_result, void* stream) {
    int rc = check_set(s);
    if (rc) return rc;
    if ((s->capacity > 0 && !d_kill) || m < 0 || (m > 0 && !d_valid)) {
        abmx_internal::set_error("bad lifecycle arguments");
        return ABMX_E_ARG;
    }
    for (int c = 0; c < s->n_state; ++c)
        if (rows && rows[c].data && rows[c].elem_size != s->state[c].elem_size) {
            abmx_internal::set_error("row column element size differs from its state column");
            return ABMX_E_SCHEMA;
        }
    if (s->capacity == 0 || m == 0 || s->n_state > kMaxCols) {  // the general two-call path
        rc = abmx_agents_remove(s, d_kill, d_killed, stream);
        if (rc) return rc;
        return abmx_agents_spawn(s, m, d_valid, rows, set_type, agent_type, nullptr, nullptr, d_result, stream);
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();
    rc = life_coop(s, d_kill, m, d_valid, rows, set_type, agent_type, d_killed, d_result, nullptr, nullptr, st);
    if (rc != kNoCoop) return rc;
    Scratch sc(st);
    const size_t n = static_cast<size_t>(s->capacity);
    const size_t ta = (n + kTile - 1) / kTile, tb = (static_cast<size_t>(m) + kTile - 1) / kTile;
    Cols Z{};  // removal: zero every state column
    Z.n = s->n_state;
    for (int c = 0; c < s->n_state; ++c) {
        Z.dst[c] = s->state[c].data;
        Z.src[c] = nullptr;
        Z.sz[c] = s->state[c].elem_size;
    }
    Cols A{};  // spawn: copy the row columns given
    A.n = 0;
    for (int c = 0; c < s->n_state; ++c) {
        if (!rows || !rows[c].data) continue;
        A.dst[A.n] = s->state[c].data;
        A.src[A.n] = rows[c].data;
        A.sz[A.n] = s->state[c].elem_size;
        ++A.n;
    }
    const Life L = life_of(s);
    const size_t wa_b = (sizeof(ScanWs) + ta * sizeof(unsigned long long) + 15) / 16 * 16;
    const size_t wb_b = (sizeof(ScanWs) + tb * sizeof(unsigned long long) + 15) / 16 * 16;
    const size_t ws_b = (wa_b + wb_b + sizeof(LifeCounts) + 15) / 16 * 16;
    // one scratch block (host submission is a large part of a cycle): [workspace | slots | rows]
    void* ws = nullptr;
    CKA(sc.get(&ws, ws_b + n * 4 + static_cast<size_t>(m) * 4));
    int32_t* slots = reinterpret_cast<int32_t*>(static_cast<char*>(ws) + ws_b);
    int32_t* rws = slots + n;
    CKA(cudaMemsetAsync(ws, 0, ws_b, st));
    ScanWs* wa = static_cast<ScanWs*>(ws);
    ScanWs* wb = reinterpret_cast<ScanWs*>(static_cast<char*>(ws) + wa_b);
    LifeCounts* cnt = reinterpret_cast<LifeCounts*>(static_cast<char*>(ws) + wa_b + wb_b);
    k_life_select<<<static_cast<unsigned>(ta + tb), kT, 0, st>>>(d_kill, n, slots, wa, static_cast<unsigned>(ta), d_valid,
                                                                 static_cast<size_t>(m), rws, wb, Z, L, cnt);
    abmx_internal::count_launch();
    CKA(cudaGetLastError());
    // the pair count is known only on the device: a grid-stride apply over at most 2 CTAs per SM
    // (a grid sized for min(n, m) pairs launched ~1200 CTAs for C2's ~14k births)
    const size_t pairs_max = n < static_cast<size_t>(m) ? n : static_cast<size_t>(m);
    const int g_apply = grid_for(pairs_max) < abmx_internal::num_sms() * 2 ? grid_for(pairs_max)
                                                                          : abmx_internal::num_sms() * 2;
    k_life_apply<<<g_apply, kT, 0, st>>>(slots, rws, cnt, A, L, set_type, agent_type, &wa->pad,
                                                     reinterpret_cast<long long*>(d_killed),
                                                     reinterpret_cast<long long*>(d_result));
    abmx_internal::count_launch();
    CKA(cudaGetLastError());
    return ABMX_OK;
}

int abmx_agents_spawn(const abmx_agent_set* s, int32_t m, const uint8_t* d_valid, const abmx_column* rows,
                      int32_t set_type, int64_t agent_type, int32_t* d_slots, int32_t* d_rows, int64_t* d_result,
                      void* stream) {
    return pair_rows(s, nullptr, true, m, d_valid, rows, set_type, agent_type, d_slots, d_rows, d_result, stream);
}

int abmx_agents_set_rm(const abmx_agent_set* s, const uint8_t* d_target, int32_t m, const uint8_t* d_valid,
                       const abmx_column* rows, int32_t* d_slots, int32_t* d_rows, int64_t* d_result,
                       void* stream) {
    return pair_rows(s, d_target, false, m, d_valid, rows, 0, 0, d_slots, d_rows, d_result, stream);
}

int abmx_agents_set_sci(const abmx_agent_set* s, const uint8_t* d_target, int32_t m, const uint8_t* d_valid,
                        const abmx_column* rows, int32_t* d_slots, int32_t* d_rows, int64_t* d_result,
                        void* stream) {
    // the column-copy apply reads only its own slot and row: SCI == RM (kernels.hpp:96-99)
    return pair_rows(s, d_target, false, m, d_valid, rows, 0, 0, d_slots, d_rows, d_result, stream);
}

int abmx_agents_set_mask(const abmx_agent_set* s, const uint8_t* d_mask, const abmx_column* values,
                         void* stream) {
    int rc = check_set(s);
    if (rc) return rc;
    if (s->capacity == 0) return ABMX_OK;
    if (!d_mask || !values) {
        abmx_internal::set_error("null mask or values");
        return ABMX_E_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();
    const size_t n = static_cast<size_t>(s->capacity);
    return for_col_chunks(s->n_state, [&](int c0, int cn) {
        Cols C{};
        C.n = 0;
        for (int c = 0; c < cn; ++c) {
            if (!values[c0 + c].data) continue;
            if (values[c0 + c].elem_size != s->state[c0 + c].elem_size) {
                abmx_internal::set_error("value column element size differs from its state column");
                return static_cast<int>(ABMX_E_SCHEMA);
            }
            C.dst[C.n] = s->state[c0 + c].data;
            C.src[C.n] = values[c0 + c].data;
            C.sz[C.n] = s->state[c0 + c].elem_size;
            ++C.n;
        }
        if (C.n == 0) return static_cast<int>(ABMX_OK);
        k_mask_apply<<<grid_for(n), kT, 0, st>>>(d_mask, n, C);
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
        return static_cast<int>(ABMX_OK);
    });
}

int abmx_agents_select(const uint8_t* d_mask, int32_t n, int32_t* d_indices, int64_t* d_count, void* stream) {
    if (n < 0 || (n > 0 && (!d_mask || !d_indices)) || !d_count) {
        abmx_internal::set_error("bad select arguments");
        return ABMX_E_ARG;
    }
    (void)cudaGetLastError();
    cudaError_t e = abmx_internal::launch_compact_indices(d_mask, d_indices, static_cast<size_t>(n),
                                                          reinterpret_cast<unsigned long long*>(d_count),
                                                          static_cast<cudaStream_t>(stream));
    if (e != cudaSuccess) {
        abmx_internal::set_error(std::string("select: ") + cudaGetErrorString(e));
        return ABMX_E_CUDA;
    }
    return ABMX_OK;
}

// pinned_keys (kernels.cpp:37-50): the keys of active slots, +inf (ascending) / -inf (descending)
// on placeholder slots so they sort to the tail
static __global__ void k_pinned_keys(const double* __restrict__ keys, const uint8_t* __restrict__ active, size_t n,
                              double pin, double* __restrict__ out) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        out[i] = active[i] ? keys[i] : pin;
}

int abmx_agents_pinned_keys(const double* d_keys, const uint8_t* d_active, int32_t n, int32_t descending,
                            double* d_out, void* stream) {
    if (n < 0 || (n > 0 && (!d_keys || !d_active || !d_out))) {
        abmx_internal::set_error("bad pinned_keys arguments");
        return ABMX_E_ARG;
    }
    if (n == 0) return ABMX_OK;
    (void)cudaGetLastError();
    const double pin = descending ? -HUGE_VAL : HUGE_VAL;
    k_pinned_keys<<<grid_for(static_cast<size_t>(n)), kT, 0, static_cast<cudaStream_t>(stream)>>>(
        d_keys, d_active, static_cast<size_t>(n), pin, d_out);
    abmx_internal::count_launch();
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        abmx_internal::set_error(std::string("pinned_keys: ") + cudaGetErrorString(e));
        return ABMX_E_CUDA;
    }
    return ABMX_OK;
}

int abmx_agents_sort_perm(const double* d_key, const uint8_t* d_active, int32_t n, int32_t descending,
                          int32_t* d_perm, void* stream) {
    if (n < 0 || (n > 0 && (!d_key || !d_active || !d_perm))) {
        abmx_internal::set_error("bad sort arguments");
        return ABMX_E_ARG;
    }
    if (n == 0) return ABMX_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();
    Scratch sc(st);
    const size_t N = static_cast<size_t>(n);
    const int tiles = static_cast<int>((N + kTile - 1) / kTile);
    unsigned long long *k0, *k1;
    int32_t* v1;
    unsigned *hist, *dtot, *bad;
    CKA(sc.get(reinterpret_cast<void**>(&k0), N * 8));
    CKA(sc.get(reinterpret_cast<void**>(&k1), N * 8));
    CKA(sc.get(reinterpret_cast<void**>(&v1), N * 4));
    CKA(sc.get(reinterpret_cast<void**>(&hist), static_cast<size_t>(tiles) * 256 * 4));
    CKA(sc.get(reinterpret_cast<void**>(&dtot), 256 * 4 + 16));
    bad = dtot + 256;
    CKA(cudaMemsetAsync(bad, 0, 4, st));
    k_sort_keys<<<grid_for(N), kT, 0, st>>>(d_key, d_active, N, descending ? 1 : 0, k0, d_perm, bad);
    abmx_internal::count_launch();
    CKA(cudaGetLastError());
    unsigned h_bad = 0;
    CKA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, st));
    CKA(cudaStreamSynchronize(st));
    if (h_bad) {
        abmx_internal::set_error("non-finite sort key on an active slot");  // kernels.cpp:57-60
        return ABMX_E_DOMAIN;
    }
    // 8 passes of 8 bits; after an even number of passes the result is back in (k0, d_perm)
    unsigned long long* kin = k0;
    unsigned long long* kout = k1;
    int32_t* vin = d_perm;
    int32_t* vout = v1;
    for (int shift = 0; shift < 64; shift += 8) {
        k_hist<<<tiles, kT, 0, st>>>(kin, N, shift, hist, tiles);
        k_digit_scan<<<256, kT, 0, st>>>(hist, tiles, dtot);
        k_scatter<<<tiles, kT, 0, st>>>(kin, vin, kout, vout, N, shift, hist, dtot, tiles);
        abmx_internal::count_launch(3);
        CKA(cudaGetLastError());
        unsigned long long* tk = kin;
        kin = kout;
        kout = tk;
        int32_t* tv = vin;
        vin = vout;
        vout = tv;
    }
    return ABMX_OK;
}

int abmx_agents_permute(const abmx_agent_set* s, const int32_t* d_perm, void* stream) {
    int rc = check_set(s);
    if (rc) return rc;
    const size_t n = static_cast<size_t>(s->capacity);
    if (n == 0) return ABMX_OK;
    if (!d_perm) {
        abmx_internal::set_error("null permutation");
        return ABMX_E_ARG;
    }
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    (void)cudaGetLastError();
    Scratch sc(st);
    unsigned* bad = nullptr;
    CKA(sc.get(reinterpret_cast<void**>(&bad), 4));
    CKA(cudaMemsetAsync(bad, 0, 4, st));
    k_check_perm<<<grid_for(n), kT, 0, st>>>(d_perm, n, bad);
    abmx_internal::count_launch();
    unsigned h_bad = 0;
    CKA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, st));
    CKA(cudaStreamSynchronize(st));
    if (h_bad) {
        abmx_internal::set_error("permutation index outside [0, capacity)");
        return ABMX_E_DOMAIN;
    }
    // every column: gather into scratch, copy back (out-of-place gather, in-place result)
    std::vector<abmx_column> cols;
    cols.push_back({s->active, 1, 0});
    cols.push_back({s->ids, 8, 0});
    cols.push_back({s->types, 8, 0});
    cols.push_back({s->ages, 8, 0});
    for (int c = 0; c < s->n_state; ++c) cols.push_back(s->state[c]);
    for (int c = 0; c < s->n_extra; ++c) cols.push_back(s->extra[c]);
    std::vector<void*> tmp(cols.size());
    for (size_t c = 0; c < cols.size(); ++c) CKA(sc.get(&tmp[c], n * static_cast<size_t>(cols[c].elem_size)));
    rc = for_col_chunks(static_cast<int>(cols.size()), [&](int c0, int cn) {
        Cols C{};
        C.n = cn;
        for (int c = 0; c < cn; ++c) {
            C.dst[c] = tmp[c0 + c];
            C.src[c] = cols[c0 + c].data;
            C.sz[c] = cols[c0 + c].elem_size;
        }
        k_gather<<<grid_for(n), kT, 0, st>>>(d_perm, n, C);
        abmx_internal::count_launch();
        CKA(cudaGetLastError());
        return static_cast<int>(ABMX_OK);
    });
    if (rc) return rc;
    for (size_t c = 0; c < cols.size(); ++c)
        CKA(cudaMemcpyAsync(cols[c].data, tmp[c], n * static_cast<size_t>(cols[c].elem_size),
                            cudaMemcpyDeviceToDevice, st));
    return ABMX_OK;
}

int abmx_agents_sort(const abmx_agent_set* s, const double* d_key, int32_t descending, int32_t* d_perm,
                     void* stream) {
    int rc = check_set(s);
    if (rc) return rc;
    const size_t n = static_cast<size_t>(s->capacity);
    if (n == 0) return ABMX_OK;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Scratch sc(st);
    int32_t* perm = d_perm;
    if (!perm) CKA(sc.get(reinterpret_cast<void**>(&perm), n * 4));
    rc = abmx_agents_sort_perm(d_key, s->active, s->capacity, descending, perm, stream);
    if (rc) return rc;
    return abmx_agents_permute(s, perm, stream);
}

}  // extern "C"
