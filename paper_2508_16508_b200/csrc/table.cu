// table.cu — sm_100a implementations of the reference KernelTable entries
// (include/abmx/simd/kernels.hpp:15-43; scalar semantics src/simd/kernels_scalar.cpp:7-54).
//
// All entries are HBM-streaming integer/bitwise kernels:
//   rank_scan        persistent count-then-scan over per-CTA chunks, TMA-pipelined (below)
//   count_true       grid-stride SWAR popcount reduction
//   compact_indices  the same kernel: count, chunk gather (gives the true total), two-run scatter
//   match_first_equal  O(n+m) first-match table (dense when rb's range is small,
//                    open-addressing hash otherwise; atomicMin keeps FIRST-match semantics)
//   blend_{i64,f64,u8}  predicated select, out may alias a or b (lifecycle.cpp:105-111)
#include <climits>
#include <cstdint>

#include "abmx_device.cuh"
#include "abmx_internal.h"

using namespace abmx_dev;

namespace abmx_table {

constexpr int kThreads = 256;
constexpr int kCountItems = 64;

// nonzero bytes of a word (SWAR): fold each byte's bits onto its bit 0, then popcount
__device__ __forceinline__ unsigned nz_bytes(uint32_t w) {
    uint32_t x = w | (w >> 4);
    x |= x >> 2;
    x |= x >> 1;
    return static_cast<unsigned>(__popc(x & 0x01010101u));
}

// number of nonzero bytes (64 per thread per iteration: four 16-byte loads in flight)
__global__ void __launch_bounds__(kThreads) count_true_kernel(const uint8_t* __restrict__ mask,
                                                              size_t n,
                                                              unsigned long long* __restrict__ out) {
    const bool vec = (reinterpret_cast<uintptr_t>(mask) & 15) == 0;
    unsigned long long c = 0;
    for (size_t base = (static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x) * kCountItems; base < n;
         base += static_cast<size_t>(gridDim.x) * kThreads * kCountItems) {
        unsigned part = 0;
        if (vec && base + kCountItems <= n) {
            uint4 v[kCountItems / 16];
#pragma unroll
            for (int q = 0; q < kCountItems / 16; ++q) v[q] = *reinterpret_cast<const uint4*>(mask + base + 16 * q);
#pragma unroll
            for (int q = 0; q < kCountItems / 16; ++q)
                part += nz_bytes(v[q].x) + nz_bytes(v[q].y) + nz_bytes(v[q].z) + nz_bytes(v[q].w);
        } else {
            for (size_t i = base; i < base + kCountItems && i < n; ++i) part += mask[i] != 0;
        }
        c += part;
    }
    c = warp_sum(c);
    __shared__ unsigned long long s[kThreads / 32];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x < 32) {
        unsigned long long v = threadIdx.x < kThreads / 32 ? s[threadIdx.x] : 0ULL;
        v = warp_sum(v);
        // launched with programmatic serialization after the zeroing of *out: wait for it only here
        asm volatile("griddepcontrol.wait;" ::: "memory");
        if (threadIdx.x == 0 && v) atomicAdd(out, v);
    }
}

// zero n words (a kernel, not a memset node, so that the next kernel can launch programmatically)
__global__ void zero_words_kernel(unsigned long long* p, size_t n) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = 0ULL;
}

// ---------------------------------------------------------------- persistent pipelined scan
// rank_scan and compact_indices at HBM speed. A persistent, co-resident grid (cooperative
// launch, 2 CTAs per SM) gives each CTA one contiguous chunk of kPTile-byte mask tiles, and each
// CTA streams its chunk twice:
//   pass 1  counts the chunk's nonzero bytes and publishes the chunk total;
//   gather  every CTA reads all chunk totals (all published at about the same time, one round
//           trip): its exclusive chunk prefix and, for compact_indices, the true total T;
//   pass 2  re-reads the chunk and writes ranks (rank_scan) or the stable partition
//           (compact_indices) with a running in-chunk prefix. No tile waits on another tile.
// A per-tile decoupled lookback was measured first (profiles/r02_table.md): with every CTA's
// tiles in flight at once, the lookbacks ran the CTAs in lock-step (6 us per tile), 3x slower
// than this extra 1-byte-per-element read. compact_indices needs no separate count kernel.
// Tiles arrive through a kPIn-stage shared-memory ring filled by 1-D bulk copies (TMA,
// cp.async.bulk -> UBLKCP), so HBM reads run ahead of the scan and the stores. A warp owns
// 1024 consecutive elements as 8 rows of 32 words; a row is scanned with three ballots of the
// per-word nonzero-byte counts (0..4). rank_scan stages its ranks in shared memory and writes
// each tile with one bulk copy (double-buffered); compact_indices partitions the tile in shared
// memory and writes its two runs with coalesced stores. Partial or unaligned tiles take the
// same path with plain loads / stores.
#ifndef ABMX_SCAN_THREADS
#define ABMX_SCAN_THREADS 256
#endif
constexpr int kPT = ABMX_SCAN_THREADS;  // threads per CTA (a warp scans 1024 elements per tile)
constexpr int kPTile = kPT * 32;        // mask bytes (elements) per tile
constexpr int kPMinB = kPT >= 512 ? 1 : 2;  // CTAs per SM (rank_scan: 104 KB of ring + output stages each)
#ifndef ABMX_COMPACT_CTAS
#define ABMX_COMPACT_CTAS 3
#endif
constexpr int kCMinB = kPT >= 512 ? 1 : ABMX_COMPACT_CTAS;  // compact_indices: 72 KB each
#ifndef ABMX_SCAN_STAGES
#define ABMX_SCAN_STAGES 5
#endif
constexpr int kPIn = ABMX_SCAN_STAGES;  // input stages
constexpr int kPOut = 2;       // rank_scan output stages

// Pass 1 only counts, so the output stages also serve as input slots: the ring is kP1 slots deep
// there (rank_scan 13, compact_indices 9) and kPIn in pass 2.
constexpr int kP1Max = 16;

struct PipeShared {
    unsigned long long bar[kP1Max];
    unsigned wtot[kPT / 32];
    unsigned wt1[2][kPT / 32];          // pass 1: warp counts of the last two tiles
    unsigned long long red[kPT / 32 + 2][2];
    unsigned long long total, base, T;
    unsigned long long jb[kPIn];        // pass 2: base of the tile queued in each slot
    int jt[kPIn];                       // ... and the tile (-1: none left)
};

template <bool kCompact>
__host__ __device__ constexpr int pipe_smem() {
    return kPIn * kPTile + (kCompact ? kPTile + 16 : kPOut * kPTile) * static_cast<int>(sizeof(int32_t));
}

#ifdef ABMX_SCAN_TRACE  // per-CTA %globaltimer stamps: start, pass 1 done, gather done, end
__device__ unsigned long long g_scan_trace[2048][4];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define SCAN_STAMP(k) \
    if (tid == 0) g_scan_trace[b][k] = gtime()
#else
#define SCAN_STAMP(k)
#endif

#ifndef ABMX_SCAN_BAR_NS
#define ABMX_SCAN_BAR_NS 0
#endif

// Workspace of one call (zeroed: the chunk totals and the three counters; the per-tile arrays
// are fully written before they are read).
struct ScanWs {
    unsigned published;    // chunks whose pass-1 total is out
    unsigned next_tile;    // pass 2: the next unclaimed tile
};

template <bool kCompact>
__global__ void __launch_bounds__(kPT, kCompact ? kCMinB : kPMinB) scan_pipe_kernel(const uint8_t* __restrict__ mask, int32_t* __restrict__ out,
                                                          size_t n, int tiles, unsigned long long* __restrict__ chunk_tot,
                                                          unsigned long long* __restrict__ true_out) {
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ PipeShared S;
    uint8_t* in = dsm;
    int32_t* ob = reinterpret_cast<int32_t*>(dsm + kPIn * kPTile);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    const int c0 = static_cast<int>(static_cast<long long>(tiles) * b / G);
    const int m = static_cast<int>(static_cast<long long>(tiles) * (b + 1) / G) - c0;  // >= 1 (grid <= tiles)
    ScanWs* ws = reinterpret_cast<ScanWs*>(chunk_tot + G);
    unsigned long long* tile_base = reinterpret_cast<unsigned long long*>(ws + 1);  // [tiles] kFlagAgg | base (zeroed)
    unsigned* tile_cnt = reinterpret_cast<unsigned*>(tile_base + tiles);             // [tiles]
    const bool in_vec = (reinterpret_cast<uintptr_t>(mask) & 15) == 0;
    const bool out_vec = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    auto is_bulk = [&](int t) { return in_vec && static_cast<size_t>(t + 1) * kPTile <= n; };
    // The mask is read twice: pass 1 keeps it in L2 (evict_last; 2^26 bytes fit), pass 2 reads it
    // for the last time and the outputs stream past it (evict_first).
    const unsigned long long keep = l2_evict_last(), stream = l2_evict_first();
    constexpr int kP1 = pipe_smem<kCompact>() / kPTile;
    static_assert(kP1 <= kP1Max && kP1 >= kPIn, "pass-1 ring");
    auto load = [&](int t, int s, unsigned long long policy) {  // one thread: tile t into ring slot s
        ABMX_ASSERT(t >= 0 && t < tiles && s >= 0 && s < kP1);
        if (is_bulk(t)) {
            mbar_expect_tx(&S.bar[s], kPTile);
            bulk_g2s_hint(in + s * kPTile, mask + static_cast<size_t>(t) * kPTile, kPTile, &S.bar[s], policy);
        }
    };
    // Pass 2: thread 0 claims the next tile of the whole mask (every CTA draws from one counter,
    // so the CTAs that stream faster take more tiles) and queues it with its base in a ring slot.
    // The claims are pipelined in thread 0's registers: the atomic of a claim is issued two
    // refills before its slot is filled and the load of its base one refill before, so neither
    // round trip is waited on where it is issued.
    unsigned q1 = 0;               // stage 1: a claimed tile index (atomic in flight)
    int q2t = -1;                  // stage 2: a claimed tile (-1: none left) ...
    unsigned long long q2b = 0;    // ... and its base word (load in flight)
    auto base_of = [&](int t, unsigned long long w) {  // the owner publishes it right after its gather
        while ((w >> 62) == 0) w = ld_word(&tile_base[t]);
        return w & kValueMask;
    };
    auto queue = [&](int s, int t, unsigned long long w) {
        S.jt[s] = t;
        if (t < 0) return;
        S.jb[s] = base_of(t, w);
        load(t, s, stream);
    };
    auto refill = [&](int s) {
        queue(s, q2t, q2b);
        q2t = q1 < static_cast<unsigned>(tiles) ? static_cast<int>(q1) : -1;
        if (q2t >= 0) q2b = ld_word(&tile_base[q2t]);
        q1 = atomicAdd(&ws->next_tile, 1u);
    };
    SCAN_STAMP(0);
    if (tid == 0) {
        for (int s = 0; s < kP1; ++s) mbar_init(&S.bar[s], 1);
        mbar_fence_init();
        for (int it = 0; it < kP1 && it < m; ++it) load(c0 + it, it, keep);
    }
    __syncthreads();
    unsigned phase = 0;  // bit s: parity of ring slot s's next bulk completion
    // the tile in ring slot s: its words, per-word nonzero counts (0..4) and the lane's total
    auto fetch = [&](int t, int s, uint32_t* wd, unsigned* c) {
        const size_t tb = static_cast<size_t>(t) * kPTile;
        const int tn = static_cast<int>(n - tb < static_cast<size_t>(kPTile) ? n - tb : kPTile);
        uint8_t* buf = in + s * kPTile;
        const bool bulk = is_bulk(t);  // uniform
        if (bulk) {
            mbar_wait(&S.bar[s], (phase >> s) & 1u);
            phase ^= 1u << s;
        } else {
            for (int j = tid; j < kPTile; j += kPT) buf[j] = j < tn ? mask[tb + j] : 0;
        }
        if (!bulk) __syncthreads();  // the plain loads are visible (outside the branch)
        const uint32_t* wbuf = reinterpret_cast<const uint32_t*>(buf) + warp * 256;
        unsigned lt = 0;  // this warp's 1024 elements: 8 rows of 32 words
#pragma unroll
        for (int r = 0; r < 8; ++r) {
            wd[r] = wbuf[r * 32 + lane];
            c[r] = nz_bytes(wd[r]);
            lt += c[r];
        }
        return lt;
    };
    // ---- pass 1: the chunk's tiles, counted (per tile, for the tile bases)
    unsigned long long lane_acc = 0;
    for (int it = 0; it < m; ++it) {
        uint32_t wd[8];
        unsigned c[8];
        const unsigned lt = fetch(c0 + it, it % kP1, wd, c);
        lane_acc += lt;
        const unsigned wt = __reduce_add_sync(0xffffffffu, lt);
        if (lane == 0) S.wt1[it & 1][warp] = wt;
        __syncthreads();  // every read of the slot is done: refill it kP1 tiles ahead
        if (tid == 0) {
            unsigned x = 0;
#pragma unroll
            for (int w = 0; w < kPT / 32; ++w) x += S.wt1[it & 1][w];
            tile_cnt[c0 + it] = x;
            if (it + kP1 < m) load(c0 + it + kP1, (it + kP1) % kP1, keep);
        }
    }
    // ---- gather: publish this chunk's total, read every chunk's (all CTAs are resident)
    SCAN_STAMP(1);
    {
        const unsigned long long wsum = warp_sum(lane_acc);
        if (lane == 0) S.red[warp][0] = wsum;
        __syncthreads();
        if (tid == 0) {
            unsigned long long x = 0;
            for (int w = 0; w < kPT / 32; ++w) x += S.red[w][0];
            st_word(&chunk_tot[b], kFlagAgg | x);
            // one counter of published chunks (release); only this thread polls it (acquire)
            red_release_add(&ws->published, 1u);
            while (ld_acquire_u32(&ws->published) < static_cast<unsigned>(G)) {
#if ABMX_SCAN_BAR_NS > 0
                __nanosleep(ABMX_SCAN_BAR_NS);  // back off: every CTA's thread 0 polls this one line
#endif
            }
        }
        __syncthreads();  // thread 0's acquire + the barrier: every chunk word is visible
        unsigned long long before = 0, all = 0;
        for (int q = tid; q < G; q += kPT) {
            const unsigned long long v = ld_word(&chunk_tot[q]) & kValueMask;
            all += v;
            if (q < b) before += v;
        }
        before = warp_sum(before);
        all = warp_sum(all);
        if (lane == 0) {
            S.red[warp][0] = before;
            S.red[warp][1] = all;
        }
        __syncthreads();
        if (tid == 0) {
            unsigned long long x = 0, y = 0;
            for (int w = 0; w < kPT / 32; ++w) {
                x += S.red[w][0];
                y += S.red[w][1];
            }
            S.base = x;
            S.T = y;
            if (kCompact && b == 0 && true_out) *true_out = y;  // count_true(mask)
        }
        __syncthreads();
        // the chunk's tile bases: chunk base + exclusive prefix of its tile counts
        unsigned long long carry = S.base;
        for (int k0 = 0; k0 < m; k0 += kPT) {
            const int k = k0 + tid;
            const unsigned long long v = k < m ? tile_cnt[c0 + k] : 0ULL;
            unsigned long long tot;
            const unsigned long long ex = block_excl_scan<kPT>(v, &S.red[0][0], &tot);
            if (k < m) st_word(&tile_base[c0 + k], kFlagAgg | (carry + ex));
            carry += tot;
            __syncthreads();  // S.red is reused by the next round / below
        }
        if (tid == 0) {  // every pass-1 slot is consumed: the first kPIn claims (one atomic, the
                         // base loads in flight together), then prime the pipeline
            const unsigned t0 = atomicAdd(&ws->next_tile, static_cast<unsigned>(kPIn));
            unsigned long long w[kPIn];
#pragma unroll
            for (int s = 0; s < kPIn; ++s) w[s] = t0 + s < static_cast<unsigned>(tiles) ? ld_word(&tile_base[t0 + s]) : 0ULL;
#pragma unroll
            for (int s = 0; s < kPIn; ++s) queue(s, t0 + s < static_cast<unsigned>(tiles) ? static_cast<int>(t0 + s) : -1, w[s]);
            q1 = atomicAdd(&ws->next_tile, 1u);
            q2t = q1 < static_cast<unsigned>(tiles) ? static_cast<int>(q1) : -1;
            if (q2t >= 0) q2b = ld_word(&tile_base[q2t]);
            q1 = atomicAdd(&ws->next_tile, 1u);
        }
        __syncthreads();
    }
    SCAN_STAMP(2);
    // ---- pass 2: claimed tiles, ranked / partitioned from their bases
    for (int p = 0;; ++p) {
        const int s = p % kPIn;
        const int tile = S.jt[s];
        if (tile < 0) break;  // the counter ran out (uniform)
        const unsigned long long run = S.jb[s];
        ABMX_ASSERT(tile < tiles && run <= n);
        const size_t tb = static_cast<size_t>(tile) * kPTile;
        const int tn = static_cast<int>(n - tb < static_cast<size_t>(kPTile) ? n - tb : kPTile);
        if (!kCompact && tid == 0) bulk_wait_read<kPOut - 1>();  // the output stage we reuse is free
        uint32_t wd[8];
        unsigned c[8];
        const unsigned lt = fetch(tile, s, wd, c);
        const unsigned wt = __reduce_add_sync(0xffffffffu, lt);
        if (lane == 0) S.wtot[warp] = wt;
        __syncthreads();  // every read of the slot is done: claim and refill it kPIn tiles ahead
        if (tid == 0) refill(s);
        if (warp == 0) {
            const unsigned v = lane < kPT / 32 ? S.wtot[lane] : 0u;
            unsigned incl = v;
#pragma unroll
            for (int d = 1; d < kPT / 32; d <<= 1) {
                const unsigned u = __shfl_up_sync(0xffffffffu, incl, d);
                if (lane >= d) incl += u;
            }
            const unsigned total = __shfl_sync(0xffffffffu, incl, kPT / 32 - 1);
            if (lane < kPT / 32) S.wtot[lane] = incl - v;  // exclusive warp offsets
            if (lane == 0) S.total = total;
        }
        __syncthreads();
        const int it = p;  // output stage
        const unsigned lt_mask = (1u << lane) - 1u;
        if constexpr (!kCompact) {
            int32_t* o = ob + (it % kPOut) * kPTile;
            int4* o4 = reinterpret_cast<int4*>(o) + warp * 256;
            unsigned x0 = static_cast<unsigned>(run) + S.wtot[warp];
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const unsigned b0 = __ballot_sync(0xffffffffu, c[r] & 1u), b1 = __ballot_sync(0xffffffffu, c[r] & 2u),
                               b2 = __ballot_sync(0xffffffffu, c[r] & 4u);
                unsigned x = x0 + __popc(b0 & lt_mask) + 2u * __popc(b1 & lt_mask) + 4u * __popc(b2 & lt_mask);
                int q[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const bool nz = ((wd[r] >> (8 * k)) & 0xFFu) != 0u;
                    x += nz;
                    q[k] = nz ? static_cast<int>(x) : 0;
                }
                o4[r * 32 + lane] = make_int4(q[0], q[1], q[2], q[3]);
                x0 += __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
            }
            fence_proxy_async_smem();
            __syncthreads();
            if (tn == kPTile && out_vec) {
                if (tid == 0) {
                    bulk_s2g_hint(out + tb, o, kPTile * static_cast<unsigned>(sizeof(int32_t)), stream);
                    bulk_commit();
                }
            } else {
                for (int j = tid; j < tn; j += kPT) out[tb + j] = o[j];
            }
        } else {
            const int ttot = static_cast<int>(S.total);
            // The tile's trues go to out[run, run + ttot), its falses to out[f_dst + ttot, ...).
            // Each run is laid out in shared memory at the same offset mod 4 as its destination,
            // so both are written with 16-byte loads and stores (scalar only at the quad edges).
            const size_t f_dst = S.T + (tb - run) - static_cast<size_t>(ttot);  // + j for false j >= ttot
            // element offset mod 4 of each run's first destination address
            const int at = static_cast<int>((reinterpret_cast<uintptr_t>(out + run) >> 2) & 3u);  // true run shift
            const int fb = ((at + ttot + 3) & ~3) +
                           static_cast<int>((reinterpret_cast<uintptr_t>(out + f_dst + ttot) >> 2) & 3u);  // false base
            int tpre = static_cast<int>(S.wtot[warp]);  // trues before this lane's word, in the tile
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const unsigned b0 = __ballot_sync(0xffffffffu, c[r] & 1u), b1 = __ballot_sync(0xffffffffu, c[r] & 2u),
                               b2 = __ballot_sync(0xffffffffu, c[r] & 4u);
                int x = tpre + __popc(b0 & lt_mask) + 2 * __popc(b1 & lt_mask) + 4 * __popc(b2 & lt_mask);
                const int e0 = warp * 1024 + r * 128 + lane * 4;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int e = e0 + k;
                    ABMX_ASSERT(at + x < kPTile + 16 && fb + e - x < kPTile + 16 && fb + e - x >= 0);
                    if (((wd[r] >> (8 * k)) & 0xFFu) != 0u)
                        ob[at + x++] = static_cast<int32_t>(tb + e);
                    else
                        ob[fb + e - x] = static_cast<int32_t>(tb + e);  // false rank e - x
                }
                tpre += __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
            }
            __syncthreads();
            // a run of len elements: dst[0..len) <- ob[o..o+len), (dst - ob + o) multiple of 4 elements
            auto write_run = [&](int32_t* dst, const int32_t* src, int len) {
                if (len <= 0) return;
                const int head = static_cast<int>((4u - (reinterpret_cast<uintptr_t>(dst) >> 2)) & 3u);
                const int h = head < len ? head : len;
                if (tid < h) dst[tid] = src[tid];
                const int body = (len - h) / 4;
                const int4* s4 = reinterpret_cast<const int4*>(src + h);
                int4* d4 = reinterpret_cast<int4*>(dst + h);
                for (int q = tid; q < body; q += kPT) st_v4_hint(d4 + q, s4[q], stream);
                const int t0 = h + 4 * body;
                if (tid < len - t0) dst[t0 + tid] = src[t0 + tid];
            };
            if ((reinterpret_cast<uintptr_t>(out) & 3) == 0) {
                write_run(out + run, ob + at, ttot);
                write_run(out + f_dst + ttot, ob + fb, tn - ttot);
            } else {  // unaligned output: plain stores
                for (int j = tid; j < tn; j += kPT) out[j < ttot ? run + j : f_dst + j] = j < ttot ? ob[at + j] : ob[fb + j - ttot];
            }
        }
    }
    if (!kCompact && tid == 0) bulk_wait_all();
    SCAN_STAMP(3);
}

// Programmatic dependent launch: a kernel launched with programmatic stream serialization may
// start while its predecessor drains; griddepcontrol.wait blocks until the predecessor has
// completed and its memory is visible.
__device__ __forceinline__ void grid_dep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// ---------------------------------------------------------------- match_first_equal
// vmin / vmax live in an order-preserving unsigned form, both reduced with atomicMin (one pair
// per CTA), so ONE cudaMemsetAsync(0xFF) initialises the workspace (capturable in a graph; no
// host staging): emin = v ^ 2^31 (min of v), emax = ~(v ^ 2^31) (min of emax = max of v).
struct MatchWs {
    unsigned emin, emax;
};
__device__ __forceinline__ int ws_vmin(const MatchWs* ws) { return static_cast<int>(ws->emin ^ 0x80000000u); }
__device__ __forceinline__ int ws_vmax(const MatchWs* ws) { return static_cast<int>(~ws->emax ^ 0x80000000u); }

// Grid-stride loops over 4-element quads (16-byte loads, U quads in flight per thread); a
// scalar loop covers the tail and unaligned inputs. `f(index, value)` sees every element once.
template <int U = 2, bool kStream = false, class F>
__device__ __forceinline__ void for_each_i32(const int32_t* __restrict__ p, size_t n, F&& f) {
    const unsigned long long stream = kStream ? l2_evict_first() : 0ULL;  // read once: do not keep in L2
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    size_t done = 0;
    if ((reinterpret_cast<uintptr_t>(p) & 15) == 0) {
        const size_t quads = n / 4;
        const int4* q = reinterpret_cast<const int4*>(p);
        for (size_t i = t0; i < quads; i += U * stride) {
            int4 a[U];
#pragma unroll
            for (int u = 0; u < U; ++u)
                a[u] = i + u * stride < quads ? (kStream ? ld_v4_hint(q + i + u * stride, stream) : q[i + u * stride])
                                              : make_int4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (i + u * stride >= quads) break;
                const size_t e = 4 * (i + u * stride);
                f(e, a[u].x);
                f(e + 1, a[u].y);
                f(e + 2, a[u].z);
                f(e + 3, a[u].w);
            }
        }
        done = 4 * quads;
    }
    for (size_t j = done + t0; j < n; j += stride) f(j, p[j]);
}

__global__ void minmax_kernel(const int32_t* __restrict__ rb, size_t m, MatchWs* ws) {
    int lo = INT_MAX, hi = INT_MIN;
    for_each_i32<8, true>(rb, m, [&](size_t, int v) {
        lo = min(lo, v);
        hi = max(hi, v);
    });
    // one atomic pair per CTA: per-warp atomics on the same two words serialise at one L2 slice
    __shared__ int s_lo[32], s_hi[32];
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane == 0) {
        s_lo[warp] = lo;
        s_hi[warp] = hi;
    }
    __syncthreads();
    if (warp == 0) {
        lo = lane < nw ? s_lo[lane] : INT_MAX;
        hi = lane < nw ? s_hi[lane] : INT_MIN;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
            hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
        }
        if (lane == 0) {
            atomicMin(&ws->emin, static_cast<unsigned>(lo) ^ 0x80000000u);
            atomicMin(&ws->emax, ~(static_cast<unsigned>(hi) ^ 0x80000000u));
        }
    }
}

__device__ __forceinline__ bool dense_mode(const MatchWs* ws, unsigned bits) {
    const long long range = static_cast<long long>(ws_vmax(ws)) - ws_vmin(ws) + 1;
    return range <= (1LL << bits);
}

__device__ __forceinline__ unsigned hash32(uint32_t k, unsigned bits) {
    return static_cast<unsigned>(mix64(k) >> (64 - bits));
}

// vals[] starts at INT_MAX; keys[] (hash mode) start at 0 = empty, else (key << 1) | 1.
// Initialise only what the chosen mode reads (after minmax): dense -> vals[0, range);
// hash -> vals[0, H) and keys[0, H). Memsetting both full tables up front wrote 12*H bytes.
__global__ void match_init_kernel(const MatchWs* ws, unsigned bits, int* __restrict__ vals,
                                  unsigned long long* __restrict__ keys) {
    grid_dep_wait();  // launched early (PDL): the previous kernel's writes are visible after this
    const bool dense = dense_mode(ws, bits);
    const size_t H = size_t{1} << bits;
    const size_t nv = dense ? static_cast<size_t>(static_cast<long long>(ws_vmax(ws)) - ws_vmin(ws) + 1) : H;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // INT_MAX = "no row": above any row index, and what the lookup maps to -1
    // the table stays in L2 for the build's atomics and the lookup's gathers (evict_last); the
    // streams of rb, ra and the output pass it by (evict_first)
    const int4 fill = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);
    const unsigned long long keep = l2_evict_last();
    for (size_t i = t0; i < nv / 4; i += stride) st_v4_hint(reinterpret_cast<int4*>(vals) + i, fill, keep);
    for (size_t i = (nv & ~size_t{3}) + t0; i < nv; i += stride) vals[i] = INT_MAX;
    if (!dense)
        for (size_t i = t0; i < H / 2; i += stride) reinterpret_cast<ulonglong2*>(keys)[i] = make_ulonglong2(0, 0);
}

__global__ void match_build_kernel(const int32_t* __restrict__ rb, size_t m, const MatchWs* ws, unsigned bits,
                                   int* __restrict__ vals, unsigned long long* __restrict__ keys) {
    grid_dep_wait();  // launched early (PDL): the previous kernel's writes are visible after this
    const bool dense = dense_mode(ws, bits);
    const unsigned mask = (1u << bits) - 1u;
    const int vmin = ws_vmin(ws);
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    if (dense && (reinterpret_cast<uintptr_t>(rb) & 15) == 0) {
        // quads: all 8 first-match checks are issued before any atomic (an atomic between two
        // checks would serialise them: the compiler cannot move a load across a possibly
        // aliasing atomic)
        // kQ quads per thread and iteration: both dependent round trips (the quads, then the
        // checks) carry 4 * kQ values
        constexpr int kQ = 4;
        const unsigned long long stream = l2_evict_first();
        const size_t quads = m / 4;
        const int4* q = reinterpret_cast<const int4*>(rb);
        for (size_t i = t0; i < quads; i += kQ * stride) {
            int v[4 * kQ];
#pragma unroll
            for (int u = 0; u < kQ; ++u) {
                const int4 a = i + u * stride < quads ? ld_v4_hint(q + i + u * stride, stream) : make_int4(0, 0, 0, 0);
                v[4 * u] = a.x;
                v[4 * u + 1] = a.y;
                v[4 * u + 2] = a.z;
                v[4 * u + 3] = a.w;
            }
            int cur[4 * kQ];
#pragma unroll
            for (int k = 0; k < 4 * kQ; ++k) cur[k] = v[k] != 0 ? __ldcg(&vals[v[k] - vmin]) : INT_MIN;
#pragma unroll
            for (int k = 0; k < 4 * kQ; ++k) {
                const int j = static_cast<int>(4 * (i + (k / 4) * stride) + (k & 3));
                if (cur[k] > j) atomicMin(&vals[v[k] - vmin], j);  // rank 0 (never looked up) skipped
            }
        }
        for (size_t j = 4 * quads + t0; j < m; j += stride) {
            const int v = rb[j];
            if (v != 0 && __ldcg(&vals[v - vmin]) > static_cast<int>(j)) atomicMin(&vals[v - vmin], static_cast<int>(j));
        }
        return;
    }
    for_each_i32(rb, m, [&](size_t j, int v) {
        // rank 0 means "not selected" and is never looked up (match_lookup_kernel): skipping it
        // removes the one hot word every unselected row would hammer
        if (v == 0) return;
        if (dense) {
            int* slot = &vals[v - vmin];
            if (__ldcg(slot) > static_cast<int>(j)) atomicMin(slot, static_cast<int>(j));  // duplicates: skip
        } else {
            const unsigned long long key = (static_cast<unsigned long long>(static_cast<uint32_t>(v)) << 1) | 1ULL;
            unsigned h = hash32(static_cast<uint32_t>(v), bits);
            for (;;) {
                const unsigned long long prev = atomicCAS(&keys[h], 0ULL, key);
                if (prev == 0ULL || prev == key) {
                    if (__ldcg(&vals[h]) > static_cast<int>(j)) atomicMin(&vals[h], static_cast<int>(j));
                    break;
                }
                h = (h + 1) & mask;
            }
        }
    });
}

__device__ __forceinline__ int match_one(int r, bool dense, unsigned bits, long long lo, long long hi, const int* vals,
                                         const unsigned long long* keys) {
    if (r == 0 || r < lo || r > hi) return -1;
    int j = INT_MAX;
    if (dense) {
        j = vals[r - lo];
    } else {
        const unsigned mask = (1u << bits) - 1u;
        const unsigned long long key = (static_cast<unsigned long long>(static_cast<uint32_t>(r)) << 1) | 1ULL;
        unsigned h = hash32(static_cast<uint32_t>(r), bits);
        for (;;) {
            const unsigned long long k = keys[h];
            if (k == key) {
                j = vals[h];
                break;
            }
            if (k == 0ULL) break;
            h = (h + 1) & mask;
        }
    }
    return j != INT_MAX ? j : -1;
}

template <bool kDense>
__device__ __forceinline__ void match_lookup_body(const int32_t* __restrict__ ra, size_t n, unsigned bits, long long lo,
                                                  long long hi, const int* __restrict__ vals,
                                                  const unsigned long long* __restrict__ keys,
                                                  int32_t* __restrict__ row_out) {
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    size_t done = 0;
    auto one = [&](int r) { return match_one(r, kDense, bits, lo, hi, vals, keys); };
    if (((reinterpret_cast<uintptr_t>(ra) | reinterpret_cast<uintptr_t>(row_out)) & 15) == 0) {
        // quads in, quads out; two quads in flight per thread
        const size_t quads = n / 4;
        const int4* q = reinterpret_cast<const int4*>(ra);
        int4* o = reinterpret_cast<int4*>(row_out);
        const unsigned long long stream = l2_evict_first();
        for (size_t i = t0; i < quads; i += 2 * stride) {
            const bool two = i + stride < quads;
            const int4 a = ld_v4_hint(q + i, stream);
            const int4 b = two ? ld_v4_hint(q + i + stride, stream) : make_int4(0, 0, 0, 0);
            st_v4_hint(o + i, make_int4(one(a.x), one(a.y), one(a.z), one(a.w)), stream);
            if (two) st_v4_hint(o + i + stride, make_int4(one(b.x), one(b.y), one(b.z), one(b.w)), stream);
        }
        done = 4 * quads;
    }
    for (size_t j = done + t0; j < n; j += stride) row_out[j] = one(ra[j]);
}

__global__ void match_lookup_kernel(const int32_t* __restrict__ ra, size_t n, const MatchWs* ws, unsigned bits,
                                    const int* __restrict__ vals,
                                    const unsigned long long* __restrict__ keys,
                                    int32_t* __restrict__ row_out) {
    grid_dep_wait();  // launched early (PDL): the build's table is visible after this
    const long long lo = ws_vmin(ws), hi = ws_vmax(ws);
    if (dense_mode(ws, bits))  // uniform: the dense loop compiles without the probing path
        match_lookup_body<true>(ra, n, bits, lo, hi, vals, keys, row_out);
    else
        match_lookup_body<false>(ra, n, bits, lo, hi, vals, keys, row_out);
}

// ---------------------------------------------------------------- blends
// Blend, lane-contiguous: a warp owns 32 * kV consecutive 16-byte vectors of a / b / out; at
// step q lane l takes vector q * 32 + l (and the mask bytes of its elements), so every load and
// store instruction covers 512 contiguous bytes. A lane owning 16 consecutive elements made
// each instruction touch 32 different lines: 420 us for 2^26 i64 against 236 us for torch.where.
template <int B>
struct MaskChunk;  // the mask bytes of one 16-byte vector of elements
template <>
struct MaskChunk<2> {
    using type = uint16_t;
    __device__ static bool on(type m, int k) { return (m >> (8 * k)) & 0xFFu; }
};
template <>
struct MaskChunk<16> {
    using type = uint4;
    __device__ static bool on(type m, int k) {
        const uint32_t w = k < 4 ? m.x : k < 8 ? m.y : k < 12 ? m.z : m.w;
        return (w >> (8 * (k & 3))) & 0xFFu;
    }
};
template <class T>
__global__ void __launch_bounds__(kThreads) blend_kernel(const uint8_t* mask, const T* a, const T* b,
                                                         T* out, size_t n) {
    constexpr int kPerVec = 16 / sizeof(T);
    constexpr int kV = 8;  // 16-byte vectors per lane: all loads in flight before any store
    constexpr size_t kChunk = static_cast<size_t>(32) * kV * kPerVec;  // elements per warp
    using MC = MaskChunk<kPerVec>;
    const bool vec = ((reinterpret_cast<uintptr_t>(mask) | reinterpret_cast<uintptr_t>(a) |
                       reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    const int lane = threadIdx.x & 31;
    const size_t warps = static_cast<size_t>(gridDim.x) * (kThreads / 32);
    for (size_t w = (static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x) >> 5; w * kChunk < n; w += warps) {
        const size_t e0 = w * kChunk;
        if (vec && e0 + kChunk <= n) {
            // `out` may alias a or b (same index only): every element is read before it is written
            const size_t v0 = e0 / kPerVec;
            const uint4* a4 = reinterpret_cast<const uint4*>(a) + v0;
            const uint4* b4 = reinterpret_cast<const uint4*>(b) + v0;
            const typename MC::type* m4 = reinterpret_cast<const typename MC::type*>(mask + e0);
            uint4 va[kV], vb[kV];
            typename MC::type mk[kV];
#pragma unroll
            for (int q = 0; q < kV; ++q) {
                va[q] = a4[q * 32 + lane];
                vb[q] = b4[q * 32 + lane];
                mk[q] = m4[q * 32 + lane];
            }
            uint4* o4 = reinterpret_cast<uint4*>(out) + v0;
#pragma unroll
            for (int q = 0; q < kV; ++q) {
                T* ea = reinterpret_cast<T*>(&va[q]);
                const T* eb = reinterpret_cast<const T*>(&vb[q]);
#pragma unroll
                for (int k = 0; k < kPerVec; ++k)
                    if (!MC::on(mk[q], k)) ea[k] = eb[k];
                o4[q * 32 + lane] = va[q];
            }
        } else {
            for (size_t i = e0 + lane; i < e0 + kChunk && i < n; i += 32) out[i] = mask[i] ? a[i] : b[i];
        }
    }
}

}  // namespace abmx_table

#ifdef ABMX_SCAN_TRACE
extern "C" int abmx_scan_trace(unsigned long long* out, int ctas) {
    return cudaMemcpyFromSymbol(out, abmx_table::g_scan_trace, sizeof(unsigned long long) * 4 * ctas) == cudaSuccess ? 0 : -1;
}
#endif

// ====================================================================== launchers
using namespace abmx_table;

namespace abmx_internal {

static int grid_for(size_t n, int per_block) {
    const size_t g = (n + per_block - 1) / per_block;
    const size_t cap = static_cast<size_t>(num_sms()) * 8;
    return static_cast<int>(g < cap ? (g > 0 ? g : 1) : cap);
}

// persistent pipelined scan (rank_scan / compact_indices): workspace = one word per CTA chunk
template <bool kCompact>
static cudaError_t launch_scan_pipe(const uint8_t* d_mask, int32_t* d_out, size_t n, unsigned long long* d_true,
                                    cudaStream_t s) {
    const size_t tiles = (n + kPTile - 1) / kPTile;
    constexpr int smem = pipe_smem<kCompact>();
    cudaError_t e = raise_dyn_smem(scan_pipe_kernel<kCompact>, static_cast<size_t>(smem));
    if (e != cudaSuccess) return e;
    // co-resident grid: every CTA waits for all chunk totals (cooperative launch guarantees it)
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, scan_pipe_kernel<kCompact>, kPT, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorLaunchOutOfResources;
    constexpr int want = kCompact ? kCMinB : kPMinB;
    const size_t cap = static_cast<size_t>(num_sms()) * static_cast<size_t>(per_sm < want ? per_sm : want);
    const unsigned grid = static_cast<unsigned>(tiles < cap ? tiles : cap);
    void* ws = nullptr;
    // chunk totals, counters and flagged tile bases (zeroed), then the tile counts (written before read)
    const size_t zero_bytes = grid * sizeof(unsigned long long) + sizeof(ScanWs) + tiles * sizeof(unsigned long long);
    const size_t ws_bytes = zero_bytes + tiles * sizeof(unsigned);
    e = abmx_internal::malloc_async(&ws, ws_bytes, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(ws, 0, zero_bytes, s);
    (void)cudaGetLastError();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kPT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, scan_pipe_kernel<kCompact>, d_mask, d_out, n, static_cast<int>(tiles),
                           static_cast<unsigned long long*>(ws), d_true);
    count_launch();
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaFreeAsync(ws, s);
    return e;
}

cudaError_t launch_rank_scan(const uint8_t* d_mask, int32_t* d_ranks, size_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    return launch_scan_pipe<false>(d_mask, d_ranks, n, nullptr, s);
}

cudaError_t launch_count_true(const uint8_t* d_mask, size_t n, unsigned long long* d_out,
                              cudaStream_t s) {
    (void)cudaGetLastError();
    zero_words_kernel<<<1, 32, 0, s>>>(d_out, 1);
    if (n == 0) {
        count_launch();
        return cudaGetLastError();
    }
    // the count streams the mask while the zeroing runs; it waits for it only before its atomic
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t c{};
    c.gridDim = dim3(static_cast<unsigned>(grid_for(n, kThreads * kCountItems)));
    c.blockDim = dim3(kThreads);
    c.stream = s;
    c.attrs = pdl;
    c.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&c, count_true_kernel, d_mask, n, d_out);
    count_launch(2);
    return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_compact_indices(const uint8_t* d_mask, int32_t* d_out, size_t n,
                                   unsigned long long* d_count, cudaStream_t s) {
    if (n == 0) return cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
    // one kernel: the false run starts at count_true(mask), which the chunk gather provides
    return launch_scan_pipe<true>(d_mask, d_out, n, d_count, s);
}

cudaError_t launch_match_first_equal(const int32_t* d_ra, size_t n, const int32_t* d_rb, size_t m,
                                     int32_t* d_out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    if (m == 0) return cudaMemsetAsync(d_out, 0xFF, n * sizeof(int32_t), s);  // all -1
    unsigned bits = 6;
    while ((1ULL << bits) < 2ULL * m) ++bits;
    const size_t H = 1ULL << bits;
    const size_t ws_bytes = 256 + H * sizeof(int) + H * sizeof(unsigned long long);
    void* ws = nullptr;
    cudaError_t e = abmx_internal::malloc_async(&ws, ws_bytes, s);
    if (e != cudaSuccess) return e;
    auto* mws = static_cast<MatchWs*>(ws);
    int* vals = reinterpret_cast<int*>(static_cast<char*>(ws) + 256);
    auto* keys = reinterpret_cast<unsigned long long*>(static_cast<char*>(ws) + 256 + H * sizeof(int));
    cudaMemsetAsync(mws, 0xFF, sizeof(MatchWs), s);  // emin = emax = UINT_MAX (see MatchWs)
    const int gm = grid_for(m, 256 * 8), gn = grid_for(n, 256 * 8);
    (void)cudaGetLastError();
    minmax_kernel<<<gm, 256, 0, s>>>(d_rb, m, mws);
    // init, build and lookup launch with programmatic stream serialization (each waits in-kernel
    // for its predecessor), so their launch latency overlaps the predecessor's tail
    cudaLaunchAttribute pdl[1];
    pdl[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    pdl[0].val.programmaticStreamSerializationAllowed = 1;
    auto cfg_of = [&](unsigned grid) {
        cudaLaunchConfig_t c{};
        c.gridDim = dim3(grid);
        c.blockDim = dim3(256);
        c.stream = s;
        c.attrs = pdl;
        c.numAttrs = 1;
        return c;
    };
    cudaLaunchConfig_t c1 = cfg_of(static_cast<unsigned>(num_sms() * 8)), c2 = cfg_of(static_cast<unsigned>(gm)),
                       c3 = cfg_of(static_cast<unsigned>(gn));
    e = cudaLaunchKernelEx(&c1, match_init_kernel, static_cast<const MatchWs*>(mws), bits, vals, keys);
    if (e == cudaSuccess)
        e = cudaLaunchKernelEx(&c2, match_build_kernel, static_cast<const int32_t*>(d_rb), m,
                               static_cast<const MatchWs*>(mws), bits, vals, keys);
    if (e == cudaSuccess)
        e = cudaLaunchKernelEx(&c3, match_lookup_kernel, static_cast<const int32_t*>(d_ra), n,
                               static_cast<const MatchWs*>(mws), bits, static_cast<const int*>(vals),
                               static_cast<const unsigned long long*>(keys), d_out);
    count_launch(4);
    if (e == cudaSuccess) e = cudaGetLastError();
    cudaFreeAsync(ws, s);
    return e;
}

template <class T>
cudaError_t launch_blend(const uint8_t* d_mask, const T* d_a, const T* d_b, T* d_out, size_t n,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    (void)cudaGetLastError();
    // one warp chunk (32 x 8 vectors of 16 bytes) per warp: a flat grid, no grid-stride rounds
    constexpr size_t kChunk = static_cast<size_t>(32) * 8 * (16 / sizeof(T));
    const size_t warps = (n + kChunk - 1) / kChunk;
    const size_t ctas = (warps + kThreads / 32 - 1) / (kThreads / 32);
    blend_kernel<T><<<static_cast<unsigned>(ctas < 0x7FFFFFFF ? ctas : 0x7FFFFFFF), kThreads, 0, s>>>(d_mask, d_a, d_b,
                                                                                                    d_out, n);
    count_launch();
    return cudaGetLastError();
}

template cudaError_t launch_blend<int64_t>(const uint8_t*, const int64_t*, const int64_t*, int64_t*,
                                           size_t, cudaStream_t);
template cudaError_t launch_blend<unsigned long long>(const uint8_t*, const unsigned long long*,
                                                      const unsigned long long*, unsigned long long*,
                                                      size_t, cudaStream_t);
template cudaError_t launch_blend<uint8_t>(const uint8_t*, const uint8_t*, const uint8_t*, uint8_t*,
                                           size_t, cudaStream_t);

}  // namespace abmx_internal
