// abmx_device.cuh — shared device primitives for the sm_100a engine.
//
//  * counter-based RNG, bit-exact with the reference RngState (src/rng.cpp:12-40)
//  * packed two-counter decoupled-lookback tile scan (single pass, warp-ballot lookback)
//  * block-level helpers
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace abmx_dev {

// ------------------------------------------------------------------ RNG
// draw(c)  = mix64(key + 0x9E3779B97F4A7C15 * (c + 1))        src/rng.cpp:22-24
// split(i) = mix64(key + 0xC2B2AE3D27D4EB4F * (i + 1))        src/rng.cpp:18-20
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__host__ __device__ __forceinline__ uint64_t split(uint64_t key, uint64_t i) {
    return mix64(key + 0xC2B2AE3D27D4EB4FULL * (i + 1));
}
__host__ __device__ __forceinline__ uint64_t draw(uint64_t key, uint64_t c) {
    return mix64(key + 0x9E3779B97F4A7C15ULL * (c + 1));
}
// uniform_int(c, 0, span) = high64(draw * span)                src/rng.cpp:30-36
__device__ __forceinline__ uint64_t uniform_span(uint64_t key, uint64_t c, uint64_t span) {
    return __umul64hi(draw(key, c), span);
}
// (draw >> 11) * 2^-53: the u64->f64 conversion is exact for 53-bit values  src/rng.cpp:26-28
__device__ __forceinline__ double uniform_double(uint64_t key, uint64_t c) {
    return __dmul_rn(__ull2double_rn(draw(key, c) >> 11), 0x1.0p-53);
}

// ------------------------------------------------------------------ memory order
// The lookback words carry their payload in the word itself (flag + counts in one u64), so
// relaxed GPU-scope accesses are enough: no other data is published through them. (An
// ld.acquire.gpu would make ptxas emit CCTL.IVALL, an L1 invalidate, on every poll.)
__device__ __forceinline__ void st_word(unsigned long long* p, unsigned long long v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_word(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void red_release_add(unsigned* p, unsigned v) {  // publishes this thread's prior writes
    asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// start a global-memory line's fetch into L2, no register result
__device__ __forceinline__ void prefetch_l2(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned ld_word_u32(const unsigned* p) {
    unsigned v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// ------------------------------------------------------------------ packed counters
// Two non-negative counts (each < 2^31) share one u64 so a tile publishes both of
// its aggregates (e.g. free-slot and valid-row counts) with one store. Bits 63..62
// hold the lookback flag.
constexpr unsigned long long kFlagAgg = 1ULL << 62;
constexpr unsigned long long kFlagPrefix = 2ULL << 62;
constexpr unsigned long long kValueMask = (1ULL << 62) - 1;

__host__ __device__ __forceinline__ unsigned long long pack2(uint32_t a, uint32_t b) {
    return (static_cast<unsigned long long>(a) << 31) | b;
}
__host__ __device__ __forceinline__ uint32_t lo31(unsigned long long v) {
    return static_cast<uint32_t>(v & 0x7FFFFFFFULL);
}
__host__ __device__ __forceinline__ uint32_t hi31(unsigned long long v) {
    return static_cast<uint32_t>((v >> 31) & 0x7FFFFFFFULL);
}

// The eight Moore moves in the order of lifecycle.cpp:87-122 (u = draw >> 61), as 2-bit fields of
// immediates: a lookup with a per-thread index into __constant__ memory serialises across the warp.
constexpr int kMoveDx[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
constexpr int kMoveDy[8] = {-1, 0, 1, -1, 1, -1, 0, 1};
constexpr unsigned move_table(const int* d) {
    unsigned v = 0;
    for (int u = 0; u < 8; ++u) v |= static_cast<unsigned>(d[u] + 1) << (2 * u);
    return v;
}
constexpr unsigned kDxTable = move_table(kMoveDx), kDyTable = move_table(kMoveDy);
__device__ __forceinline__ int move_dx(int u) { return static_cast<int>((kDxTable >> (2 * u)) & 3u) - 1; }
__device__ __forceinline__ int move_dy(int u) { return static_cast<int>((kDyTable >> (2 * u)) & 3u) - 1; }

// Device asserts of checked builds (-DABMX_CHECKED; compute-sanitizer is closed on the GPU pool):
// a failed condition traps, so the launch fails with an error the caller sees. No code otherwise.
#ifdef ABMX_CHECKED
#define ABMX_ASSERT(cond) \
    do {                  \
        if (!(cond)) __trap(); \
    } while (0)
#else
#define ABMX_ASSERT(cond) ((void)0)
#endif

// Warp-inclusive scan of packed u64 values (fields never overflow by construction).
__device__ __forceinline__ unsigned long long warp_incl_scan(unsigned long long v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const unsigned long long n = __shfl_up_sync(0xffffffffu, v, d);
        if (lane >= d) v += n;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}

// Block exclusive scan of a packed value. `smem` needs (blockDim/32 + 1) entries.
// Returns the exclusive prefix for this thread; *block_total receives the tile sum.
template <int kThreads>
__device__ __forceinline__ unsigned long long block_excl_scan(unsigned long long v,
                                                              unsigned long long* smem,
                                                              unsigned long long* block_total) {
    if constexpr (kThreads == 32) {  // one-warp CTA: no shared memory, warp barriers only
        __syncwarp();
        const unsigned long long incl1 = warp_incl_scan(v);
        *block_total = __shfl_sync(0xffffffffu, incl1, 31);
        __syncwarp();
        return incl1 - v;
    }
    constexpr int kWarps = kThreads / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned long long incl = warp_incl_scan(v);
    if (lane == 31) smem[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < kWarps ? smem[lane] : 0ULL;
        const unsigned long long wi = warp_incl_scan(w);
        if (lane < kWarps) smem[lane] = wi - w;  // exclusive warp offsets
        if (lane == kWarps - 1) smem[kWarps] = wi;
    }
    __syncthreads();
    *block_total = smem[kWarps];
    return smem[warp] + incl - v;
}

// Block exclusive scan of a small count (the block total stays below 2^32).
template <int kThreads>
__device__ __forceinline__ unsigned block_excl_count(unsigned v, unsigned long long* smem, unsigned* block_total) {
    if constexpr (kThreads == 32) {
        __syncwarp();
        const int lane = threadIdx.x & 31;
        unsigned x = v;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const unsigned n = __shfl_up_sync(0xffffffffu, x, d);
            if (lane >= d) x += n;
        }
        *block_total = __shfl_sync(0xffffffffu, x, 31);
        __syncwarp();
        return x - v;
    } else {
        unsigned long long t;
        const unsigned long long e = block_excl_scan<kThreads>(v, smem, &t);
        *block_total = static_cast<unsigned>(t);
        return static_cast<unsigned>(e);
    }
}

// Decoupled lookback (single pass). Called by ONE full warp of the tile after the tile
// aggregate is known. `status` entries start at 0 (invalid). Tiles must be processed in
// ticket order (tile k obtained its ticket after tiles < k), which guarantees progress.
// Returns the exclusive prefix of this tile (flag bits stripped), valid in all lanes.
__device__ __forceinline__ unsigned long long tile_lookback(unsigned long long* status, int tile,
                                                            unsigned long long aggregate) {
    const int lane = threadIdx.x & 31;
    if (tile == 0) {
        if (lane == 0) st_word(&status[0], kFlagPrefix | aggregate);
        return 0ULL;
    }
    if (lane == 0) st_word(&status[tile], kFlagAgg | aggregate);
    unsigned long long excl = 0ULL;
    int end = tile - 1;  // closest predecessor examined by lane 0
    for (;;) {
        const int j = end - lane;
        unsigned long long sv = j >= 0 ? ld_word(&status[j]) : kFlagPrefix;
        // spin (convergently) until every examined predecessor has published something
        while (__any_sync(0xffffffffu, (sv >> 62) == 0)) {
            if ((sv >> 62) == 0) {
                __nanosleep(32);
                sv = ld_word(&status[j]);
            }
        }
        const unsigned pmask = __ballot_sync(0xffffffffu, (sv >> 62) == 2);
        unsigned long long contrib = sv & kValueMask;
        if (pmask) {
            const int first = __ffs(pmask) - 1;  // closest tile with an inclusive prefix
            if (lane > first) contrib = 0ULL;
            excl += warp_sum(contrib);
            break;
        }
        excl += warp_sum(contrib);
        end -= 32;
    }
    if (lane == 0) st_word(&status[tile], kFlagPrefix | (excl + aggregate));
    return excl;
}

// Block-wide decoupled lookback: every thread of the CTA inspects one predecessor, so one
// round trip covers kThreads tiles (the warp-wide version needs tile/32 round trips when the
// predecessors have only published aggregates, which is the common case for a wide first
// wave). Called by ALL threads; returns the exclusive prefix (flags stripped) in all threads.
// `red` needs kThreads/32 + 2 entries.
template <int kThreads>
__device__ __forceinline__ unsigned long long block_lookback(unsigned long long* status, int tile,
                                                             unsigned long long aggregate,
                                                             unsigned long long* red) {
    constexpr int kWarps = kThreads / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tile == 0) {
        if (tid == 0) st_word(&status[0], kFlagPrefix | aggregate);
        return 0ULL;
    }
    if (tid == 0) st_word(&status[tile], kFlagAgg | aggregate);
    unsigned long long excl = 0ULL;
    int end = tile - 1;
    for (;;) {
        const int j = end - tid;
        unsigned long long v = kFlagPrefix;  // virtual zero prefix before tile 0
        if (j >= 0) {
            v = ld_word(&status[j]);
            while ((v >> 62) == 0) {
                __nanosleep(20);
                v = ld_word(&status[j]);
            }
        }
        // closest predecessor (smallest tid) holding an inclusive prefix
        const unsigned pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        if (lane == 0) red[warp] = pm ? static_cast<unsigned long long>(warp * 32 + __ffs(pm) - 1) : ~0ULL;
        __syncthreads();
        if (tid == 0) {
            unsigned long long f = ~0ULL;
            for (int w = 0; w < kWarps; ++w) f = red[w] < f ? red[w] : f;
            red[kWarps] = f;
        }
        __syncthreads();
        const unsigned long long first = red[kWarps];
        unsigned long long c = (static_cast<unsigned long long>(tid) <= first) ? (v & kValueMask) : 0ULL;
        c = warp_sum(c);
        __syncthreads();
        if (lane == 0) red[warp] = c;
        __syncthreads();
        if (tid == 0) {
            unsigned long long t = 0;
            for (int w = 0; w < kWarps; ++w) t += red[w];
            red[kWarps + 1] = t;
        }
        __syncthreads();
        excl += red[kWarps + 1];
        if (first != ~0ULL) break;
        end -= kThreads;
        __syncthreads();
    }
    if (tid == 0) st_word(&status[tile], kFlagPrefix | (excl + aggregate));
    return excl;
}


// ---------------------------------------------------------------- TMA bulk copies + mbarriers
// 1-D bulk copies (cp.async.bulk; SASS UBLKCP): 16-byte aligned addresses, sizes multiple of 16.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n }" ::"r"(
            smem_u32(bar)),
        "r"(phase)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
                 : "memory");
}
// L2 eviction-priority policies for the .L2::cache_hint forms below (createpolicy)
__device__ __forceinline__ unsigned long long l2_evict_last() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ unsigned long long l2_evict_first() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void* dst, const void* src, unsigned bytes, unsigned long long policy) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"(smem_u32(src)), "r"(bytes), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ int4 ld_v4_hint(const int4* p, unsigned long long policy) {
    int4 v;
    asm volatile("ld.global.L2::cache_hint.v4.s32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p), "l"(policy));
    return v;
}
__device__ __forceinline__ void st_v4_hint(int4* p, int4 v, unsigned long long policy) {
    asm volatile("st.global.L2::cache_hint.v4.s32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w), "l"(policy)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // <= N groups still reading shared memory
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// generic-proxy shared-memory writes -> visible to the async proxy (before a bulk store)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Warp-aggregated atomic increment: every lane with `pred` receives a unique index.
__device__ __forceinline__ unsigned warp_append(unsigned* counter, bool pred) {
    const unsigned mask = __ballot_sync(__activemask(), pred);
    if (!pred) return 0u;
    const int lane = threadIdx.x & 31;
    const int leader = __ffs(mask) - 1;
    unsigned base = 0;
    if (lane == leader) base = atomicAdd(counter, static_cast<unsigned>(__popc(mask)));
    base = __shfl_sync(mask, base, leader);
    return base + __popc(mask & ((1u << lane) - 1u));
}

}  // namespace abmx_dev
