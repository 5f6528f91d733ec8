// table.cu — sm_100a implementations of the reference KernelTable entries
// (include/abmx/simd/kernels.hpp:15-43; scalar semantics src/simd/kernels_scalar.cpp:7-54).
//
// All entries are HBM-streaming integer/bitwise kernels:
//   rank_scan        single-pass decoupled-lookback scan, 16 mask bytes per thread
//   count_true       grid-stride popcount reduction
//   compact_indices  count, then single-pass scan with a two-sided scatter
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
constexpr int kItems = 16;  // mask bytes per thread
constexpr int kTile = kThreads * kItems;
constexpr int kCountItems = 64;
#ifndef ABMX_SCAN_ITEMS
#define ABMX_SCAN_ITEMS 64
#endif
constexpr int kScanItems = ABMX_SCAN_ITEMS;  // mask bytes per thread in rank_scan / compact
constexpr int kScanTile = kThreads * kScanItems;
#ifndef ABMX_COMPACT_ITEMS
#define ABMX_COMPACT_ITEMS 64
#endif
constexpr int kCompactItems = ABMX_COMPACT_ITEMS;  // the tile is staged in dynamic SMEM
constexpr int kCompactTile = kThreads * kCompactItems;

struct ScanWs {
    unsigned ticket;
    unsigned pad;
    unsigned long long status[1];  // [tiles]
};

template <int I>
__device__ __forceinline__ void load_mask(const uint8_t* mask, size_t base, size_t n, bool vec_ok,
                                          uint8_t (&b)[I]) {
    if (vec_ok && base + I <= n) {
#pragma unroll
        for (int q = 0; q < I / 16; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(mask + base + 16 * q);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 16; ++k) b[16 * q + k] = static_cast<uint8_t>(w[k >> 2] >> (8 * (k & 3)));
        }
    } else {
#pragma unroll
        for (int k = 0; k < I; ++k) b[k] = base + k < n ? mask[base + k] : 0;
    }
}

__device__ __forceinline__ void load_mask16(const uint8_t* mask, size_t base, size_t n,
                                            bool vec_ok, uint8_t (&b)[kItems]) {
    load_mask<kItems>(mask, base, n, vec_ok, b);
}

// ranks[i] = mask[i] ? inclusive_prefix_sum(mask != 0)[i] : 0
template <int I>
__global__ void __launch_bounds__(kThreads) rank_scan_kernel(const uint8_t* __restrict__ mask,
                                                             int32_t* __restrict__ ranks, size_t n,
                                                             ScanWs* ws) {
    __shared__ unsigned long long s_scan[kThreads / 32 + 1];
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_look[kThreads / 32 + 2];
    if (threadIdx.x == 0) s_tile = atomicAdd(&ws->ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const size_t base = static_cast<size_t>(tile) * (kThreads * I) + static_cast<size_t>(threadIdx.x) * I;
    const bool vec_in = (reinterpret_cast<uintptr_t>(mask) & 15) == 0;
    uint8_t b[I];
    load_mask<I>(mask, base, n, vec_in, b);
    unsigned cnt = 0;
#pragma unroll
    for (int k = 0; k < I; ++k) cnt += b[k] != 0;
    unsigned long long total;
    const unsigned long long excl = block_excl_scan<kThreads>(cnt, s_scan, &total);
    __syncthreads();
    const unsigned long long tile_prefix = block_lookback<kThreads>(ws->status, static_cast<int>(tile), total, s_look);
    int32_t run = static_cast<int32_t>(tile_prefix + excl);
    // Stage the tile's ranks in SMEM (row stride I + 1: conflict-free both ways), then store
    // coalesced; each thread's own 4*I contiguous bytes made every warp store touch 32 sectors.
    extern __shared__ int32_t s_r[];  // [kThreads * (I + 1)], dynamic
#pragma unroll
    for (int k = 0; k < I; ++k) {
        run += b[k] != 0;
        s_r[threadIdx.x * (I + 1) + k] = b[k] ? run : 0;
    }
    __syncthreads();
    const size_t tile_base = static_cast<size_t>(tile) * (kThreads * I);
    const int tile_n = static_cast<int>(n - tile_base < static_cast<size_t>(kThreads * I) ? n - tile_base
                                                                                       : kThreads * I);
    for (int j = threadIdx.x; j < tile_n; j += kThreads) ranks[tile_base + j] = s_r[j + j / I];
}

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
        if (threadIdx.x == 0 && v) atomicAdd(out, v);
    }
}

// Stable partition of 0..n-1: true indices first (ascending), then false indices.
// `true_total` is the precomputed count_true (device memory).
template <int I>
__global__ void __launch_bounds__(kThreads) compact_kernel(const uint8_t* __restrict__ mask,
                                                           int32_t* __restrict__ out, size_t n,
                                                           const unsigned long long* __restrict__ true_total,
                                                           ScanWs* ws) {
    __shared__ unsigned long long s_scan[kThreads / 32 + 1];
    __shared__ unsigned s_tile;
    __shared__ unsigned long long s_look[kThreads / 32 + 2];
    if (threadIdx.x == 0) s_tile = atomicAdd(&ws->ticket, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const size_t base = static_cast<size_t>(tile) * (kThreads * I) + static_cast<size_t>(threadIdx.x) * I;
    const bool vec_in = (reinterpret_cast<uintptr_t>(mask) & 15) == 0;
    uint8_t b[I];
    load_mask<I>(mask, base, n, vec_in, b);
    unsigned cnt = 0;
#pragma unroll
    for (int k = 0; k < I; ++k) cnt += b[k] != 0;
    unsigned long long total;
    const unsigned long long excl = block_excl_scan<kThreads>(cnt, s_scan, &total);
    __syncthreads();
    const unsigned long long tile_prefix = block_lookback<kThreads>(ws->status, static_cast<int>(tile), total, s_look);
    // Partition the tile in shared memory (trues then falses, both ascending), then write the
    // two runs out coalesced: per-thread scattered stores left each warp instruction touching
    // 32 sectors.
    extern __shared__ int32_t s_out[];  // [kThreads * I], dynamic
    const size_t T = *true_total;
    const size_t tile_base = static_cast<size_t>(tile) * (kThreads * I);
    const int tile_n = static_cast<int>(n - tile_base < static_cast<size_t>((kThreads * I)) ? n - tile_base : (kThreads * I));
    const int ttot = static_cast<int>(total);
    int t_loc = static_cast<int>(excl);
    int f_loc = ttot + static_cast<int>(threadIdx.x) * I - static_cast<int>(excl);
#pragma unroll
    for (int k = 0; k < I; ++k) {
        const size_t i = base + k;
        if (i < n) s_out[b[k] ? t_loc++ : f_loc++] = static_cast<int32_t>(i);
    }
    __syncthreads();
    const size_t f_dst = T + (tile_base - tile_prefix) - static_cast<size_t>(ttot);
    for (int j = threadIdx.x; j < tile_n; j += kThreads)
        out[j < ttot ? tile_prefix + j : f_dst + j] = s_out[j];
}

// ---------------------------------------------------------------- match_first_equal
struct MatchWs {
    int vmin, vmax;
    unsigned hbits;  // table size = 1 << hbits
    unsigned pad;
};

__global__ void minmax_kernel(const int32_t* __restrict__ rb, size_t m, MatchWs* ws) {
    int lo = INT_MAX, hi = INT_MIN;
    for (size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
         j += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int v = rb[j];
        lo = min(lo, v);
        hi = max(hi, v);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, d));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, d));
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(&ws->vmin, lo);
        atomicMax(&ws->vmax, hi);
    }
}

__device__ __forceinline__ bool dense_mode(const MatchWs* ws) {
    const long long range = static_cast<long long>(ws->vmax) - ws->vmin + 1;
    return range <= (1LL << ws->hbits);
}

__device__ __forceinline__ unsigned hash32(uint32_t k, unsigned bits) {
    return static_cast<unsigned>(mix64(k) >> (64 - bits));
}

// vals[] starts at INT_MAX; keys[] (hash mode) start at 0 = empty, else (key << 1) | 1.
// Initialise only what the chosen mode reads (after minmax): dense -> vals[0, range);
// hash -> vals[0, H) and keys[0, H). Memsetting both full tables up front wrote 12*H bytes.
__global__ void match_init_kernel(const MatchWs* ws, int* __restrict__ vals,
                                  unsigned long long* __restrict__ keys) {
    const bool dense = dense_mode(ws);
    const size_t H = size_t{1} << ws->hbits;
    const size_t nv = dense ? static_cast<size_t>(static_cast<long long>(ws->vmax) - ws->vmin + 1) : H;
    const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
    const size_t t0 = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    // INT_MAX = "no row": above any row index, and what the lookup maps to -1
    const int4 fill = make_int4(INT_MAX, INT_MAX, INT_MAX, INT_MAX);
    for (size_t i = t0; i < nv / 4; i += stride) reinterpret_cast<int4*>(vals)[i] = fill;
    for (size_t i = (nv & ~size_t{3}) + t0; i < nv; i += stride) vals[i] = INT_MAX;
    if (!dense)
        for (size_t i = t0; i < H / 2; i += stride) reinterpret_cast<ulonglong2*>(keys)[i] = make_ulonglong2(0, 0);
}

__global__ void match_build_kernel(const int32_t* __restrict__ rb, size_t m, const MatchWs* ws,
                                   int* __restrict__ vals, unsigned long long* __restrict__ keys) {
    const bool dense = dense_mode(ws);
    const unsigned bits = ws->hbits;
    const unsigned mask = (1u << bits) - 1u;
    for (size_t j = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
         j += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int v = rb[j];
        // rank 0 means "not selected" and is never looked up (match_lookup_kernel): skipping it
        // removes the one hot word every unselected row would hammer
        if (v == 0) continue;
        if (dense) {
            int* slot = &vals[v - ws->vmin];
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
    }
}

__global__ void match_lookup_kernel(const int32_t* __restrict__ ra, size_t n, const MatchWs* ws,
                                    const int* __restrict__ vals,
                                    const unsigned long long* __restrict__ keys,
                                    int32_t* __restrict__ row_out) {
    const bool dense = dense_mode(ws);
    const unsigned bits = ws->hbits;
    const unsigned mask = (1u << bits) - 1u;
    const long long lo = ws->vmin, hi = ws->vmax;
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const int r = ra[i];
        int out = -1;
        if (r != 0 && r >= lo && r <= hi) {
            int j = INT_MAX;
            if (dense) {
                j = vals[r - lo];
            } else {
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
            if (j != INT_MAX) out = j;
        }
        row_out[i] = out;
    }
}

// ---------------------------------------------------------------- blends
template <class T>
__global__ void __launch_bounds__(kThreads) blend_kernel(const uint8_t* mask, const T* a, const T* b,
                                                         T* out, size_t n) {
    constexpr int kVecBytes = 16;
    constexpr int kPerVec = kVecBytes / sizeof(T);
    const bool vec = ((reinterpret_cast<uintptr_t>(mask) | reinterpret_cast<uintptr_t>(a) |
                       reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) & 15) == 0;
    for (size_t base = (static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x) * kItems; base < n;
         base += static_cast<size_t>(gridDim.x) * kThreads * kItems) {
        uint8_t m[kItems];
        load_mask16(mask, base, n, vec, m);
        if (vec && base + kItems <= n) {
            // All loads before any store: `out` may alias a or b (same index only), and
            // interleaving would let the compiler keep just two loads in flight.
            constexpr int kVecs = kItems / kPerVec;
            uint4 va[kVecs], vb[kVecs];
#pragma unroll
            for (int q = 0; q < kVecs; ++q) {
                va[q] = *reinterpret_cast<const uint4*>(a + base + q * kPerVec);
                vb[q] = *reinterpret_cast<const uint4*>(b + base + q * kPerVec);
            }
#pragma unroll
            for (int q = 0; q < kVecs; ++q) {
                T* ea = reinterpret_cast<T*>(&va[q]);
                const T* eb = reinterpret_cast<const T*>(&vb[q]);
#pragma unroll
                for (int k = 0; k < kPerVec; ++k)
                    if (!m[q * kPerVec + k]) ea[k] = eb[k];
                *reinterpret_cast<uint4*>(out + base + q * kPerVec) = va[q];
            }
        } else {
#pragma unroll
            for (int k = 0; k < kItems; ++k)
                if (base + k < n) out[base + k] = m[k] ? a[base + k] : b[base + k];
        }
    }
}

}  // namespace abmx_table

// ====================================================================== launchers
using namespace abmx_table;

namespace abmx_internal {

static int grid_for(size_t n, int per_block) {
    const size_t g = (n + per_block - 1) / per_block;
    const size_t cap = static_cast<size_t>(num_sms()) * 8;
    return static_cast<int>(g < cap ? (g > 0 ? g : 1) : cap);
}

cudaError_t launch_rank_scan(const uint8_t* d_mask, int32_t* d_ranks, size_t n, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const size_t tiles = (n + kScanTile - 1) / kScanTile;
    const size_t ws_bytes = sizeof(ScanWs) + tiles * sizeof(unsigned long long);
    void* ws = nullptr;
    cudaError_t e = abmx_internal::malloc_async(&ws, ws_bytes, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(ws, 0, ws_bytes, s);
    (void)cudaGetLastError();
    constexpr int smem = kThreads * (kScanItems + 1) * static_cast<int>(sizeof(int32_t));
    static const cudaError_t attr = cudaFuncSetAttribute(
        rank_scan_kernel<kScanItems>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr != cudaSuccess) { cudaFreeAsync(ws, s); return attr; }
    rank_scan_kernel<kScanItems><<<static_cast<unsigned>(tiles), kThreads, smem, s>>>(d_mask, d_ranks, n,
                                                                      static_cast<ScanWs*>(ws));
    count_launch();
    e = cudaGetLastError();
    cudaFreeAsync(ws, s);
    return e;
}

cudaError_t launch_count_true(const uint8_t* d_mask, size_t n, unsigned long long* d_out,
                              cudaStream_t s) {
    cudaMemsetAsync(d_out, 0, sizeof(unsigned long long), s);
    if (n == 0) return cudaGetLastError();
    (void)cudaGetLastError();
    count_true_kernel<<<grid_for(n, kThreads * kCountItems), kThreads, 0, s>>>(d_mask, n, d_out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_compact_indices(const uint8_t* d_mask, int32_t* d_out, size_t n,
                                   unsigned long long* d_count, cudaStream_t s) {
    if (n == 0) return cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s);
    cudaError_t e = launch_count_true(d_mask, n, d_count, s);
    if (e != cudaSuccess) return e;
    const size_t tiles = (n + kCompactTile - 1) / kCompactTile;
    const size_t ws_bytes = sizeof(ScanWs) + tiles * sizeof(unsigned long long);
    void* ws = nullptr;
    e = abmx_internal::malloc_async(&ws, ws_bytes, s);
    if (e != cudaSuccess) return e;
    cudaMemsetAsync(ws, 0, ws_bytes, s);
    (void)cudaGetLastError();
    constexpr int smem = kCompactTile * static_cast<int>(sizeof(int32_t));
    static const cudaError_t attr = cudaFuncSetAttribute(
        compact_kernel<kCompactItems>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (attr != cudaSuccess) { cudaFreeAsync(ws, s); return attr; }
    compact_kernel<kCompactItems><<<static_cast<unsigned>(tiles), kThreads, smem, s>>>(d_mask, d_out, n, d_count,
                                                                    static_cast<ScanWs*>(ws));
    count_launch();
    e = cudaGetLastError();
    cudaFreeAsync(ws, s);
    return e;
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
    const MatchWs init{INT_MAX, INT_MIN, bits, 0u};
    cudaMemcpyAsync(mws, &init, sizeof init, cudaMemcpyHostToDevice, s);
    const int gm = grid_for(m, 256), gn = grid_for(n, 256);
    (void)cudaGetLastError();
    minmax_kernel<<<gm, 256, 0, s>>>(d_rb, m, mws);
    match_init_kernel<<<num_sms() * 8, 256, 0, s>>>(mws, vals, keys);
    match_build_kernel<<<gm, 256, 0, s>>>(d_rb, m, mws, vals, keys);
    match_lookup_kernel<<<gn, 256, 0, s>>>(d_ra, n, mws, vals, keys, d_out);
    count_launch(4);
    e = cudaGetLastError();
    cudaFreeAsync(ws, s);
    return e;
}

template <class T>
cudaError_t launch_blend(const uint8_t* d_mask, const T* d_a, const T* d_b, T* d_out, size_t n,
                         cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    (void)cudaGetLastError();
    blend_kernel<T><<<grid_for(n, kTile), kThreads, 0, s>>>(d_mask, d_a, d_b, d_out, n);
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
