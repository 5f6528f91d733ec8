// finance.cu — the limit-order-book market (src/models/finance.cpp) on sm_100a for M markets at
// once, bit-exact with the reference.
//
// Books never read trader state (placement reads only the trader params and the book's last
// price) and holdings_k is written only by book k, so every (market, book) pair is independent:
// ONE CTA per book, the whole book resident in shared memory across the steps of a launch.
// Cash is the only value summed across books; every amount is qty x (a multiple of 2^-8) and the
// sums stay far below 2^45, so all additions are exact and their order cannot change a bit —
// per-book partial sums are folded into the traders with double atomics.
//
// A step of one book (finance.cpp:203-247):
//   place    traders in order: bernoulli(4i, p), side (4i+1), epsilon (4i+2), qty (4i+3) from
//            seed.split(8).split(t).split(book); valid rows rank-matched into the lowest free slots
//            (block scans of the row and free-slot masks), ids next_id + k, placed = t.
//   match    active orders sorted by (side, price desc for buys / asc for sells, placed, id) with
//            an in-CTA bitonic sort; cumulative quantities by block scan; the executed volume =
//            max over buys of min(buy cum, sell cum at the last sell priced <= the buy) (binary
//            search per buy); marginal orders, midpoint clearing price; fill of sorted order j =
//            min(qty_j, max(0, volume - cum_{j-1})) — the reference's sequential fill loop in
//            closed form; exhausted orders removed.
//   cancel   t - placed >= max_order_age.
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

namespace abmx_fin {

constexpr int kNTLarge = 256;  // CTA size for books whose order window exceeds kSmallWindow
#ifndef ABMX_FIN_SMALL_NT
#define ABMX_FIN_SMALL_NT 32
#endif
constexpr int kNTSmall = ABMX_FIN_SMALL_NT;  // one warp per book: C5 2.0 ms vs 2.4 (64), 3.2 (128)
constexpr int kSmallWindow = 512;
constexpr double kTick = 0x1p-7;  // finance.hpp:37
constexpr unsigned short kPad = 0xFFFF;
// Cash amounts are multiples of 2^-8 (quantity x a midpoint of 2^-7 ticks), so every partial
// sum below 2^45 is exact and the order of the (atomic) additions cannot change a bit. A sum
// reaching 2^44 leaves that envelope: flagged, reported by the host instead of a result that
// could differ from the reference's sequential sums.
constexpr double kCashExact = 0x1p44;

struct BookS {  // per-book scalars
    double last_price, clearing;
    long long next_id, dropped, volume;
    int num_active, pad;
};

struct FParams {
    int M, K, T, cap, sort_n;  // sort_n: power of two >= W
    int W;     // order window: every active order of every book lies in slots [0, W) (see launch)
    int* err;  // set if a book ever needed a slot >= W (cannot happen; checked on every readback)
    long long id_span;  // keyed: alive ids lie in [next_id - id_span, next_id + T*steps)
    double p_order, delta, init_price;
    long long qmax, max_age;
    long long t0, steps;
    int match_only;  // 1: one match_book pass, fills recorded (no placement, no cancel)
    const unsigned long long* seeds;  // [M]
    // books [M][K][cap]
    uint8_t* active;
    long long* ids;
    int* trader;
    uint8_t* side;
    double* price;
    int* qty;
    long long* placed;
    BookS* bs;           // [M][K]
    double* cash;        // [M][T]
    long long* holdings; // [M][K][T]
    double* metrics;     // [M][steps][K][6]
    // match_only outputs (book 0 of market 0)
    long long* f_trader;
    long long* f_side;
    long long* f_qty;
    double* f_amount;
    int* n_fills;
};

__device__ __forceinline__ double quantize(double raw) {  // finance.cpp:56-61
    double p = __dmul_rn(round(raw / kTick), kTick);
    if (p < kTick) p = kTick;
    return p;
}

struct Smem {
    uint8_t* act;
    long long* id;
    int* tr;
    uint8_t* sd;
    double* pr;
    int* q;
    long long* pl;
    unsigned short* list;  // sorted order (sort_n entries)
    unsigned short* list2; // ping-pong buffer of the sorted order
    unsigned short* nl;    // this step's new orders, trader order (T entries)
    unsigned short* nsr;   // ... sorted (T entries)
    long long* cum;        // cumulative qty along the sorted list (cap entries)
    // placement rows (T entries)
    int* rq;
    double* rp;
    uint8_t* rs;
    int* rt;
    unsigned long long* key;  // kKeyed: (side, price) priority packed in one word, per slot
    // kKeyed compact fields: id - idbase, placed and the cumulative quantities in 32 bits (side
    // and price live in `key`)
    int* id32;
    int* pl32;
    int* cum32;
    long long idbase;
    double* dcash;       // [T] cash delta of this book
    long long* dhold;    // [T] holdings delta of this book
};

// (side, price) priority of an order placed by the kernel (side 0/1, price a positive finite
// double): one unsigned compare orders buys first by price desc, then sells by price asc.
__device__ __forceinline__ unsigned long long prio_key(uint8_t side, double price) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(price));
    return side ? (1ULL << 63) | b : ~b & 0x7FFFFFFFFFFFFFFFULL;
}

// the price of a packed key (the inverse of prio_key)
__device__ __forceinline__ double key_price(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : (~k & 0x7FFFFFFFFFFFFFFFULL);
    return __longlong_as_double(static_cast<long long>(b));
}

// order fields in either layout
template <bool kK>
__device__ __forceinline__ int o_side(const Smem& S, int i) {
    if constexpr (kK) return static_cast<int>(S.key[i] >> 63);
    else return S.sd[i];
}
template <bool kK>
__device__ __forceinline__ double o_price(const Smem& S, int i) {
    if constexpr (kK) return key_price(S.key[i]);
    else return S.pr[i];
}
template <bool kK>
__device__ __forceinline__ long long o_id(const Smem& S, int i) {
    if constexpr (kK) return S.idbase + S.id32[i];
    else return S.id[i];
}
template <bool kK>
__device__ __forceinline__ long long o_placed(const Smem& S, int i) {
    if constexpr (kK) return S.pl32[i];
    else return S.pl[i];
}
template <bool kK>
__device__ __forceinline__ long long o_cum(const Smem& S, int j) {
    if constexpr (kK) return S.cum32[j];
    else return S.cum[j];
}
template <bool kK>
__device__ __forceinline__ void set_cum(const Smem& S, int j, long long v) {
    if constexpr (kK) S.cum32[j] = static_cast<int>(v);
    else S.cum[j] = v;
}
template <bool kK>
__device__ __forceinline__ void set_order(const Smem& S, int i, long long id, int tr, int side, double price,
                                          int q, long long placed) {
    S.act[i] = 1;
    S.tr[i] = tr;
    S.q[i] = q;
    if constexpr (kK) {
        S.id32[i] = static_cast<int>(id - S.idbase);
        S.pl32[i] = static_cast<int>(placed);
        S.key[i] = prio_key(static_cast<uint8_t>(side), price);
    } else {
        S.id[i] = id;
        S.sd[i] = static_cast<uint8_t>(side);
        S.pr[i] = price;
        S.pl[i] = placed;
    }
}

// sort order: buys before sells; buys by price desc, sells by price asc; then placed, id, slot.
// kKeyed: every order was placed by this kernel (launches with strictly increasing t), so
// (side, price) is the packed key, and ids -- unique, handed out in placement order -- order
// (placed, id) on their own.
template <bool kKeyed>
__device__ __forceinline__ bool before_live(const Smem& S, unsigned short a, unsigned short b);
template <bool kKeyed>
__device__ __forceinline__ bool before(const Smem& S, unsigned short a, unsigned short b) {
    if (b == kPad) return a != kPad;
    if (a == kPad) return false;
    return before_live<kKeyed>(S, a, b);
}
// before() for two live orders (no padding entries: the merge's ranks and binary searches)
template <bool kKeyed>
__device__ __forceinline__ bool before_live(const Smem& S, unsigned short a, unsigned short b) {
    if constexpr (kKeyed) {
        const unsigned long long ka = S.key[a], kb = S.key[b];
        return ka != kb ? ka < kb : S.id32[a] < S.id32[b];
    }
    if (S.sd[a] != S.sd[b]) return S.sd[a] < S.sd[b];
    if (S.pr[a] != S.pr[b]) return S.sd[a] == 0 ? S.pr[a] > S.pr[b] : S.pr[a] < S.pr[b];
    if (S.pl[a] != S.pl[b]) return S.pl[a] < S.pl[b];
    if (S.id[a] != S.id[b]) return S.id[a] < S.id[b];
    return a < b;
}

template <bool kK>
__device__ __forceinline__ void reset_slot(const Smem& S, int i) {  // agent_set.cpp:45-58
    S.act[i] = 0;
    S.tr[i] = 0;
    S.q[i] = 0;
    if constexpr (kK) {  // stored back as zeros (inactive)
        S.id32[i] = 0;
        S.pl32[i] = 0;
        S.key[i] = 0;
    } else {
        S.id[i] = 0;
        S.sd[i] = 0;
        S.pr[i] = 0.0;
        S.pl[i] = 0;
    }
}

template <int kNT, bool kKeyed>
__global__ void __launch_bounds__(kNT) k_fin(FParams P) {
    extern __shared__ unsigned char smraw[];
    __shared__ unsigned long long s_scan[kNT / 32 + 1];
    __shared__ long long s_red[kNT / 32];
    __shared__ int s_n, s_nb;
    __shared__ long long s_vol;
    const int m = blockIdx.x / P.K, k = blockIdx.x % P.K;
    const int W = P.W, T = P.T, N = P.sort_n, tid = threadIdx.x;
    // shared layout (8-byte fields first)
    Smem S{};
    const size_t bo = (static_cast<size_t>(m) * P.K + k) * P.cap;
    BookS B = P.bs[static_cast<size_t>(m) * P.K + k];
    unsigned char* p = smraw;
    if constexpr (kKeyed) {
        S.key = reinterpret_cast<unsigned long long*>(p);
        p += 8 * W;
    } else {
        S.id = reinterpret_cast<long long*>(p);
        p += 8 * W;
        S.pr = reinterpret_cast<double*>(p);
        p += 8 * W;
        S.pl = reinterpret_cast<long long*>(p);
        p += 8 * W;
        S.cum = reinterpret_cast<long long*>(p);
        p += 8 * W;
    }
    S.rp = reinterpret_cast<double*>(p);
    p += 8 * T;
    S.dcash = reinterpret_cast<double*>(p);
    p += 8 * T;
    S.dhold = reinterpret_cast<long long*>(p);
    p += 8 * T;
    if constexpr (kKeyed) {
        S.id32 = reinterpret_cast<int*>(p);
        p += 4 * W;
        S.pl32 = reinterpret_cast<int*>(p);
        p += 4 * W;
        S.cum32 = reinterpret_cast<int*>(p);
        p += 4 * W;
        S.idbase = B.next_id - P.id_span;
    }
    S.tr = reinterpret_cast<int*>(p);
    p += 4 * W;
    S.q = reinterpret_cast<int*>(p);
    p += 4 * W;
    S.rq = reinterpret_cast<int*>(p);
    p += 4 * T;
    S.rt = reinterpret_cast<int*>(p);
    p += 4 * T;
    S.list = reinterpret_cast<unsigned short*>(p);
    p += 2 * N;
    // the ping-pong order buffer is used only by the merge (before matching) and the compaction
    // (after it), never while the cumulative quantities are live: it aliases them (4*W or 8*W
    // bytes >= 2*sort_n bytes, since sort_n < 2W)
    S.list2 = kKeyed ? reinterpret_cast<unsigned short*>(S.cum32) : reinterpret_cast<unsigned short*>(S.cum);
    S.nl = reinterpret_cast<unsigned short*>(p);
    p += 2 * T;
    S.nsr = reinterpret_cast<unsigned short*>(p);
    p += 2 * T;
    S.act = p;
    p += W;
    if constexpr (!kKeyed) {
        S.sd = p;
        p += W;
    }
    S.rs = p;
    // load the book
    for (int i = tid; i < W; i += kNT) {
        const uint8_t a = P.active[bo + i];
        S.act[i] = a;
        S.tr[i] = P.trader[bo + i];
        S.q[i] = P.qty[bo + i];
        if constexpr (kKeyed) {  // windowed books: inactive slots hold zeros
            S.id32[i] = a ? static_cast<int>(P.ids[bo + i] - S.idbase) : 0;
            S.pl32[i] = static_cast<int>(P.placed[bo + i]);
            S.key[i] = a ? prio_key(P.side[bo + i], P.price[bo + i]) : 0ULL;
        } else {
            S.id[i] = P.ids[bo + i];
            S.sd[i] = P.side[bo + i];
            S.pr[i] = P.price[bo + i];
            S.pl[i] = P.placed[bo + i];
        }
    }
    for (int i = tid; i < T; i += kNT) {
        S.dcash[i] = 0.0;
        S.dhold[i] = 0;
    }
    // The priority order of resting orders never changes (price, placed and id are fixed), so
    // the sorted order list is built once per launch and then maintained: new orders are
    // merged in by rank + binary search, filled / cancelled orders compacted out.
    unsigned short* const L = S.list;
    unsigned short* const L2 = S.list2;
    int n = 0;
    {
        unsigned long long carry = 0;
        for (int i0 = 0; i0 < N; i0 += kNT) {
            const int i = i0 + tid;
            const bool a = i < W && S.act[i];
            unsigned tot;
            const unsigned ex = block_excl_count<kNT>(a ? 1u : 0u, s_scan, &tot);
            if (a) L[carry + ex] = static_cast<unsigned short>(i);
            carry += tot;
            __syncthreads();
        }
        n = static_cast<int>(carry);
        for (int i = n + tid; i < N; i += kNT) L[i] = kPad;
        int ns2 = 1;
        while (ns2 < n) ns2 <<= 1;
        __syncthreads();
        for (int size = 2; size <= ns2; size <<= 1)
            for (int stride = size >> 1; stride > 0; stride >>= 1) {
                for (int j = tid; j < ns2 / 2; j += kNT) {
                    const int lo = 2 * j - (j & (stride - 1));
                    const int hi = lo + stride;
                    const bool up = (lo & size) == 0;
                    const unsigned short a = L[lo], b = L[hi];
                    if (before<kKeyed>(S, b, a) == up) {
                        L[lo] = b;
                        L[hi] = a;
                    }
                }
                __syncthreads();
            }
    }
    const unsigned long long root = split(P.seeds[m], 8);  // FinancePlace
    const long long t_end = P.match_only ? P.t0 + 1 : P.t0 + P.steps;
    for (long long t = P.t0; t < t_end; ++t) {
        if (!P.match_only) {
            // ---------------- place_orders (finance.cpp:74-123)
            const unsigned long long key = split(split(root, static_cast<unsigned long long>(t)),
                                                 static_cast<unsigned long long>(k));
            unsigned long long carry = 0;
            for (int i0 = 0; i0 < T; i0 += kNT) {  // valid rows, compacted in trader order
                const int i = i0 + tid;
                bool v = false;
                int sd = 0, qt = 0;
                double pr = 0.0;
                if (i < T) {
                    const unsigned long long base = 4ULL * static_cast<unsigned long long>(i);
                    v = uniform_double(key, base) < P.p_order;
                    if (v) {
                        sd = static_cast<int>(uniform_span(key, base + 1, 2));
                        const double eps = __dadd_rn(-P.delta, __dmul_rn(__dmul_rn(2.0, P.delta), uniform_double(key, base + 2)));
                        qt = 1 + static_cast<int>(uniform_span(key, base + 3, static_cast<unsigned long long>(P.qmax)));
                        pr = quantize(__dmul_rn(B.last_price, __dadd_rn(1.0, eps)));
                    }
                }
                unsigned tot;
                const unsigned ex = block_excl_count<kNT>(v ? 1u : 0u, s_scan, &tot);
                if (v) {
                    const int r = static_cast<int>(carry + ex);
                    S.rt[r] = i;
                    S.rs[r] = static_cast<uint8_t>(sd);
                    S.rp[r] = pr;
                    S.rq[r] = qt;
                }
                carry += tot;
                __syncthreads();
            }
            const int q = static_cast<int>(carry);
            // k-th free slot <- k-th valid row (lifecycle.cpp:144-195)
            unsigned long long fcarry = 0;
            for (int i0 = 0; i0 < W && static_cast<long long>(fcarry) < q; i0 += kNT) {
                const int i = i0 + tid;
                const bool fr = i < W && !S.act[i];
                unsigned tot;
                const unsigned ex = block_excl_count<kNT>(fr ? 1u : 0u, s_scan, &tot);
                const long long r = static_cast<long long>(fcarry + ex);
                if (fr && r < q) {
                    set_order<kKeyed>(S, i, B.next_id + r, S.rt[r], S.rs[r], S.rp[r], S.rq[r], t);
                    S.nl[r] = static_cast<unsigned short>(i);
                }
                fcarry += tot;
                __syncthreads();
            }
            const int spawned = static_cast<long long>(fcarry) < q ? static_cast<int>(fcarry) : q;
            if (static_cast<long long>(fcarry) < q && W < P.cap && tid == 0) atomicOr(P.err, 1);
            B.next_id += spawned;
            B.dropped = q - spawned;
            if (spawned > 0) {
                // merge: rank the new orders among themselves, then every element's merged
                // position = its own index + the other list's elements before it
                for (int j = tid; j < spawned; j += kNT) {
                    const unsigned short x = S.nl[j];
                    int rk = 0;
                    for (int y = 0; y < spawned; ++y) rk += before_live<kKeyed>(S, S.nl[y], x);
                    S.nsr[rk] = x;
                }
                __syncthreads();
                for (int e = tid; e < n; e += kNT) {
                    const unsigned short a = L[e];
                    int lo = 0, hi = spawned;  // new orders before a
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (before_live<kKeyed>(S, S.nsr[mid], a))
                            lo = mid + 1;
                        else
                            hi = mid;
                    }
                    L2[e + lo] = a;
                }
                for (int j = tid; j < spawned; j += kNT) {
                    const unsigned short b = S.nsr[j];
                    int lo = 0, hi = n;  // resting orders before b
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (before_live<kKeyed>(S, L[mid], b))
                            lo = mid + 1;
                        else
                            hi = mid;
                    }
                    L2[j + lo] = b;
                }
                __syncthreads();
                n += spawned;
                for (int e = tid; e < n; e += kNT) L[e] = L2[e];  // back out of the cum alias
                __syncthreads();
            }
        }
        // ---------------- match_book (finance.cpp:125-190) on the sorted order list
        {
            // cumulative quantities along the sorted list; buys precede sells
            unsigned long long qcarry = 0;
            for (int i0 = 0; i0 < n; i0 += kNT) {
                const int i = i0 + tid;
                const unsigned short s = i < n ? L[i] : kPad;
                unsigned long long tot;
                const unsigned long long ex =
                    block_excl_scan<kNT>(s != kPad ? static_cast<unsigned long long>(S.q[s]) : 0ULL, s_scan, &tot);
                if (s != kPad) set_cum<kKeyed>(S, i, static_cast<long long>(qcarry + ex) + S.q[s]);
                qcarry += tot;
                __syncthreads();
            }
            int nbuy;
            {
                int lo = 0, hi = n;  // first sell in the list
                while (lo < hi) {
                    const int mid = (lo + hi) >> 1;
                    if (o_side<kKeyed>(S, L[mid]) == 0)
                        lo = mid + 1;
                    else
                        hi = mid;
                }
                nbuy = lo;
            }
            const int nsell = n - nbuy;
            const long long btot = nbuy > 0 ? o_cum<kKeyed>(S, nbuy - 1) : 0;  // sells' cum = cum - btot
            // executed volume: max over buys of min(buy cum, sell cum at upper_bound(buy price))
            long long vmax = 0;
            if (nbuy > 0 && nsell > 0)
                for (int i = tid; i < nbuy; i += kNT) {
                    int lo = 0, hi = nsell;  // first sell with price > bp
                    if constexpr (kKeyed) {  // sells' keys are 2^63 | bits(price): compare keys
                        const unsigned long long kb = (1ULL << 63) | (~S.key[L[i]] & 0x7FFFFFFFFFFFFFFFULL);
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (kb < S.key[L[nbuy + mid]])
                                hi = mid;
                            else
                                lo = mid + 1;
                        }
                    } else {
                        const double bp = S.pr[L[i]];
                        while (lo < hi) {
                            const int mid = (lo + hi) >> 1;
                            if (bp < S.pr[L[nbuy + mid]])
                                hi = mid;
                            else
                                lo = mid + 1;
                        }
                    }
                    if (lo == 0) continue;
                    const long long bc = o_cum<kKeyed>(S, i), sc = o_cum<kKeyed>(S, nbuy + lo - 1) - btot;
                    const long long v = bc < sc ? bc : sc;
                    if (v > vmax) vmax = v;
                }
            for (int d = 16; d > 0; d >>= 1) {
                const long long o = __shfl_xor_sync(0xffffffffu, vmax, d);
                vmax = o > vmax ? o : vmax;
            }
            if ((tid & 31) == 0) s_red[tid >> 5] = vmax;
            __syncthreads();
            long long volume = 0;
            for (int w = 0; w < kNT / 32; ++w) volume = s_red[w] > volume ? s_red[w] : volume;
            B.volume = 0;
            if (volume > 0) {
                // marginal orders: first cum >= volume on each side
                int mb, ms;
                {
                    int lo = 0, hi = nbuy - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (o_cum<kKeyed>(S, mid) >= volume)
                            hi = mid;
                        else
                            lo = mid + 1;
                    }
                    mb = lo;
                    lo = 0;
                    hi = nsell - 1;
                    while (lo < hi) {
                        const int mid = (lo + hi) >> 1;
                        if (o_cum<kKeyed>(S, nbuy + mid) - btot >= volume)
                            hi = mid;
                        else
                            lo = mid + 1;
                    }
                    ms = lo;
                }
                const double clearing = __dadd_rn(o_price<kKeyed>(S, L[mb]), o_price<kKeyed>(S, L[nbuy + ms])) / 2.0;
                __syncthreads();  // every thread has read the sorted prices before fills reset slots
                // fills: sorted order j gets min(qty_j, volume - cum_{j-1}) while positive
                for (int j = tid; j < n; j += kNT) {
                    const unsigned short s = L[j];
                    const bool buy = j < nbuy;
                    const long long before_j =
                        buy ? (j > 0 ? o_cum<kKeyed>(S, j - 1) : 0) : (j > nbuy ? o_cum<kKeyed>(S, j - 1) - btot : 0);
                    const long long rem = volume - before_j;
                    if (rem <= 0) continue;
                    const long long f = S.q[s] < rem ? S.q[s] : rem;
                    const double amount = __dmul_rn(static_cast<double>(f), clearing);
                    const int tr = S.tr[s];
                    if (P.match_only) {
                        const int fi = buy ? j : (mb + 1) + (j - nbuy);
                        P.f_trader[fi] = tr;
                        P.f_side[fi] = buy ? 0 : 1;
                        P.f_qty[fi] = f;
                        P.f_amount[fi] = amount;
                    } else if (tr >= 0 && tr < T) {
                        const double dv = buy ? -amount : amount;
                        if (fabs(atomicAdd(&S.dcash[tr], dv) + dv) >= kCashExact) atomicOr(P.err, 2);
                        atomicAdd(reinterpret_cast<unsigned long long*>(&S.dhold[tr]),
                                  static_cast<unsigned long long>(buy ? f : -f));
                    }
                    S.q[s] -= static_cast<int>(f);
                    if (S.q[s] == 0) reset_slot<kKeyed>(S, s);  // exhausted: remove_agents
                }
                if (P.match_only && tid == 0) *P.n_fills = (mb + 1) + (ms + 1);
                B.last_price = clearing;
                B.clearing = clearing;
                B.volume = volume;
            } else if (P.match_only && tid == 0) {
                *P.n_fills = 0;
            }
            __syncthreads();
        }
        if (P.match_only) break;
        // ---------------- cancel at the age limit (finance.cpp:236-245) and compact the order
        // list: one scan of packed (alive, alive buy) counters over the sorted list
        {
            unsigned long long carry = 0;
            for (int i0 = 0; i0 < n; i0 += kNT) {
                const int i = i0 + tid;
                bool alive = false, buy = false;
                unsigned short s = kPad;
                if (i < n) {
                    s = L[i];
                    if (S.act[s]) {
                        if (t - o_placed<kKeyed>(S, s) >= P.max_age)
                            reset_slot<kKeyed>(S, s);
                        else
                            alive = true;
                    }
                    buy = alive && o_side<kKeyed>(S, s) == 0;
                }
                unsigned tot;  // packed (alive << 16 | alive buy): at most kNT per field
                const unsigned ex = block_excl_count<kNT>((alive ? (1u << 16) : 0u) | (buy ? 1u : 0u), s_scan, &tot);
                if (alive) L2[(carry >> 32) + (ex >> 16)] = s;
                carry += (static_cast<unsigned long long>(tot >> 16) << 32) | (tot & 0xFFFFu);
                __syncthreads();
            }
            n = static_cast<int>(carry >> 32);
            for (int e = tid; e < n; e += kNT) L[e] = L2[e];  // back out of the cum alias
            __syncthreads();
            const long long nb = static_cast<long long>(carry & 0xFFFFFFFFULL);
            B.num_active = n;
            if (tid == 0) {  // collect_metrics (finance.cpp:262-276)
                double* row = P.metrics + ((static_cast<size_t>(m) * P.steps + (t - P.t0)) * P.K + k) * 6;
                row[0] = static_cast<double>(k);
                row[1] = B.last_price;
                row[2] = static_cast<double>(nb);
                row[3] = static_cast<double>(n - nb);
                row[4] = static_cast<double>(B.volume);
                row[5] = static_cast<double>(B.dropped);
            }
        }
    }
    // store the book, fold this book's settlement into the traders
    for (int i = tid; i < W; i += kNT) {
        const uint8_t a = S.act[i];
        P.active[bo + i] = a;
        P.trader[bo + i] = S.tr[i];
        P.qty[bo + i] = S.q[i];
        if constexpr (kKeyed) {  // inactive slots are all zeros (reset_slot)
            P.ids[bo + i] = a ? o_id<kKeyed>(S, i) : 0;
            P.side[bo + i] = a ? static_cast<uint8_t>(o_side<kKeyed>(S, i)) : 0;
            P.price[bo + i] = a ? o_price<kKeyed>(S, i) : 0.0;
            P.placed[bo + i] = a ? o_placed<kKeyed>(S, i) : 0;
        } else {
            P.ids[bo + i] = S.id[i];
            P.side[bo + i] = S.sd[i];
            P.price[bo + i] = S.pr[i];
            P.placed[bo + i] = S.pl[i];
        }
    }
    if (!P.match_only)
        for (int i = tid; i < T; i += kNT) {
            if (S.dcash[i] != 0.0 &&
                fabs(atomicAdd(&P.cash[static_cast<size_t>(m) * T + i], S.dcash[i]) + S.dcash[i]) >= kCashExact)
                atomicOr(P.err, 2);
            P.holdings[(static_cast<size_t>(m) * P.K + k) * T + i] += S.dhold[i];
        }
    if (tid == 0) {
        if (P.match_only) B.num_active = 0;  // recomputed on the host from the mask
        P.bs[static_cast<size_t>(m) * P.K + k] = B;
    }
}

__global__ void k_fin_init(FParams P, double last_price) {
    const size_t nb = static_cast<size_t>(P.M) * P.K;
    const size_t n0 = nb * P.cap, n1 = nb * P.T;
    const size_t n = n0 > n1 ? n0 : n1;  // covers the orders, the books and every trader array
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        if (i < n0) {
            P.active[i] = 0;
            P.ids[i] = 0;
            P.trader[i] = 0;
            P.side[i] = 0;
            P.price[i] = 0.0;
            P.qty[i] = 0;
            P.placed[i] = 0;
        }
        if (i < nb) P.bs[i] = BookS{last_price, 0.0, 0, 0, 0, 0, 0};
        if (i < static_cast<size_t>(P.M) * P.T) P.cash[i] = 0.0;
        if (i < n1) P.holdings[i] = 0;
    }
}

}  // namespace abmx_fin

// ====================================================================== host side
using namespace abmx_fin;

#define CKF(x)                                                                        \
    do {                                                                              \
        cudaError_t e_ = (x);                                                         \
        if (e_ != cudaSuccess) {                                                      \
            abmx_internal::set_error(std::string(#x) + ": " + cudaGetErrorString(e_)); \
            return ABMX_E_CUDA;                                                       \
        }                                                                             \
    } while (0)

namespace {

double quantize_host(double raw) {
    double p = std::round(raw / kTick) * kTick;
    if (p < kTick) p = kTick;
    return p;
}

int check_cfg(const abmx_finance_config& c) {
    if (c.books < 1 || c.traders < 0 || c.book_capacity < 1) {
        abmx_internal::set_error("finance: books/book_capacity must be >= 1, traders >= 0");  // config.cpp:210-211
        return ABMX_E_DOMAIN;
    }
    if (c.p_order < 0.0 || c.p_order > 1.0) {
        abmx_internal::set_error("finance: p_order must lie in [0, 1]");
        return ABMX_E_DOMAIN;
    }
    if (c.qmax < 1) {
        abmx_internal::set_error("finance: qmax must be >= 1");  // uniform_int(1, qmax+1) needs qmax >= 1
        return ABMX_E_DOMAIN;
    }
    if (c.qmax > INT32_MAX) {
        abmx_internal::set_error("finance: qmax above 2^31-1 is not supported (32-bit order quantities)");
        return ABMX_E_CAPACITY;
    }
    if (c.book_capacity > 4096 || c.traders > 4096) {
        abmx_internal::set_error("finance: book_capacity and traders above 4096 are not supported "
                                 "(one shared-memory-resident CTA per book)");
        return ABMX_E_CAPACITY;
    }
    return ABMX_OK;
}

size_t fin_smem(const abmx_finance_config& c, int window, int sort_n, bool keyed) {
    const size_t cap = static_cast<size_t>(window), T = static_cast<size_t>(c.traders);
    if (keyed)  // key 8 + id32 / placed32 / cum32 / trader / qty 4 each + active 1 per slot
        return 29 * cap + 37 * T + 2 * static_cast<size_t>(sort_n) + 64;
    return 32 * cap + 24 * T + 8 * cap + 8 * T + 2 * static_cast<size_t>(sort_n) + 4 * T + 2 * cap + T + 64;
}

}  // namespace

struct abmx_finance {
    abmx_finance_config cfg{};
    FParams P{};
    cudaStream_t stream = nullptr;
    std::vector<void*> allocs;
    size_t smem = 0;
    double* d_metrics = nullptr;
    size_t metrics_bytes = 0;
    long long last_steps = 0;
    int M = 0;
    // The order window. Placement takes the lowest free slots, so no order ever sits at a slot
    // >= the number of orders alive at once. Orders alive after the cancel of step t were placed
    // at steps t-max_age+1 .. t (at most traders each, when launches come with strictly
    // increasing t), so a book never holds more than traders x (max_age + 1) orders and its
    // slots >= that bound stay empty. Such books keep only the window in shared memory (C5: 210
    // of 1000 slots, ~9 KB instead of ~45 KB: four times the resident books per SM). An
    // imported book or a repeated / decreasing t drops back to the whole capacity for good.
    int window = 0;
    bool windowed = true;
    long long last_t = LLONG_MIN;
    int* d_err = nullptr;
    bool keyed_ok = false;  // the windowed layout plus the priority keys fits in shared memory
    // the keyed layout keeps ids (relative to next_id - id_span), placed and the cumulative
    // quantities in 32 bits: a launch qualifies when all three ranges fit
    bool compact_fits(long long t0, long long steps) const {
        const long long age = cfg.max_order_age > 0 ? cfg.max_order_age : 0;
        return P.id_span + P.T * steps <= INT32_MAX && t0 - age - 1 >= INT32_MIN && t0 + steps <= INT32_MAX &&
               cfg.qmax <= INT32_MAX / (window > 0 ? window : 1);
    }
    static int pow2_at_least(int n) {
        int q = 1;
        while (q < n) q <<= 1;
        return q;
    }
    void set_window(bool use, bool keyed) {
        P.W = use ? window : P.cap;
        P.sort_n = pow2_at_least(P.W);
        smem = fin_smem(cfg, P.W, P.sort_n, keyed);
#ifdef ABMX_FIN_SMEM_PAD  // occupancy experiments only (tools/fin_nt_sweep.sh)
        smem += ABMX_FIN_SMEM_PAD;
#endif
    }
    int check_err() {  // after a stream sync
        int e = 0;
        CKF(cudaMemcpy(&e, d_err, 4, cudaMemcpyDeviceToHost));
        if (e & 1) {
            abmx_internal::set_error("finance: an order outside the order window (internal invariant broken)");
            return ABMX_E_CUDA;
        }
        if (e & 2) {
            abmx_internal::set_error("finance: a cash sum reached 2^44, outside the exact-summation envelope "
                                     "(results could differ from the reference's sequential sums)");
            return ABMX_E_DOMAIN;
        }
        return ABMX_OK;
    }

    ~abmx_finance() {
        for (void* p : allocs) cudaFree(p);
        if (d_metrics) cudaFree(d_metrics);
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
    int create(const abmx_finance_config& c, const uint64_t* seeds, int markets) {
        int rc = check_cfg(c);
        if (rc) return rc;
        if (markets < 1) {
            abmx_internal::set_error("markets must be >= 1");
            return ABMX_E_DOMAIN;
        }
        cfg = c;
        M = markets;
        CKF(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
        memset(&P, 0, sizeof P);
        P.M = M;
        P.K = static_cast<int>(c.books);
        P.T = static_cast<int>(c.traders);
        P.cap = static_cast<int>(c.book_capacity);
        {
            const long long age = c.max_order_age > 0 ? c.max_order_age : 0;
            const long long bound = age < P.cap ? c.traders * (age + 1) : P.cap;  // no overflow: T, cap <= 4096
            window = static_cast<int>(bound < P.cap ? (bound > 1 ? bound : 1) : P.cap);
            if (window > P.cap) window = P.cap;
            P.id_span = c.traders * (age + 1);  // ids handed out while an order stays alive
        }
        P.p_order = c.p_order;
        P.delta = c.delta;
        P.init_price = c.init_price;
        P.qmax = c.qmax;
        P.max_age = c.max_order_age;
        const size_t nb = static_cast<size_t>(M) * P.K, n = nb * P.cap;
#define ALF(ptr, bytes)                                                 \
    if ((rc = alloc(reinterpret_cast<void**>(&(ptr)), (bytes))) != 0) \
        return rc;
        unsigned long long* sd = nullptr;
        ALF(sd, static_cast<size_t>(M) * 8);
        ALF(P.active, n);
        ALF(P.ids, n * 8);
        ALF(P.trader, n * 4);
        ALF(P.side, n);
        ALF(P.price, n * 8);
        ALF(P.qty, n * 4);
        ALF(P.placed, n * 8);
        ALF(P.bs, nb * sizeof(BookS));
        ALF(P.cash, static_cast<size_t>(M) * P.T * 8);
        ALF(P.holdings, nb * P.T * 8);
        ALF(P.f_trader, static_cast<size_t>(P.cap) * 8 + 8);
        ALF(P.f_side, static_cast<size_t>(P.cap) * 8 + 8);
        ALF(P.f_qty, static_cast<size_t>(P.cap) * 8 + 8);
        ALF(P.f_amount, static_cast<size_t>(P.cap) * 8 + 8);
        ALF(P.n_fills, 8);
        ALF(d_err, 8);
#undef ALF
        P.err = d_err;
        CKF(cudaMemset(d_err, 0, 8));
        P.seeds = sd;
        CKF(cudaMemcpy(sd, seeds, static_cast<size_t>(M) * 8, cudaMemcpyHostToDevice));
        set_window(false, false);  // the whole capacity must fit: the window can be dropped at any time
        if (smem > 226 * 1024) {  // sm_100: 227 KB of dynamic shared memory per CTA (minus static)
            abmx_internal::set_error("finance: book_capacity / traders too large for one shared-memory book");
            return ABMX_E_CAPACITY;
        }
        {
            const void* fns[4] = {reinterpret_cast<const void*>(k_fin<kNTLarge, false>),
                                  reinterpret_cast<const void*>(k_fin<kNTSmall, false>),
                                  reinterpret_cast<const void*>(k_fin<kNTLarge, true>),
                                  reinterpret_cast<const void*>(k_fin<kNTSmall, true>)};
            const size_t ks = fin_smem(cfg, window, pow2_at_least(window), true);
            // prices stay positive and never NaN (so their bit patterns order them) when the
            // placement factor 1 + eps stays positive and the initial price is a number
            keyed_ok = ks <= 226 * 1024 && c.delta < 1.0 && !std::isnan(c.init_price);
            const int lim = static_cast<int>(keyed_ok && ks > smem ? ks : smem);
            for (const void* f : fns)
                CKF(abmx_internal::raise_dyn_smem(f, static_cast<size_t>(lim)));
        }
        (void)cudaGetLastError();
        k_fin_init<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(P, quantize_host(c.init_price));
        abmx_internal::count_launch();
        CKF(cudaGetLastError());
        CKF(cudaStreamSynchronize(stream));
        return ABMX_OK;
    }
    int reserve(long long steps) {  // the metrics rows of a `steps` launch
        const size_t mb = static_cast<size_t>(M) * static_cast<size_t>(steps > 0 ? steps : 1) * P.K * 6 * 8;
        if (mb > metrics_bytes) {
            CKF(cudaStreamSynchronize(stream));
            if (d_metrics) cudaFree(d_metrics);
            d_metrics = nullptr;
            metrics_bytes = 0;
            CKF(cudaMalloc(&d_metrics, mb));
            metrics_bytes = mb;
        }
        return ABMX_OK;
    }
    int launch(long long t0, long long steps, int match_only) {
        if (const int rc = reserve(steps)) return rc;
        P.metrics = d_metrics;
        P.t0 = t0;
        P.steps = steps;
        P.match_only = match_only;
        if (!match_only) {
            if (t0 <= last_t) windowed = false;
            last_t = t0 + steps - 1;
        }
        const bool keyed = windowed && !match_only && keyed_ok && compact_fits(t0, steps);
        set_window(windowed && !match_only, keyed);
        (void)cudaGetLastError();
        const unsigned grid = match_only ? 1u : static_cast<unsigned>(M * P.K);
        if (P.W <= kSmallWindow) {
            if (keyed)
                k_fin<kNTSmall, true><<<grid, kNTSmall, smem, stream>>>(P);
            else
                k_fin<kNTSmall, false><<<grid, kNTSmall, smem, stream>>>(P);
        } else if (keyed) {
            k_fin<kNTLarge, true><<<grid, kNTLarge, smem, stream>>>(P);
        } else {
            k_fin<kNTLarge, false><<<grid, kNTLarge, smem, stream>>>(P);
        }
        abmx_internal::count_launch();
        CKF(cudaGetLastError());
        last_steps = steps;
        return ABMX_OK;
    }
};

extern "C" {

int abmx_finance_create(const abmx_finance_config* cfg, const uint64_t* seeds, int32_t markets,
                        abmx_finance** out) {
    if (!cfg || !seeds || !out) {
        abmx_internal::set_error("null argument");
        return ABMX_E_ARG;
    }
    auto* h = new abmx_finance();
    const int rc = h->create(*cfg, seeds, markets);
    if (rc) {
        delete h;
        *out = nullptr;
        return rc;
    }
    *out = h;
    return ABMX_OK;
}
int abmx_finance_destroy(abmx_finance* h) {
    delete h;
    return ABMX_OK;
}
int abmx_finance_run(abmx_finance* h, int64_t t0, int64_t steps, double* rows) {
    if (!h) return ABMX_E_ARG;
    if (steps <= 0) return ABMX_OK;
    int rc = h->launch(t0, steps, 0);
    if (rc) return rc;
    if (rows) {
        CKF(cudaMemcpyAsync(rows, h->d_metrics, static_cast<size_t>(h->M) * steps * h->P.K * 48, cudaMemcpyDeviceToHost,
                            h->stream));
        CKF(cudaStreamSynchronize(h->stream));
        return h->check_err();
    }
    return ABMX_OK;
}
int abmx_finance_step(abmx_finance* h, int64_t t) { return abmx_finance_run(h, t, 1, nullptr); }
int abmx_finance_metrics(abmx_finance* h, double* rows) {
    if (!h) return ABMX_E_ARG;
    const size_t per = static_cast<size_t>(h->P.K) * 6;
    if (h->last_steps <= 0) {
        for (int m = 0; m < h->M; ++m)
            for (int k = 0; k < h->P.K; ++k) {
                double* r = rows + (static_cast<size_t>(m) * h->P.K + k) * 6;
                r[0] = k;
                r[1] = quantize_host(h->cfg.init_price);
                r[2] = r[3] = r[4] = r[5] = 0.0;
            }
        return ABMX_OK;
    }
    for (int m = 0; m < h->M; ++m)
        CKF(cudaMemcpyAsync(rows + static_cast<size_t>(m) * per,
                            h->d_metrics + (static_cast<size_t>(m) * h->last_steps + h->last_steps - 1) * per,
                            per * 8, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaStreamSynchronize(h->stream));
    return h->check_err();
}
int abmx_finance_export_book(abmx_finance* h, int32_t market, int32_t book, uint8_t* active, int64_t* ids,
                             int64_t* trader, int64_t* side, double* price, int64_t* qty, int64_t* placed,
                             double* scalars) {
    if (!h) return ABMX_E_ARG;
    if (market < 0 || market >= h->M || book < 0 || book >= h->P.K) {
        abmx_internal::set_error("market / book index out of range");
        return ABMX_E_DOMAIN;
    }
    const size_t cap = static_cast<size_t>(h->P.cap);
    const size_t bo = (static_cast<size_t>(market) * h->P.K + book) * cap;
    std::vector<int> tr(cap), q(cap);
    std::vector<uint8_t> sd(cap);
    BookS B;
    CKF(cudaMemcpyAsync(active, h->P.active + bo, cap, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(ids, h->P.ids + bo, cap * 8, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(tr.data(), h->P.trader + bo, cap * 4, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(sd.data(), h->P.side + bo, cap, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(price, h->P.price + bo, cap * 8, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(q.data(), h->P.qty + bo, cap * 4, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(placed, h->P.placed + bo, cap * 8, cudaMemcpyDeviceToHost, h->stream));
    CKF(cudaMemcpyAsync(&B, h->P.bs + static_cast<size_t>(market) * h->P.K + book, sizeof B, cudaMemcpyDeviceToHost,
                        h->stream));
    CKF(cudaStreamSynchronize(h->stream));
    if (const int rc = h->check_err()) return rc;
    int na = 0;
    for (size_t i = 0; i < cap; ++i) {
        trader[i] = tr[i];
        side[i] = sd[i];
        qty[i] = q[i];
        na += active[i] ? 1 : 0;
    }
    if (scalars) {  // last_price, dropped, volume, clearing, next_id, num_active
        scalars[0] = B.last_price;
        scalars[1] = static_cast<double>(B.dropped);
        scalars[2] = static_cast<double>(B.volume);
        scalars[3] = B.clearing;
        scalars[4] = static_cast<double>(B.next_id);
        scalars[5] = na;
    }
    return ABMX_OK;
}
int abmx_finance_import_book(abmx_finance* h, int32_t market, int32_t book, const uint8_t* active, const int64_t* ids,
                             const int64_t* trader, const int64_t* side, const double* price, const int64_t* qty,
                             const int64_t* placed, int64_t next_id, double last_price) {
    if (!h) return ABMX_E_ARG;
    if (market < 0 || market >= h->M || book < 0 || book >= h->P.K) {
        abmx_internal::set_error("market / book index out of range");
        return ABMX_E_DOMAIN;
    }
    const size_t cap = static_cast<size_t>(h->P.cap);
    const size_t bo = (static_cast<size_t>(market) * h->P.K + book) * cap;
    std::vector<int> tr(cap), q(cap);
    std::vector<uint8_t> sd(cap), act(cap);
    int na = 0;
    for (size_t i = 0; i < cap; ++i) {
        act[i] = active[i] ? 1 : 0;
        na += act[i];
        if (trader[i] < INT32_MIN || trader[i] > INT32_MAX || qty[i] < INT32_MIN || qty[i] > INT32_MAX ||
            side[i] < 0 || side[i] > 255) {
            abmx_internal::set_error("order field outside the device layout");
            return ABMX_E_DOMAIN;
        }
        tr[i] = static_cast<int>(trader[i]);
        q[i] = static_cast<int>(qty[i]);
        sd[i] = static_cast<uint8_t>(side[i]);
    }
    BookS B{last_price, 0.0, next_id, 0, 0, na, 0};
    h->windowed = false;
    CKF(cudaStreamSynchronize(h->stream));
    CKF(cudaMemcpy(h->P.active + bo, act.data(), cap, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.ids + bo, ids, cap * 8, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.trader + bo, tr.data(), cap * 4, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.side + bo, sd.data(), cap, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.price + bo, price, cap * 8, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.qty + bo, q.data(), cap * 4, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.placed + bo, placed, cap * 8, cudaMemcpyHostToDevice));
    CKF(cudaMemcpy(h->P.bs + static_cast<size_t>(market) * h->P.K + book, &B, sizeof B, cudaMemcpyHostToDevice));
    return ABMX_OK;
}
int abmx_finance_export_traders(abmx_finance* h, int32_t market, double* cash, int64_t* holdings) {
    if (!h) return ABMX_E_ARG;
    if (market < 0 || market >= h->M) {
        abmx_internal::set_error("market index out of range");
        return ABMX_E_DOMAIN;
    }
    const size_t T = static_cast<size_t>(h->P.T), K = static_cast<size_t>(h->P.K);
    if (T) {
        CKF(cudaMemcpyAsync(cash, h->P.cash + static_cast<size_t>(market) * T, T * 8, cudaMemcpyDeviceToHost, h->stream));
        CKF(cudaMemcpyAsync(holdings, h->P.holdings + static_cast<size_t>(market) * K * T, K * T * 8,
                            cudaMemcpyDeviceToHost, h->stream));
    }
    CKF(cudaStreamSynchronize(h->stream));
    return ABMX_OK;
}
// match_book (finance.cpp:125-190) on one host book: arrays are updated in place, fills written
// in the reference order (buys by priority, then sells); returns the number of fills or < 0.
int32_t abmx_finance_match(int32_t capacity, double last_price, uint8_t* active, int64_t* ids, int64_t* trader,
                           int64_t* side, double* price, int64_t* qty, int64_t* placed, int64_t* f_trader,
                           int64_t* f_side, int64_t* f_qty, double* f_amount, double* scalars) {
    abmx_finance_config c{1, 0, capacity, 0.0, 0.0, 1, 1, last_price};
    uint64_t seed = 0;
    abmx_finance* h = nullptr;
    int rc = abmx_finance_create(&c, &seed, 1, &h);
    if (rc) return -rc;
    rc = abmx_finance_import_book(h, 0, 0, active, ids, trader, side, price, qty, placed, 0, last_price);
    if (!rc) rc = h->launch(0, 1, 1);
    int nf = 0;
    if (!rc) {
        // the engine stream is non-blocking: order the host reads after the match kernel
        cudaError_t e = cudaStreamSynchronize(h->stream);
        if (e == cudaSuccess) e = cudaMemcpy(&nf, h->P.n_fills, 4, cudaMemcpyDeviceToHost);
        if (e == cudaSuccess && nf > 0) {
            cudaMemcpy(f_trader, h->P.f_trader, static_cast<size_t>(nf) * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(f_side, h->P.f_side, static_cast<size_t>(nf) * 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(f_qty, h->P.f_qty, static_cast<size_t>(nf) * 8, cudaMemcpyDeviceToHost);
            e = cudaMemcpy(f_amount, h->P.f_amount, static_cast<size_t>(nf) * 8, cudaMemcpyDeviceToHost);
        }
        if (e != cudaSuccess) {
            abmx_internal::set_error(std::string("finance match: ") + cudaGetErrorString(e));
            rc = ABMX_E_CUDA;
        }
    }
    if (!rc) rc = abmx_finance_export_book(h, 0, 0, active, ids, trader, side, price, qty, placed, scalars);
    abmx_finance_destroy(h);
    return rc ? -rc : nf;
}
double abmx_finance_quantize_price(double raw) { return quantize_host(raw); }
int abmx_finance_run_batch(const abmx_finance_config* cfg, uint64_t master, int32_t replica_begin, int32_t count,
                           int64_t steps, double* rows, double* kernel_ms) {
    if (!cfg || count < 0) {
        abmx_internal::set_error("bad run_batch arguments");
        return ABMX_E_ARG;
    }
    int rc = check_cfg(*cfg);
    if (rc) return rc;
    if (count == 0 || steps <= 0) return ABMX_OK;
    std::vector<uint64_t> seeds(static_cast<size_t>(count));
    const unsigned long long base = abmx_dev::split(master, 2);  // batch.cpp:12-19
    for (int32_t q = 0; q < count; ++q)
        seeds[static_cast<size_t>(q)] = abmx_dev::split(base, static_cast<unsigned long long>(replica_begin + q));
    abmx_finance* h = nullptr;
    rc = abmx_finance_create(cfg, seeds.data(), count, &h);
    if (rc) return rc;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    rc = h->reserve(steps);  // allocate outside the timed region
    cudaEventRecord(a, h->stream);
    if (!rc) rc = h->launch(1, steps, 0);
    cudaEventRecord(b, h->stream);
    if (!rc && rows) {
        cudaError_t e = cudaMemcpyAsync(rows, h->d_metrics, static_cast<size_t>(count) * steps * h->P.K * 48,
                                        cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
        if (e != cudaSuccess) {
            abmx_internal::set_error(std::string("finance run_batch: ") + cudaGetErrorString(e));
            rc = ABMX_E_CUDA;
        } else {
            rc = h->check_err();
        }
    }
    cudaEventSynchronize(b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (kernel_ms) *kernel_ms = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    abmx_finance_destroy(h);
    return rc;
}

}  // extern "C"
