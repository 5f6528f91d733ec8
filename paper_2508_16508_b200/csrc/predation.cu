// predation.cu — the predation step (src/models/predation.cpp:167-263) as four fused
// sm_100a kernels over device-resident SoA state, for R replicas at once.
//
// Per step (all launches stream-ordered, captured once in a CUDA graph):
//   K1 k_move       per slot: RNG move + toroidal wrap + age++ (step_agents, lifecycle.cpp:87-122),
//                   then spatial binning into per-cell epoch-stamped lists (wolves first, then
//                   sheep; ticket-ordered CTAs) and an atomicMin "lowest sheep slot" per cell.
//   K2 k_predation  one thread per cell holding >= 1 wolf: stable (slot-sorted) wolf and sheep
//                   lists, k-th wolf <-> k-th sheep (predation.cpp:197-239).
//   K3 k_update     per slot: graze (lowest slot on a ready cell), predation kill, metabolise,
//                   starve, reproduce (Bernoulli + quantised child energy); the free-slot and
//                   valid-row masks are scanned in ONE single-pass decoupled lookback (two
//                   counters packed per tile) and compacted (spawn_agents rank-match,
//                   lifecycle.cpp:144-195).
//   K4 k_spawn      k-th free slot <- k-th valid row, fresh ids; plus the cell regrow sweep
//                   (predation.cpp:252-258) and the grass count for the metrics row.
//
// HBM layout (per species, per replica, stride Npad): active u8, cell i32 (= y*W + x),
// age i32, energy f64, id i64. Cells: one u8 code per cell (0 = ready, 1..254 = regrow
// countdown, 255 = not ready and frozen: grazed with regrow_delay <= 0, and padding).
// Placeholder slots hold zeros (agent_set.cpp:45-58); the agent type is implied by species.
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

// neighbour order of the move draw (predation.cpp:13-15)
__constant__ int c_dx[8] = {-1, -1, -1, 0, 0, 1, 1, 1};
__constant__ int c_dy[8] = {-1, 0, 1, -1, 1, -1, 0, 1};

__device__ __forceinline__ size_t sidx(const Params& P, int s, int r, int i) {
    return static_cast<size_t>(r) * P.Npad[s] + i;
}
__device__ __forceinline__ size_t cidx(const Params& P, int r, int c) {
    return static_cast<size_t>(r) * P.Cpad + c;
}
__device__ __forceinline__ unsigned long long inv_key(unsigned long long epoch, int slot) {
    return ((0xFFFFFFFFULL - (epoch & 0xFFFFFFFFULL)) << 32) | static_cast<uint32_t>(slot);
}
// exact fixed-point image of an energy on the 2^-20 grid (predation.hpp:60-63)
__device__ __forceinline__ long long to_fx(double e) {
    return __double2ll_rn(__dmul_rn(e, 1048576.0));
}

__device__ __forceinline__ void load8_u8(const uint8_t* p, uint8_t (&v)[kS]) {
    const uint2 w = *reinterpret_cast<const uint2*>(p);
#pragma unroll
    for (int k = 0; k < kS; ++k) v[k] = static_cast<uint8_t>((k < 4 ? w.x : w.y) >> (8 * (k & 3)));
}
__device__ __forceinline__ void store8_u8(uint8_t* p, const uint8_t (&v)[kS]) {
    uint2 w;
    w.x = v[0] | (v[1] << 8) | (v[2] << 16) | (static_cast<uint32_t>(v[3]) << 24);
    w.y = v[4] | (v[5] << 8) | (v[6] << 16) | (static_cast<uint32_t>(v[7]) << 24);
    *reinterpret_cast<uint2*>(p) = w;
}
__device__ __forceinline__ void load8_i32(const int* p, int (&v)[kS]) {
    const int4 a = reinterpret_cast<const int4*>(p)[0], b = reinterpret_cast<const int4*>(p)[1];
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
}
__device__ __forceinline__ void store8_i32(int* p, const int (&v)[kS]) {
    reinterpret_cast<int4*>(p)[0] = make_int4(v[0], v[1], v[2], v[3]);
    reinterpret_cast<int4*>(p)[1] = make_int4(v[4], v[5], v[6], v[7]);
}
__device__ __forceinline__ void load8_f64(const double* p, double (&v)[kS]) {
#pragma unroll
    for (int q = 0; q < kS / 2; ++q) {
        const double2 d = reinterpret_cast<const double2*>(p)[q];
        v[2 * q] = d.x;
        v[2 * q + 1] = d.y;
    }
}
__device__ __forceinline__ void store8_f64(double* p, const double (&v)[kS]) {
#pragma unroll
    for (int q = 0; q < kS / 2; ++q) reinterpret_cast<double2*>(p)[q] = make_double2(v[2 * q], v[2 * q + 1]);
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

// ============================================================== K1: move + bin
__global__ void __launch_bounds__(kT) k_move(Params P) {
    __shared__ unsigned s_ticket;
    __shared__ unsigned long long s_key;
    Ctl* ctl = P.ctl;
    if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->k1_ticket, 1u);
    __syncthreads();
    const unsigned ticket = s_ticket;
    const unsigned long long epoch = ctl->epoch;
    const long long t = ctl->t;
    const unsigned wolf_ctas = static_cast<unsigned>(P.R * P.tiles[1]);
    int s, r, tile;
    if (ticket < wolf_ctas) {
        s = 1;
        r = ticket / P.tiles[1];
        tile = ticket % P.tiles[1];
    } else {
        s = 0;
        const unsigned u = ticket - wolf_ctas;
        r = u / P.tiles[0];
        tile = u % P.tiles[0];
    }
    // zero this parity's event accumulators (consumed by K2..K4 of this step)
    {
        Events* ev = P.ev + static_cast<size_t>(epoch & 1) * P.R;
        for (int rr = ticket; rr < P.R; rr += gridDim.x)
            if (threadIdx.x == 0) memset(&ev[rr], 0, sizeof(Events));
    }
    if (threadIdx.x == 0) {
        if (s == 0) {  // sheep bin only after every wolf is binned (sheep lists are built
                       // only for cells that hold a wolf)
            while (ld_acquire_u32(&ctl->k1_wolves_done) < wolf_ctas) __nanosleep(64);
        }
        s_key = split(split(split(P.seeds[r], 3), static_cast<unsigned long long>(t)), s);
    }
    __syncthreads();
    const unsigned long long key = s_key;
    const int i0 = tile * kTile + threadIdx.x * kS;
    const int W = P.W, H = P.H;
    if (i0 < P.N[s]) {
        const size_t base = sidx(P, s, r, i0);
        uint8_t act[kS];
        load8_u8(P.active[s] + base, act);
        bool any = false;
#pragma unroll
        for (int k = 0; k < kS; ++k) any |= act[k] != 0;
        int cell[kS], age[kS];
        bool first[kS];
        if (any) {
            load8_i32(P.cell[s] + base, cell);
            load8_i32(P.age[s] + base, age);
        }
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            first[k] = false;
            if (!act[k]) continue;
            const int i = i0 + k;
            const int u = static_cast<int>(draw(key, static_cast<unsigned long long>(i)) >> 61);
            const int c = cell[k];
            const int y = c / W, x = c - y * W;
            int nx = x + c_dx[u], ny = y + c_dy[u];
            nx = nx < 0 ? nx + W : (nx >= W ? nx - W : nx);
            ny = ny < 0 ? ny + H : (ny >= H ? ny - H : ny);
            const int nc = ny * W + nx;
            cell[k] = nc;
            age[k] += 1;
            const unsigned long long stamp = (epoch << 32) | static_cast<uint32_t>(i);
            const size_t ci = cidx(P, r, nc);
            if (s == 1) {
                const unsigned long long old = atomicExch(&P.head[1][ci], stamp);
                first[k] = (old >> 32) != (epoch & 0xFFFFFFFFULL);
                P.next[1][base + k] = first[k] ? -1 : static_cast<int>(static_cast<uint32_t>(old));
            } else {
                atomicMin(&P.smin[ci], inv_key(epoch, i));
                const unsigned long long hw = __ldcg(&P.head[1][ci]);
                if ((hw >> 32) == (epoch & 0xFFFFFFFFULL)) {
                    const unsigned long long old = atomicExch(&P.head[0][ci], stamp);
                    P.next[0][base + k] =
                        (old >> 32) == (epoch & 0xFFFFFFFFULL) ? static_cast<int>(static_cast<uint32_t>(old)) : -1;
                }
            }
        }
        if (any) {
            store8_i32(P.cell[s] + base, cell);
            store8_i32(P.age[s] + base, age);
        }
        if (ctl->needs_blend) {  // step_agents masks placeholder state back to defaults
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (!act[k] && i0 + k < P.N[s]) {
                    P.cell[s][base + k] = 0;
                    P.energy[s][base + k] = 0.0;
                }
        }
        if (s == 1) {
#pragma unroll
            for (int k = 0; k < kS; ++k) {
                const unsigned pos = warp_append(&ctl->wcell_count, first[k]);
                if (first[k]) P.wcells[pos] = (static_cast<unsigned long long>(r) << 32) | static_cast<uint32_t>(cell[k]);
            }
        }
    } else if (s == 1) {
        // keep warp_append convergent: nothing to append
    }
    if (s == 1) {
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            atomicAdd(&ctl->k1_wolves_done, 1u);
        }
    }
}

// ============================================================== K2: predation pairing
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

__global__ void __launch_bounds__(256) k_predation(Params P) {
    Ctl* ctl = P.ctl;
    const unsigned count = *reinterpret_cast<volatile unsigned*>(&ctl->wcell_count);
    const unsigned long long epoch = ctl->epoch & 0xFFFFFFFFULL;
    Events* ev = P.ev + static_cast<size_t>(ctl->epoch & 1) * P.R;
    for (unsigned e = blockIdx.x * blockDim.x + threadIdx.x; e < count; e += gridDim.x * blockDim.x) {
        const unsigned long long ent = P.wcells[e];
        const int r = static_cast<int>(ent >> 32), c = static_cast<int>(static_cast<uint32_t>(ent));
        const size_t ci = cidx(P, r, c);
        const size_t wb = static_cast<size_t>(r) * P.Npad[1], sb = static_cast<size_t>(r) * P.Npad[0];
        const unsigned long long hw = P.head[1][ci];
        const unsigned long long hs = P.head[0][ci];
        const int w0 = static_cast<int>(static_cast<uint32_t>(hw));
        const int s0 = (hs >> 32) == epoch ? static_cast<int>(static_cast<uint32_t>(hs)) : -1;
        int lw = 0, ls = 0;
        for (int w = w0; w >= 0; w = P.next[1][wb + w]) ++lw;
        for (int v = s0; v >= 0; v = P.next[0][sb + v]) ++ls;
        if (ls == 0) continue;
        const int pairs = lw < ls ? lw : ls;
        if (lw <= kSmallList && ls <= kSmallList) {
            int wl[kSmallList], sl[kSmallList];
            int k = 0;
            for (int w = w0; w >= 0; w = P.next[1][wb + w]) wl[k++] = w;
            k = 0;
            for (int v = s0; v >= 0; v = P.next[0][sb + v]) sl[k++] = v;
            insertion_sort(wl, lw);
            insertion_sort(sl, ls);
            for (int q = 0; q < pairs; ++q) {
                P.flag[0][sb + sl[q]] = 1;  // eaten
                P.flag[1][wb + wl[q]] = 1;  // ate
            }
        } else {
            const unsigned off = atomicAdd(&ctl->pool_top, static_cast<unsigned>(lw + ls));
            if (static_cast<long long>(off) + lw + ls > P.pool_size) {
                atomicExch(&ctl->error, 1u);
                continue;
            }
            int* wl = P.pool + off;
            int* sl = wl + lw;
            int k = 0;
            for (int w = w0; w >= 0; w = P.next[1][wb + w]) wl[k++] = w;
            k = 0;
            for (int v = s0; v >= 0; v = P.next[0][sb + v]) sl[k++] = v;
            heap_sort(wl, lw);
            heap_sort(sl, ls);
            for (int q = 0; q < pairs; ++q) {
                P.flag[0][sb + sl[q]] = 1;
                P.flag[1][wb + wl[q]] = 1;
            }
        }
        atomicAdd(&ev[r].sheep_eaten, static_cast<unsigned long long>(pairs));
    }
}

// ============================================================== K3: per-slot update + scans
__global__ void __launch_bounds__(kT) k_update(Params P) {
    __shared__ unsigned s_ticket;
    __shared__ unsigned long long s_key;
    __shared__ unsigned long long s_scan[kT / 32 + 1];
    __shared__ unsigned long long s_prefix;
    __shared__ long long s_red[kT / 32];
    Ctl* ctl = P.ctl;
    if (threadIdx.x == 0) s_ticket = atomicAdd(&ctl->k3_ticket, 1u);
    __syncthreads();
    const unsigned ticket = s_ticket;
    const unsigned long long epoch = ctl->epoch;
    const int p = static_cast<int>(epoch & 1);
    const unsigned sheep_ctas = static_cast<unsigned>(P.R * P.tiles[0]);
    int s, r, tile;
    if (ticket < sheep_ctas) {
        s = 0;
        r = ticket / P.tiles[0];
        tile = ticket % P.tiles[0];
    } else {
        s = 1;
        const unsigned u = ticket - sheep_ctas;
        r = u / P.tiles[1];
        tile = u % P.tiles[1];
    }
    if (threadIdx.x == 0) {
        s_key = split(split(split(P.seeds[r], 4), static_cast<unsigned long long>(ctl->t)), s);
        // clear this tile's lookback word of the other parity for the next step
        P.status[((static_cast<size_t>(1 - p) * 2 + s) * P.R + r) * P.status_stride + tile] = 0ULL;
    }
    __syncthreads();
    const unsigned long long key = s_key;
    unsigned long long* status = P.status + ((static_cast<size_t>(p) * 2 + s) * P.R + r) * P.status_stride;
    const int N = P.N[s];
    const int i0 = tile * kTile + threadIdx.x * kS;
    const size_t base = sidx(P, s, r, i0);
    const double gain = P.gain[s], metab = P.metab, prob = P.prob[s], frac = P.frac;

    uint8_t act[kS], flg[kS];
    double E[kS], child[kS];
    int cell[kS];
    bool valid[kS], freek[kS];
    unsigned n_graze = 0, n_metab = 0, n_death = 0;
    long long fx_removed = 0;
    if (i0 < N) {
        load8_u8(P.active[s] + base, act);
        load8_u8(P.flag[s] + base, flg);
        bool any = false, anyflag = false;
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            any |= act[k] != 0;
            anyflag |= flg[k] != 0;
        }
        if (anyflag) {
            const uint8_t z[kS] = {0, 0, 0, 0, 0, 0, 0, 0};
            store8_u8(P.flag[s] + base, z);
        }
        if (any) {
            load8_f64(P.energy[s] + base, E);
            if (s == 0) load8_i32(P.cell[s] + base, cell);
        }
        bool died_any = false;
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            valid[k] = false;
            child[k] = 0.0;
            const int i = i0 + k;
            bool alive = act[k] != 0;
            if (alive) {
                if (s == 0) {
                    // graze: lowest active sheep slot on a ready cell eats (predation.cpp:178-195)
                    const size_t ci = cidx(P, r, cell[k]);
                    if (static_cast<int>(static_cast<uint32_t>(P.smin[ci])) == i && P.g[ci] == 0) {
                        P.g[ci] = static_cast<uint8_t>(P.delay_code);
                        E[k] = __dadd_rn(E[k], gain);
                        ++n_graze;
                    }
                    if (flg[k]) {  // eaten by a wolf this step (predation.cpp:224-238)
                        fx_removed += to_fx(E[k]);
                        ++n_death;
                        alive = false;
                    }
                } else if (flg[k]) {
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
        if (any) store8_f64(P.energy[s] + base, E);
        if (died_any) {
            store8_u8(P.active[s] + base, act);
#pragma unroll
            for (int k = 0; k < kS; ++k)
                if (!act[k] && i0 + k < N) {
                    P.cell[s][base + k] = 0;
                    P.age[s][base + k] = 0;
                    P.id[s][base + k] = 0;
                }
        }
    } else {
#pragma unroll
        for (int k = 0; k < kS; ++k) {
            valid[k] = false;
            freek[k] = false;
            child[k] = 0.0;
        }
    }
    unsigned nf = 0, nv = 0;
#pragma unroll
    for (int k = 0; k < kS; ++k) {
        nf += freek[k];
        nv += valid[k];
    }
    unsigned long long tile_total;
    const unsigned long long excl = block_excl_scan<kT>(pack2(nf, nv), s_scan, &tile_total);
    if (threadIdx.x < 32) {
        const unsigned long long pre = tile_lookback(status, tile, tile_total);
        if (threadIdx.x == 0) s_prefix = pre;
    }
    __syncthreads();
    const unsigned long long pre = s_prefix + excl;
    int fr = static_cast<int>(hi31(pre)), vr = static_cast<int>(lo31(pre));
    const size_t rb = static_cast<size_t>(r) * P.Npad[s];
#pragma unroll
    for (int k = 0; k < kS; ++k) {
        if (freek[k]) P.free_at[s][rb + fr++] = i0 + k;
        if (valid[k]) {
            int c = (s == 0) ? cell[k] : P.cell[s][base + k];
            P.row_at[s][rb + vr] = i0 + k;
            P.rowcell[s][rb + vr] = c;
            P.rowE[s][rb + vr] = child[k];
            ++vr;
        }
    }
    // event reductions
    Events* ev = P.ev + static_cast<size_t>(p) * P.R + r;
    const long long g_sum = block_sum<long long>(n_graze, s_red);
    const long long m_sum = block_sum<long long>(n_metab, s_red);
    const long long d_sum = block_sum<long long>(n_death, s_red);
    const long long x_sum = block_sum<long long>(fx_removed, s_red);
    if (threadIdx.x == 0) {
        if (g_sum) atomicAdd(&ev->grass_eaten, static_cast<unsigned long long>(g_sum));
        if (m_sum) atomicAdd(&ev->metabolized[s], static_cast<unsigned long long>(m_sum));
        if (d_sum) atomicAdd(&ev->deaths[s], static_cast<unsigned long long>(d_sum));
        if (x_sum) atomicAdd(reinterpret_cast<unsigned long long*>(&ev->e_removed_fx[s]), static_cast<unsigned long long>(x_sum));
        if (tile == P.tiles[s] - 1) {
            // last tile: totals known -> spawn plan, counters and the metrics row
            const unsigned long long tot = s_prefix + tile_total;
            const int F = static_cast<int>(hi31(tot)), Q = static_cast<int>(lo31(tot));
            const int pairs = F < Q ? F : Q;
            SpeciesRep* sr = &P.rep[static_cast<size_t>(r) * 2 + s];
            sr->base_id = sr->next_id;
            sr->pairs = pairs;
            sr->Q = Q;
            sr->next_id += pairs;
            sr->num_active = N - F + pairs;
            atomicAdd(&ev->births[s], static_cast<unsigned long long>(pairs));
            atomicAdd(&ev->dropped[s], static_cast<unsigned long long>(Q - pairs));
            long long* row = ctl->metrics + (static_cast<size_t>(r) * ctl->metrics_stride + ctl->run_step) * 4;
            row[s] = sr->num_active;
            if (Q - pairs) atomicAdd(reinterpret_cast<unsigned long long*>(&row[3]), static_cast<unsigned long long>(Q - pairs));
        }
    }
}

// ============================================================== K4: spawn + regrow
__global__ void __launch_bounds__(kT) k_spawn_regrow(Params P) {
    __shared__ long long s_red[kT / 32];
    __shared__ bool s_last;
    Ctl* ctl = P.ctl;
    const unsigned long long epoch = ctl->epoch;
    if (static_cast<int>(blockIdx.x) < P.spawn_ctas) {
        const int rs = blockIdx.x / P.spawn_cps, local = blockIdx.x % P.spawn_cps;
        const int s = rs / P.R, r = rs % P.R;
        const SpeciesRep sr = P.rep[static_cast<size_t>(r) * 2 + s];
        const size_t rb = static_cast<size_t>(r) * P.Npad[s];
        long long fx_dropped = 0;
        for (int k = local * kT + threadIdx.x; k < sr.Q; k += P.spawn_cps * kT) {
            if (k < sr.pairs) {
                const size_t slot = rb + P.free_at[s][rb + k];
                P.active[s][slot] = 1;
                P.cell[s][slot] = P.rowcell[s][rb + k];
                P.energy[s][slot] = P.rowE[s][rb + k];
                P.age[s][slot] = 0;
                P.id[s][slot] = sr.base_id + k;
            } else {
                fx_dropped += to_fx(P.rowE[s][rb + k]);  // predation.cpp:121-135
            }
        }
        if (sr.Q > sr.pairs) {
            const long long tot = block_sum<long long>(fx_dropped, s_red);
            if (threadIdx.x == 0 && tot) {
                Events* ev = P.ev + static_cast<size_t>(epoch & 1) * P.R + r;
                atomicAdd(reinterpret_cast<unsigned long long*>(&ev->e_dropped_fx[s]), static_cast<unsigned long long>(tot));
            }
        }
    } else {
        // regrow: 16 cells per thread (Cpad is a multiple of 16, so a chunk never straddles replicas)
        const size_t q = static_cast<size_t>(blockIdx.x - P.spawn_ctas) * kT + threadIdx.x;
        const size_t c0 = q * 16;
        unsigned ready = 0;
        int r = -1;
        if (c0 < static_cast<size_t>(P.R) * P.Cpad) {
            r = static_cast<int>(c0 / P.Cpad);
            uint4 v = *reinterpret_cast<const uint4*>(P.g + c0);
            uint32_t w[4] = {v.x, v.y, v.z, v.w};
            bool changed = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t o = 0;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    uint32_t x = (w[j] >> (8 * b)) & 0xFF;
                    if (x >= 1 && x <= 254) {
                        --x;
                        changed = true;
                    }
                    ready += x == 0;
                    o |= x << (8 * b);
                }
                w[j] = o;
            }
            if (changed) *reinterpret_cast<uint4*>(P.g + c0) = make_uint4(w[0], w[1], w[2], w[3]);
        }
        // per-replica grass count, aggregated over the lanes of a warp sharing a replica
        const unsigned grp = __match_any_sync(0xffffffffu, r);
        const unsigned tot = __reduce_add_sync(grp, ready);
        if (r >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1 && tot) {
            long long* row = ctl->metrics + (static_cast<size_t>(r) * ctl->metrics_stride + ctl->run_step) * 4;
            atomicAdd(reinterpret_cast<unsigned long long*>(&row[2]), static_cast<unsigned long long>(tot));
        }
    }
    // the last CTA to finish closes the step
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        s_last = atomicAdd(&ctl->k4_done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        ctl->epoch = epoch + 1;
        ctl->t += 1;
        ctl->run_step += 1;
        ctl->k1_ticket = 0;
        ctl->k1_wolves_done = 0;
        ctl->k3_ticket = 0;
        ctl->wcell_count = 0;
        ctl->pool_top = 0;
        ctl->needs_blend = 0;
        ctl->k4_done = 0;
        __threadfence();
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
        P.g[q] = c < P.C ? 0 : 255;  // full grass; padding frozen
    }
}

}  // namespace abmx_pred

// ====================================================================== host engine
namespace abmx_pred {

static const char* kKernelNames[kNumKernels] = {"k_move", "k_predation", "k_update", "k_spawn_regrow"};

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
    for (auto& ev : tev)
        if (ev) cudaEventDestroy(ev);
    for (void* p : allocs) cudaFree(p);
    if (d_run_metrics) cudaFree(d_run_metrics);
    if (flush_buf) cudaFree(flush_buf);
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

int Engine::create(const abmx_predation_config& c, const uint64_t* seeds, int R_) {
    cfg = c;
    R = R_;
    if (R < 1) {
        abmx_internal::set_error("replicas must be >= 1");
        return ABMX_E_DOMAIN;
    }
    if (c.width < 1 || c.height < 1) {
        abmx_internal::set_error("width and height must be >= 1");
        return ABMX_E_DOMAIN;
    }
    if (c.sheep_capacity < 0 || c.wolf_capacity < 0 || c.n_sheep0 < 0 || c.n_wolves0 < 0) {
        abmx_internal::set_error("negative capacity");
        return ABMX_E_CAPACITY;
    }
    if (c.n_sheep0 > c.sheep_capacity || c.n_wolves0 > c.wolf_capacity) {
        abmx_internal::set_error("initial counts exceed capacities");  // predation.cpp:155-156
        return ABMX_E_CAPACITY;
    }
    if (c.regrow_delay > 254) {
        abmx_internal::set_error("regrow_delay > 254 is not representable in the u8 cell layout");
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
        P.Npad[s] = (N[s] + 15) / 16 * 16;
        if (P.Npad[s] == 0) P.Npad[s] = 16;
        P.tiles[s] = (N[s] + kTile - 1) / kTile;
        if (P.tiles[s] == 0) P.tiles[s] = 1;
    }
    P.gain[0] = c.energy_gain_sheep;
    P.gain[1] = c.energy_gain_wolf;
    P.metab = c.metabolism;
    P.prob[0] = c.reproduce_prob_sheep;
    P.prob[1] = c.reproduce_prob_wolf;
    P.frac = c.reproduce_energy_frac;
    P.delay_code = c.regrow_delay >= 1 ? static_cast<unsigned>(c.regrow_delay) : 255u;
    const int maxN = N[0] > N[1] ? N[0] : N[1];
    P.spawn_cps = maxN / 8192;
    if (P.spawn_cps < 1) P.spawn_cps = 1;
    if (P.spawn_cps > 64) P.spawn_cps = 64;
    P.spawn_ctas = 2 * R * P.spawn_cps;
    const long long chunks = (static_cast<long long>(R) * P.Cpad) / 16;
    P.regrow_ctas = static_cast<int>((chunks + kT - 1) / kT);
    P.k2_ctas = abmx_internal::num_sms() * 4;
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
        AL(P.free_at[s], n * 4);
        AL(P.row_at[s], n * 4);
        AL(P.rowcell[s], n * 4);
        AL(P.rowE[s], n * 8);
        AL(P.head[s], static_cast<size_t>(R) * P.Cpad * 8);
    }
    AL(P.g, static_cast<size_t>(R) * P.Cpad);
    AL(P.smin, static_cast<size_t>(R) * P.Cpad * 8);
    AL(P.status, static_cast<size_t>(2) * 2 * R * P.status_stride * 8);
    AL(P.wcells, static_cast<size_t>(R) * (P.Npad[1]) * 8);
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
    for (int s = 0; s < 2; ++s) {
        CK(cudaMemsetAsync(P.head[s], 0, static_cast<size_t>(R) * P.Cpad * 8, stream));
        CK(cudaMemsetAsync(P.next[s], 0xFF, static_cast<size_t>(R) * P.Npad[s] * 4, stream));
    }
    CK(cudaMemsetAsync(P.smin, 0xFF, static_cast<size_t>(R) * P.Cpad * 8, stream));
    CK(cudaMemsetAsync(P.status, 0, static_cast<size_t>(2) * 2 * R * P.status_stride * 8, stream));
    CK(cudaMemsetAsync(P.ev, 0, sizeof(Events) * 2 * R, stream));
    Ctl ctl;
    memset(&ctl, 0, sizeof ctl);
    ctl.epoch = 1;
    ctl.t = 1;
    ctl.metrics = d_metrics_step;
    ctl.metrics_stride = 1;
    cur_metrics = d_metrics_step;
    cur_stride = 1;
    CK(cudaMemcpyAsync(P.ctl, &ctl, sizeof ctl, cudaMemcpyHostToDevice, stream));
    next_t = 1;
    std::vector<SpeciesRep> rep(static_cast<size_t>(2) * R);
    for (int r = 0; r < R; ++r) {
        rep[2 * r + 0] = SpeciesRep{c.n_sheep0, 0, c.n_sheep0, 0, 0, 0};
        rep[2 * r + 1] = SpeciesRep{c.n_wolves0, 0, c.n_wolves0, 0, 0, 0};
    }
    CK(cudaMemcpyAsync(P.rep, rep.data(), sizeof(SpeciesRep) * rep.size(), cudaMemcpyHostToDevice, stream));
    CK(cudaStreamSynchronize(stream));  // rep (a host vector) must be consumed
    const int g = abmx_internal::num_sms() * 8;
    (void)cudaGetLastError();
    k_init_species<<<g, 256, 0, stream>>>(P, 0, c.n_sheep0);
    k_init_species<<<g, 256, 0, stream>>>(P, 1, c.n_wolves0);
    k_init_cells<<<g, 256, 0, stream>>>(P);
    abmx_internal::count_launch(3);
    CK(cudaGetLastError());
    CK(cudaMemsetAsync(d_metrics_step, 0, sizeof(long long) * 4 * R, stream));
    for (int k = 0; k < kNumKernels; ++k) {
        CK(cudaEventCreate(&tev[2 * k]));
        CK(cudaEventCreate(&tev[2 * k + 1]));
    }
    return ABMX_OK;
}

void Engine::launch_step_kernels(bool timed) {
    const Params& P = params;
    const unsigned k1 = static_cast<unsigned>(P.R * (P.tiles[0] + P.tiles[1]));
    if (timed) cudaEventRecord(tev[0], stream);
    k_move<<<k1, kT, 0, stream>>>(P);
    if (timed) {
        cudaEventRecord(tev[1], stream);
        cudaEventRecord(tev[2], stream);
    }
    k_predation<<<P.k2_ctas, 256, 0, stream>>>(P);
    if (timed) {
        cudaEventRecord(tev[3], stream);
        cudaEventRecord(tev[4], stream);
    }
    k_update<<<k1, kT, 0, stream>>>(P);
    if (timed) {
        cudaEventRecord(tev[5], stream);
        cudaEventRecord(tev[6], stream);
    }
    k_spawn_regrow<<<P.spawn_ctas + P.regrow_ctas, kT, 0, stream>>>(P);
    if (timed) cudaEventRecord(tev[7], stream);
    abmx_internal::count_launch(kNumKernels);
}

int Engine::accumulate_times() {
    CK(cudaEventSynchronize(tev[7]));
    for (int k = 0; k < kNumKernels; ++k) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, tev[2 * k], tev[2 * k + 1]));
        kernel_ms[k] += ms;
        kernel_launches[k] += 1;
    }
    return ABMX_OK;
}

int Engine::set_t(long long t) {
    if (t != next_t) {
        staged_t = t;
        CK(cudaMemcpyAsync(&params.ctl->t, &staged_t, sizeof(long long), cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        next_t = t;
    }
    return ABMX_OK;
}

int Engine::set_metrics_target(long long* d_metrics, unsigned stride) {
    if (d_metrics != cur_metrics || stride != cur_stride) {
        staged_ptr = d_metrics;
        staged_u[0] = 0;
        staged_u[1] = stride;
        CK(cudaMemcpyAsync(&params.ctl->metrics, &staged_ptr, sizeof(long long*), cudaMemcpyHostToDevice, stream));
        CK(cudaMemcpyAsync(&params.ctl->run_step, staged_u, sizeof(unsigned) * 2, cudaMemcpyHostToDevice, stream));
        CK(cudaStreamSynchronize(stream));
        cur_metrics = d_metrics;
        cur_stride = stride;
    } else {
        CK(cudaMemsetAsync(&params.ctl->run_step, 0, sizeof(unsigned), stream));
    }
    return ABMX_OK;
}

int Engine::launch_steps(long long steps) {
    (void)cudaGetLastError();  // drop stale non-sticky errors of unrelated runtime calls
    for (long long q = 0; q < steps; ++q) {
        if (timing) {
            launch_step_kernels(true);
            int rc = accumulate_times();
            if (rc) return rc;
        } else {
            if (!graph_exec) {
                cudaGraph_t graph;
                CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeThreadLocal));
                launch_step_kernels(false);
                CK(cudaStreamEndCapture(stream, &graph));
                CK(cudaGraphInstantiate(&graph_exec, graph, 0));
                cudaGraphDestroy(graph);
                abmx_internal::count_launch(-kNumKernels);  // capture launched nothing
            }
            CK(cudaGraphLaunch(graph_exec, stream));
            abmx_internal::count_launch(kNumKernels);
        }
        ++next_t;
        ++host_epoch;
    }
    CK(cudaGetLastError());
    return ABMX_OK;
}

int Engine::step(long long t) {
    // the step index is this call's only input: always ship it (8 B H2D), then launch
    staged_t = t;
    CK(cudaMemcpyAsync(&params.ctl->t, &staged_t, sizeof(long long), cudaMemcpyHostToDevice, stream));
    next_t = t;
    int rc = ABMX_OK;
    CK(cudaMemsetAsync(d_metrics_step, 0, sizeof(long long) * 4 * R, stream));
    rc = set_metrics_target(d_metrics_step, 1);
    if (rc) return rc;
    rc = launch_steps(1);
    last_run_steps = 0;
    return rc;
}

int Engine::run_async(long long t0, long long steps) {
    if (steps <= 0) return ABMX_OK;
    if (steps > 0x7FFFFFFFLL) {
        abmx_internal::set_error("too many steps in one run");
        return ABMX_E_DOMAIN;
    }
    int rc = set_t(t0);
    if (rc) return rc;
    const size_t mbytes = sizeof(long long) * 4 * static_cast<size_t>(R) * static_cast<size_t>(steps);
    if (mbytes > run_metrics_bytes) {
        CK(cudaStreamSynchronize(stream));
        if (d_run_metrics) cudaFree(d_run_metrics);
        cur_metrics = nullptr;
        CK(cudaMalloc(&d_run_metrics, mbytes));
        run_metrics_bytes = mbytes;
    }
    CK(cudaMemsetAsync(d_run_metrics, 0, mbytes, stream));
    rc = set_metrics_target(d_run_metrics, static_cast<unsigned>(steps));
    if (rc) return rc;
    rc = launch_steps(steps);
    last_run_steps = steps;
    return rc;
}

int Engine::fetch_run_metrics(double* out) {
    const size_t n = static_cast<size_t>(R) * static_cast<size_t>(last_run_steps) * 4;
    std::vector<long long> h(n);
    if (n) {
        CK(cudaMemcpyAsync(h.data(), d_run_metrics, n * sizeof(long long), cudaMemcpyDeviceToHost, stream));
    }
    CK(cudaStreamSynchronize(stream));
    for (size_t i = 0; i < n; ++i) out[i] = static_cast<double>(h[i]);
    return ABMX_OK;
}

int Engine::last_metrics(long long* out) {
    if (last_run_steps == 0) {
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
    *num_active = sr.num_active;
    *next_id = sr.next_id;
    return ABMX_OK;
}

int Engine::import_species(int r, int s, const uint8_t* active, const int64_t* ids, const int64_t* ages,
                           const int64_t* x, const int64_t* y, const double* energy, int32_t num_active,
                           int64_t next_id) {
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
        if (act[i]) {
            if (x[i] < 0 || x[i] >= P.W || y[i] < 0 || y[i] >= P.H) {
                abmx_internal::set_error("active agent outside the lattice");
                return ABMX_E_DOMAIN;
            }
            cell[i] = static_cast<int>(y[i] * P.W + x[i]);
        } else {
            // placeholder state must be representable; step_agents blends it to zero
            if (x[i] < 0 || x[i] >= P.W || y[i] < 0 || y[i] >= P.H) {
                abmx_internal::set_error("placeholder coordinates outside the lattice");
                return ABMX_E_DOMAIN;
            }
            cell[i] = static_cast<int>(y[i] * P.W + x[i]);
        }
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
    SpeciesRep sr{num_active, 0, next_id, 0, 0, 0};
    CK(cudaMemcpy(P.rep + static_cast<size_t>(r) * 2 + s, &sr, sizeof sr, cudaMemcpyHostToDevice));
    const unsigned one = 1;
    CK(cudaMemcpy(&P.ctl->needs_blend, &one, sizeof one, cudaMemcpyHostToDevice));
    return ABMX_OK;
}

int Engine::export_world(int r, uint8_t* ready, int64_t* regrow) {
    const Params& P = params;
    const size_t C = static_cast<size_t>(P.C);
    std::vector<uint8_t> g(C);
    CK(cudaMemcpyAsync(g.data(), P.g + static_cast<size_t>(r) * P.Cpad, C, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    for (size_t c = 0; c < C; ++c) {
        ready[c] = g[c] == 0;
        regrow[c] = g[c] == 255 ? (cfg.regrow_delay <= 0 ? cfg.regrow_delay : 0) : g[c];
    }
    return ABMX_OK;
}

int Engine::import_world(int r, const uint8_t* ready, const int64_t* regrow) {
    const Params& P = params;
    const size_t C = static_cast<size_t>(P.C);
    std::vector<uint8_t> g(C);
    for (size_t c = 0; c < C; ++c) {
        if (ready[c]) {
            if (regrow[c] != 0) {
                abmx_internal::set_error("grass_ready cell with a nonzero regrow counter");
                return ABMX_E_DOMAIN;
            }
            g[c] = 0;
        } else if (regrow[c] >= 1 && regrow[c] <= 254) {
            g[c] = static_cast<uint8_t>(regrow[c]);
        } else if (regrow[c] <= 0) {
            g[c] = 255;  // not ready and never regrowing (predation.cpp:254 guard)
        } else {
            abmx_internal::set_error("regrow counter > 254 not representable");
            return ABMX_E_DOMAIN;
        }
    }
    CK(cudaStreamSynchronize(stream));
    CK(cudaMemcpy(P.g + static_cast<size_t>(r) * P.Cpad, g.data(), C, cudaMemcpyHostToDevice));
    return ABMX_OK;
}

int Engine::birth_pairs(int r, int s, int32_t* parent, int32_t* child, int32_t cap) {
    const Params& P = params;
    SpeciesRep sr;
    CK(cudaMemcpyAsync(&sr, P.rep + static_cast<size_t>(r) * 2 + s, sizeof sr, cudaMemcpyDeviceToHost, stream));
    CK(cudaStreamSynchronize(stream));
    const int n = sr.pairs < cap ? sr.pairs : cap;
    const size_t off = static_cast<size_t>(r) * P.Npad[s];
    if (n > 0) {
        CK(cudaMemcpyAsync(parent, P.row_at[s] + off, n * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaMemcpyAsync(child, P.free_at[s] + off, n * 4, cudaMemcpyDeviceToHost, stream));
        CK(cudaStreamSynchronize(stream));
    }
    return sr.pairs;
}

// L2 flush: overwrite a buffer larger than the 126 MB L2 between timed steps.
__global__ void k_flush(uint4* p, size_t n) {
    for (size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = make_uint4(static_cast<unsigned>(i), 0u, 0u, 0u);
}

int Engine::bench(long long t0, long long steps, size_t flush_bytes, bool per_kernel, double* step_ms) {
    if (steps <= 0) return ABMX_OK;
    int rc = set_t(t0);
    if (rc) return rc;
    const size_t mbytes = sizeof(long long) * 4 * static_cast<size_t>(R) * static_cast<size_t>(steps);
    if (mbytes > run_metrics_bytes) {
        CK(cudaStreamSynchronize(stream));
        if (d_run_metrics) cudaFree(d_run_metrics);
        cur_metrics = nullptr;
        CK(cudaMalloc(&d_run_metrics, mbytes));
        run_metrics_bytes = mbytes;
    }
    CK(cudaMemsetAsync(d_run_metrics, 0, mbytes, stream));
    rc = set_metrics_target(d_run_metrics, static_cast<unsigned>(steps));
    if (rc) return rc;
    if (flush_bytes > flush_cap) {
        if (flush_buf) cudaFree(flush_buf);
        CK(cudaMalloc(&flush_buf, flush_bytes));
        flush_cap = flush_bytes;
    }
    std::vector<cudaEvent_t> ev(2 * static_cast<size_t>(steps));
    for (auto& e : ev) CK(cudaEventCreate(&e));
    const bool saved_timing = timing;
    timing = per_kernel;
    for (long long q = 0; q < steps; ++q) {
        if (flush_bytes) {
            k_flush<<<abmx_internal::num_sms() * 4, 256, 0, stream>>>(static_cast<uint4*>(flush_buf), flush_bytes / 16);
        }
        CK(cudaEventRecord(ev[2 * q], stream));
        rc = launch_steps(1);
        if (rc) {
            timing = saved_timing;
            return rc;
        }
        CK(cudaEventRecord(ev[2 * q + 1], stream));
    }
    timing = saved_timing;
    CK(cudaStreamSynchronize(stream));
    for (long long q = 0; q < steps; ++q) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ev[2 * q], ev[2 * q + 1]));
        step_ms[q] = ms;
    }
    for (auto& e : ev) cudaEventDestroy(e);
    last_run_steps = steps;
    return ABMX_OK;
}

}  // namespace abmx_pred
