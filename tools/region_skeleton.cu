// Feasibility probe for a region-decomposed predation step (DESIGN.md §12 "next"): the memory
// traffic and synchronisation skeleton of one step on C2 (2048x2048 cells, ~390k agents),
// without the model logic. One CTA per 32x32-cell region (4096 CTAs), in ticket order:
//   read own agent records (32 B each, coalesced) + the neighbours' edge sub-buckets (halo),
//   read the region's 1024 grass-due words, move every record (counter RNG), keep those landing
//   in the region, bin them into shared-memory cell lists (shared atomics), read the cell heads
//   back, classify into 9 sub-buckets, get the region's output offset by a decoupled lookback
//   over the region counts, write the records and the due words, a few global atomics.
// L2 is flushed between timed launches.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o region_skeleton tools/region_skeleton.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

constexpr int S = 32, W = 2048, H = 2048, RW = W / S, RH = H / S, NREG = RW * RH;
constexpr int kT = 128, kMaxRec = 320;

struct Rec {
    unsigned slot, cell, age, flags;
    double energy;
    long long id;
};

__device__ __forceinline__ unsigned long long mix(unsigned long long z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ int sub_of(int lx, int ly) {  // 0..3 corners, 4..7 edges, 8 interior
    const bool l = lx == 0, r = lx == S - 1, b = ly == 0, t = ly == S - 1;
    if (b && l) return 0;
    if (b && r) return 1;
    if (t && l) return 2;
    if (t && r) return 3;
    if (b) return 4;
    if (t) return 5;
    if (l) return 6;
    if (r) return 7;
    return 8;
}

struct P {
    const Rec* in;
    Rec* out;
    const unsigned* in_off;  // [NREG][10] sub-bucket offsets (prefix, 10 entries)
    unsigned* out_off;
    unsigned* due;           // [NREG][1024]
    unsigned long long* status;  // lookback [NREG]
    unsigned* ticket;
    unsigned* tile_cnt;      // fake slot-space counters
    unsigned salt;
    int mode;  // bit 0: no lookback (fixed per-region output slots), bit 1: no output writes, bit 2: blockIdx order (no ticket)
};

__global__ void __launch_bounds__(kT) k_step(P p) {
    __shared__ Rec rec[kMaxRec];
    __shared__ unsigned head[S * S];
    __shared__ unsigned short nxt[kMaxRec];
    __shared__ unsigned lowest[S * S];
    __shared__ unsigned s_due[S * S];
    __shared__ unsigned s_n, s_region, s_cnt[9], s_base;
    __shared__ unsigned long long s_excl;
    __shared__ unsigned s_lo[9], s_len[9];
    const int reg = blockIdx.x, rx = reg % RW, ry = reg / RW;
    if (threadIdx.x == 0) {
        s_n = 0;
        for (int k = 0; k < 9; ++k) s_cnt[k] = 0;
    }
    if (threadIdx.x < 9) {  // the 9 source ranges (own region + the facing halo of 8 neighbours)
        const int dx = static_cast<int>(threadIdx.x) % 3 - 1, dy = static_cast<int>(threadIdx.x) / 3 - 1;
        const int nx = (rx + dx + RW) % RW, ny = (ry + dy + RH) % RH, nr = ny * RW + nx;
        const unsigned* o = p.in_off + static_cast<size_t>(nr) * 10;
        unsigned lo, hi;
        if (dx == 0 && dy == 0) {
            lo = o[0];
            hi = o[9];
        } else {
            int sb;
            if (dx == 0) sb = dy < 0 ? 5 : 4;
            else if (dy == 0) sb = dx < 0 ? 7 : 6;
            else sb = (dy < 0 ? 2 : 0) + (dx < 0 ? 1 : 0);
            lo = o[sb];
            hi = o[sb + 1];
        }
        s_lo[threadIdx.x] = lo;
        s_len[threadIdx.x] = hi - lo;
    }
    for (int c = threadIdx.x; c < S * S; c += kT) {
        head[c] = 0xFFFFu;
        lowest[c] = 0xFFFFFFFFu;
        s_due[c] = p.due[static_cast<size_t>(reg) * S * S + c];
    }
    __syncthreads();
    unsigned total = 0, pre[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        pre[k] = total;
        total += s_len[k];
    }
    for (unsigned i = threadIdx.x; i < total; i += kT) {
        int k = 0;
#pragma unroll
        for (int q = 1; q < 9; ++q) k += i >= pre[q];
        Rec r = p.in[s_lo[k] + (i - pre[k])];
        const unsigned long long h = mix((static_cast<unsigned long long>(r.slot) << 20) ^ p.salt);
        const int u = static_cast<int>(h >> 61);
        const int x = static_cast<int>(r.cell % W), y = static_cast<int>(r.cell / W);
        const int ddx = static_cast<int>((0x22211000u >> (4 * u)) & 0xF) - 1;  // {-1,-1,-1,0,0,1,1,1}
        const int ddy = static_cast<int>((0x21202010u >> (4 * u)) & 0xF) - 1;  // {-1,0,1,-1,1,-1,0,1}
        const int mx = (x + ddx + W) % W, my = (y + ddy + H) % H;
        if (mx / S != rx || my / S != ry) continue;
        r.cell = static_cast<unsigned>(my * W + mx);
        r.age += 1;
        const unsigned kk = atomicAdd(&s_n, 1u);
        if (kk < kMaxRec) rec[kk] = r;
    }
    __syncthreads();
    const unsigned n = s_n < kMaxRec ? s_n : kMaxRec;
    for (unsigned k = threadIdx.x; k < n; k += kT) {
        const int lc = static_cast<int>((rec[k].cell / W) % S) * S + static_cast<int>(rec[k].cell % W % S);
        const bool sheep = !(rec[k].slot >> 31);
        if (sheep) {
            nxt[k] = static_cast<unsigned short>(atomicExch(&head[lc], k));
            atomicMin(&lowest[lc], rec[k].slot);
        }
    }
    __syncthreads();
    for (unsigned k = threadIdx.x; k < n; k += kT) {
        const int lx = static_cast<int>(rec[k].cell % W % S), ly = static_cast<int>((rec[k].cell / W) % S);
        const int lc = ly * S + lx;
        if (lowest[lc] == rec[k].slot && s_due[lc] <= p.salt) {
            s_due[lc] = p.salt + 30;
            rec[k].energy += 4.0;
        }
        rec[k].energy -= 1.0;
        rec[k].flags = sub_of(lx, ly);
        atomicAdd(&s_cnt[rec[k].flags], 1u);
        if ((mix(rec[k].slot ^ p.salt) & 63) == 0) atomicAdd(&p.tile_cnt[(rec[k].slot >> 10) & 1023], 1u);
    }
    __syncthreads();
    // decoupled lookback over regions (ticket order)
    if (threadIdx.x == 0) s_region = (p.mode & 4) ? blockIdx.x : atomicAdd(p.ticket, 1u);  // output order
    __syncthreads();
    const int tk = static_cast<int>(s_region);
    if (p.mode & 1) {
        if (threadIdx.x == 0) {
            unsigned acc = static_cast<unsigned>(reg) * kMaxRec;
            for (int k = 0; k < 9; ++k) {
                const unsigned c = s_cnt[k];
                s_cnt[k] = acc;
                acc += c;
            }
        }
    } else if (threadIdx.x < 32) {
        unsigned tot = 0;
        for (int k = 0; k < 9; ++k) tot += s_cnt[k];
        const unsigned long long agg = (1ULL << 62) | tot;
        unsigned long long excl = 0;
        if (threadIdx.x == 0) {
            if (tk == 0) {
                atomicExch(&p.status[0], (2ULL << 62) | tot);
            } else {
                atomicExch(&p.status[tk], agg);
            }
        }
        if (tk > 0) {
            int j = tk - 1;
            for (;;) {
                const int q = j - static_cast<int>(threadIdx.x);
                unsigned long long v = q >= 0 ? *(volatile unsigned long long*)&p.status[q] : (2ULL << 62);
                const unsigned flag = static_cast<unsigned>(v >> 62);
                const unsigned invalid = __ballot_sync(0xffffffffu, flag == 0);
                const unsigned incl = __ballot_sync(0xffffffffu, flag == 2);
                // first lane (lowest q offset) that is invalid or inclusive
                const unsigned stop = invalid | incl;
                if (stop == 0) {
                    unsigned long long s = v & ((1ULL << 62) - 1);
                    for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
                    excl += s;
                    j -= 32;
                    continue;
                }
                const int first = __ffs(stop) - 1;
                if ((invalid >> first) & 1u) continue;  // wait (spin)
                unsigned long long s = static_cast<int>(threadIdx.x) <= first ? (v & ((1ULL << 62) - 1)) : 0ULL;
                for (int d = 16; d > 0; d >>= 1) s += __shfl_xor_sync(0xffffffffu, s, d);
                excl += s;
                break;
            }
            if (threadIdx.x == 0) atomicExch(&p.status[tk], (2ULL << 62) | (excl + tot));
        }
        if (threadIdx.x == 0) {
            s_excl = excl;
            unsigned* o = p.out_off + static_cast<size_t>(reg) * 10;
            unsigned acc = static_cast<unsigned>(excl);
            for (int k = 0; k < 9; ++k) {
                o[k] = acc;
                acc += s_cnt[k];
                s_cnt[k] = o[k];
            }
            o[9] = acc;
        }
    }
    __syncthreads();
    if (!(p.mode & 2))
        for (unsigned k = threadIdx.x; k < n; k += kT) {
            const unsigned pos = atomicAdd(&s_cnt[rec[k].flags], 1u);
            p.out[pos] = rec[k];
        }
    for (int c = threadIdx.x; c < S * S; c += kT) p.due[static_cast<size_t>(reg) * S * S + c] = s_due[c];
}

__global__ void k_read(const uint4* q, size_t n, unsigned* sink) {  // leave L2 holding clean lines
    unsigned acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        acc ^= q[i].x;
    if (acc == 0x12345678u) *sink = acc;
}
__global__ void k_flush(uint4* q, size_t n, unsigned s) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        q[i] = make_uint4(s, (unsigned)i, 0, 0);
}

int main() {
    // initial pool: ~95 agents per region (C2: ~360k sheep + ~35k wolves), region order, sub-buckets
    std::vector<std::vector<Rec>> byreg(NREG);
    srand(7);
    const int nagents = 395000;
    for (int a = 0; a < nagents; ++a) {
        Rec r{};
        r.slot = (a < 360000 ? 0u : (1u << 31)) | static_cast<unsigned>(rand() % 524288);
        const int x = rand() % W, y = rand() % H;
        r.cell = static_cast<unsigned>(y * W + x);
        r.energy = 5.0;
        r.id = a;
        byreg[(y / S) * RW + x / S].push_back(r);
    }
    std::vector<Rec> pool;
    std::vector<unsigned> off(static_cast<size_t>(NREG) * 10);
    for (int g = 0; g < NREG; ++g) {
        std::vector<Rec> sb[9];
        for (const Rec& r : byreg[g]) {
            const int lx = static_cast<int>(r.cell % W % S), ly = static_cast<int>((r.cell / W) % S);
            const bool l = lx == 0, rr = lx == S - 1, b = ly == 0, t = ly == S - 1;
            int k = 8;
            if (b && l) k = 0; else if (b && rr) k = 1; else if (t && l) k = 2; else if (t && rr) k = 3;
            else if (b) k = 4; else if (t) k = 5; else if (l) k = 6; else if (rr) k = 7;
            sb[k].push_back(r);
        }
        for (int k = 0; k < 9; ++k) {
            off[static_cast<size_t>(g) * 10 + k] = static_cast<unsigned>(pool.size());
            pool.insert(pool.end(), sb[k].begin(), sb[k].end());
        }
        off[static_cast<size_t>(g) * 10 + 9] = static_cast<unsigned>(pool.size());
    }
    Rec *in, *out;
    unsigned *in_off, *out_off, *due, *ticket, *tile;
    unsigned long long* status;
    uint4* fl;
    const size_t flush_n = (256u << 20) / 16;
    cudaMalloc(&in, 1400000 * sizeof(Rec));
    cudaMalloc(&out, 1400000 * sizeof(Rec));
    cudaMalloc(&in_off, off.size() * 4);
    cudaMalloc(&out_off, off.size() * 4);
    cudaMalloc(&due, static_cast<size_t>(W) * H * 4);
    cudaMalloc(&ticket, 4);
    cudaMalloc(&tile, 4096);
    cudaMalloc(&status, NREG * 8);
    cudaMalloc(&fl, flush_n * 16);
    uint4* fl2;
    cudaMalloc(&fl2, flush_n * 16);
    cudaMemset(fl2, 0, flush_n * 16);
    cudaMemcpy(in, pool.data(), pool.size() * sizeof(Rec), cudaMemcpyHostToDevice);
    cudaMemcpy(in_off, off.data(), off.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(due, 0, static_cast<size_t>(W) * H * 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
  for (int mode = 0; mode < 8; ++mode) {
    float best = 1e9f, sum = 0.f;
    const int reps = 20;
    for (int r = 0; r < reps + 3; ++r) {
        cudaMemset(ticket, 0, 4);
        cudaMemset(status, 0, NREG * 8);
        k_flush<<<148 * 4, 256>>>(fl, flush_n, r);
        k_read<<<148 * 4, 256>>>(fl2, flush_n, tile);
        P p{r % 2 ? out : in, r % 2 ? in : out, r % 2 ? out_off : in_off, r % 2 ? in_off : out_off, due, status,
            ticket, tile, 1000u + r, mode};
        cudaEventRecord(a);
        k_step<<<NREG, kT>>>(p);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        if (r >= 3) {
            best = ms < best ? ms : best;
            sum += ms;
        }
    }
    std::printf("mode %d: min %.2f us mean %.2f us\n", mode, best * 1e3, sum / reps * 1e3);
    if (mode) continue;
    cudaError_t e = cudaGetLastError();
    std::vector<unsigned> o2(off.size());
    cudaMemcpy(o2.data(), (reps + 2) % 2 ? in_off : out_off, o2.size() * 4, cudaMemcpyDeviceToHost);
    std::printf("region skeleton step (4096 CTAs x %d thr, L2 flushed): min %.2f us mean %.2f us; agents after %u (%s)\n",
                kT, best * 1e3, sum / reps * 1e3, o2[static_cast<size_t>(NREG - 1) * 10 + 9], cudaGetErrorString(e));
  }
    return 0;
}
