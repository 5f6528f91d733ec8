// capi.cu — the extern "C" boundary (include/abmx_cuda.h) over the sm_100a kernels.
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/abmx_cuda.h"
#include "abmx_device.cuh"
#include "abmx_internal.h"
#include "ensemble.h"
#include "predation_engine.h"

namespace abmx_internal {

static std::atomic<unsigned long long> g_launches{0};
static thread_local std::string t_error;

static int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return 0;
    return dev;
}

// SM count of the CURRENT device (cached per device: a process may drive several GPUs)
int num_sms() {
    static std::atomic<int> cache[kMaxDevices] = {};
    const int dev = current_device();
    int n = cache[dev].load(std::memory_order_relaxed);
    if (n > 0) return n;
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
    cache[dev].store(v, std::memory_order_relaxed);
    return v;
}

// The library's scratch memory comes from its OWN stream-ordered pool per device (the device's
// default pool, which other libraries in the process use, is left alone). The pool keeps up to
// kScratchKeep bytes across synchronisations: its default release threshold (0) would hand the
// memory back at every sync and the next call would map it afresh.
constexpr unsigned long long kScratchKeep = 1ULL << 30;
cudaError_t malloc_async(void** p, size_t bytes, cudaStream_t s) {
    static std::mutex mu;
    static cudaMemPool_t pools[kMaxDevices] = {};
    const int dev = current_device();
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lock(mu);
        if (!pools[dev]) {
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            cudaError_t e = cudaMemPoolCreate(&pools[dev], &props);
            if (e != cudaSuccess) {
                pools[dev] = nullptr;
                return e;
            }
            unsigned long long thr = kScratchKeep;
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &thr);
        }
        pool = pools[dev];
    }
    return cudaMallocFromPoolAsync(p, bytes, pool, s);
}

// cudaFuncAttributeMaxDynamicSharedMemorySize is ONE setting per function and device for the
// whole process: engines of different sizes (and host threads) share it. It only ever grows,
// under a lock, so a smaller engine created later never lowers the limit a larger one needs.
cudaError_t raise_dyn_smem(const void* fn, size_t bytes) {
    static std::mutex mu;
    static std::vector<std::pair<std::pair<int, const void*>, size_t>> seen;
    const int dev = current_device();
    std::lock_guard<std::mutex> lock(mu);
    for (auto& e : seen)
        if (e.first.first == dev && e.first.second == fn) {
            if (bytes <= e.second) return cudaSuccess;
            const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
            if (r == cudaSuccess) e.second = bytes;
            return r;
        }
    const cudaError_t r = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes));
    if (r == cudaSuccess) seen.push_back({{dev, fn}, bytes});
    return r;
}
void count_launch(int k) { g_launches.fetch_add(static_cast<unsigned long long>(static_cast<long long>(k))); }
unsigned long long launches() { return g_launches.load(); }
void set_error(const std::string& msg) { t_error = msg; }
const char* last_error() { return t_error.c_str(); }

// Per-thread staging context for the synchronous host-pointer KernelTable entries:
// run_batch worker threads call the table concurrently (batch.cpp:37-80), so every
// thread gets its own stream and growable device buffers.
struct HostCtx {
    cudaStream_t stream = nullptr;
    void* buf[4] = {nullptr, nullptr, nullptr, nullptr};
    size_t cap[4] = {0, 0, 0, 0};
    ~HostCtx() {
        for (void* p : buf)
            if (p) cudaFree(p);
        if (stream) cudaStreamDestroy(stream);
    }
};

// The synchronous KernelTable entries are void (kernels.hpp:15-43 fixes their signatures), so
// a CUDA failure cannot be returned. It is recorded instead: a sticky process-wide code
// (abmx_cuda_table_status) plus the thread's message (abmx_cuda_last_error). The failing call
// leaves its outputs unwritten (count_true returns -1), and later calls keep running.
static std::atomic<int> g_table_status{ABMX_OK};
static bool table_fail(const char* what, cudaError_t e) {
    (void)cudaGetLastError();  // clear a non-sticky error so later calls can proceed
    set_error(std::string("KernelTable: ") + what + ": " + cudaGetErrorString(e));
    int expect = ABMX_OK;
    g_table_status.compare_exchange_strong(expect, ABMX_E_CUDA);
    return false;
}
#define TRY(x)                                          \
    do {                                                \
        cudaError_t e_ = (x);                           \
        if (e_ != cudaSuccess) return table_fail(#x, e_); \
    } while (0)

static HostCtx* host_ctx() {
    static thread_local HostCtx ctx;
    if (!ctx.stream) {
        const cudaError_t e = cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) {
            ctx.stream = nullptr;
            table_fail("cudaStreamCreateWithFlags", e);
            return nullptr;
        }
    }
    return &ctx;
}
static void* host_buf(HostCtx& c, int k, size_t bytes) {
    if (bytes > c.cap[k]) {
        if (c.buf[k]) cudaFree(c.buf[k]);
        c.buf[k] = nullptr;
        c.cap[k] = 0;
        const cudaError_t e = cudaMalloc(&c.buf[k], bytes);
        if (e != cudaSuccess) {
            c.buf[k] = nullptr;
            table_fail("cudaMalloc", e);
            return nullptr;
        }
        c.cap[k] = bytes;
    }
    return c.buf[k];
}

}  // namespace abmx_internal

using namespace abmx_internal;

template <class T, class D>
static bool blend_host(const uint8_t* mask, const T* a, const T* b, T* out, size_t n) {
    if (n == 0) return true;
    HostCtx* c = host_ctx();
    if (!c) return false;
    auto* dm = static_cast<uint8_t*>(host_buf(*c, 0, n));
    auto* da = static_cast<D*>(host_buf(*c, 1, n * sizeof(T)));
    auto* db = static_cast<D*>(host_buf(*c, 2, n * sizeof(T)));
    auto* dout = static_cast<D*>(host_buf(*c, 3, n * sizeof(T)));
    if (!dm || !da || !db || !dout) return false;
    TRY(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, c->stream));
    TRY(cudaMemcpyAsync(da, a, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    TRY(cudaMemcpyAsync(db, b, n * sizeof(T), cudaMemcpyHostToDevice, c->stream));
    TRY(launch_blend<D>(dm, da, db, dout, n, c->stream));
    TRY(cudaMemcpyAsync(out, dout, n * sizeof(T), cudaMemcpyDeviceToHost, c->stream));
    TRY(cudaStreamSynchronize(c->stream));
    return true;
}

static bool rank_scan_host(const uint8_t* mask, int32_t* ranks, size_t n) {
    HostCtx* c = host_ctx();
    if (!c) return false;
    auto* dm = static_cast<uint8_t*>(host_buf(*c, 0, n));
    auto* dr = static_cast<int32_t*>(host_buf(*c, 1, n * 4));
    if (!dm || !dr) return false;
    TRY(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, c->stream));
    TRY(launch_rank_scan(dm, dr, n, c->stream));
    TRY(cudaMemcpyAsync(ranks, dr, n * 4, cudaMemcpyDeviceToHost, c->stream));
    TRY(cudaStreamSynchronize(c->stream));
    return true;
}

static bool count_true_host(const uint8_t* mask, size_t n, unsigned long long* h) {
    HostCtx* c = host_ctx();
    if (!c) return false;
    auto* dm = static_cast<uint8_t*>(host_buf(*c, 0, n));
    auto* dc = static_cast<unsigned long long*>(host_buf(*c, 1, 8));
    if (!dm || !dc) return false;
    TRY(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, c->stream));
    TRY(launch_count_true(dm, n, dc, c->stream));
    TRY(cudaMemcpyAsync(h, dc, 8, cudaMemcpyDeviceToHost, c->stream));
    TRY(cudaStreamSynchronize(c->stream));
    return true;
}

static bool compact_host(const uint8_t* mask, int32_t* out, size_t n) {
    HostCtx* c = host_ctx();
    if (!c) return false;
    auto* dm = static_cast<uint8_t*>(host_buf(*c, 0, n));
    auto* dout = static_cast<int32_t*>(host_buf(*c, 1, n * 4));
    auto* dc = static_cast<unsigned long long*>(host_buf(*c, 2, 8));
    if (!dm || !dout || !dc) return false;
    TRY(cudaMemcpyAsync(dm, mask, n, cudaMemcpyHostToDevice, c->stream));
    TRY(launch_compact_indices(dm, dout, n, dc, c->stream));
    TRY(cudaMemcpyAsync(out, dout, n * 4, cudaMemcpyDeviceToHost, c->stream));
    TRY(cudaStreamSynchronize(c->stream));
    return true;
}

static bool match_host(const int32_t* ra, size_t n, const int32_t* rb, size_t m, int32_t* row_out) {
    HostCtx* c = host_ctx();
    if (!c) return false;
    auto* da = static_cast<int32_t*>(host_buf(*c, 0, n * 4));
    auto* db = static_cast<int32_t*>(host_buf(*c, 1, (m ? m : 1) * 4));
    auto* dout = static_cast<int32_t*>(host_buf(*c, 2, n * 4));
    if (!da || !db || !dout) return false;
    TRY(cudaMemcpyAsync(da, ra, n * 4, cudaMemcpyHostToDevice, c->stream));
    if (m) TRY(cudaMemcpyAsync(db, rb, m * 4, cudaMemcpyHostToDevice, c->stream));
    TRY(launch_match_first_equal(da, n, db, m, dout, c->stream));
    TRY(cudaMemcpyAsync(row_out, dout, n * 4, cudaMemcpyDeviceToHost, c->stream));
    TRY(cudaStreamSynchronize(c->stream));
    return true;
}

extern "C" {

const char* abmx_cuda_last_error(void) { return last_error(); }
const char* abmx_cuda_version(void) { return "abmx-b200 0.1.0 (sm_100a)"; }
uint64_t abmx_fnv1a64(uint64_t h, const void* data, size_t n) {
    const unsigned char* p = static_cast<const unsigned char*>(data);
    for (size_t i = 0; i < n; ++i) h = (h ^ p[i]) * 0x100000001b3ULL;
    return h;
}
uint64_t abmx_cuda_launch_count(void) { return launches(); }

// ---------------------------------------------------------------- 1. KernelTable (host ptrs)
int abmx_cuda_table_status(void) { return g_table_status.load(); }
void abmx_cuda_table_clear_status(void) { g_table_status.store(ABMX_OK); }

void abmx_cuda_rank_scan(const uint8_t* mask, int32_t* ranks, size_t n) {
    if (n) rank_scan_host(mask, ranks, n);
}

int64_t abmx_cuda_count_true(const uint8_t* mask, size_t n) {
    if (n == 0) return 0;
    unsigned long long h = 0;
    return count_true_host(mask, n, &h) ? static_cast<int64_t>(h) : -1;
}

void abmx_cuda_compact_indices(const uint8_t* mask, int32_t* out, size_t n) {
    if (n) compact_host(mask, out, n);
}

void abmx_cuda_match_first_equal(const int32_t* ra, size_t n, const int32_t* rb, size_t m,
                                 int32_t* row_out) {
    if (n) match_host(ra, n, rb, m, row_out);
}

void abmx_cuda_blend_i64(const uint8_t* mask, const int64_t* a, const int64_t* b, int64_t* out, size_t n) {
    blend_host<int64_t, int64_t>(mask, a, b, out, n);
}
void abmx_cuda_blend_f64(const uint8_t* mask, const double* a, const double* b, double* out, size_t n) {
    blend_host<double, unsigned long long>(mask, a, b, out, n);  // bitwise select
}
void abmx_cuda_blend_u8(const uint8_t* mask, const uint8_t* a, const uint8_t* b, uint8_t* out, size_t n) {
    blend_host<uint8_t, uint8_t>(mask, a, b, out, n);
}

static const abmx_kernel_table g_table = {
    "cuda",
    &abmx_cuda_rank_scan,
    &abmx_cuda_count_true,
    &abmx_cuda_compact_indices,
    &abmx_cuda_match_first_equal,
    &abmx_cuda_blend_i64,
    &abmx_cuda_blend_f64,
    &abmx_cuda_blend_u8,
};
const abmx_kernel_table* abmx_cuda_kernel_table(void) { return &g_table; }

// ---------------------------------------------------------------- 2. device variants
static int ret(cudaError_t e) {
    if (e == cudaSuccess) return ABMX_OK;
    set_error(cudaGetErrorString(e));
    return ABMX_E_CUDA;
}
#define STREAM(s) static_cast<cudaStream_t>(s)

int abmx_cuda_rank_scan_async(const uint8_t* d_mask, int32_t* d_ranks, size_t n, void* stream) {
    return ret(launch_rank_scan(d_mask, d_ranks, n, STREAM(stream)));
}
int abmx_cuda_count_true_async(const uint8_t* d_mask, size_t n, int64_t* d_count, void* stream) {
    return ret(launch_count_true(d_mask, n, reinterpret_cast<unsigned long long*>(d_count), STREAM(stream)));
}
int abmx_cuda_compact_indices_async(const uint8_t* d_mask, int32_t* d_out, size_t n, int64_t* d_count,
                                    void* stream) {
    if (!d_count) {
        set_error("d_count is required (it carries the true total between the two passes)");
        return ABMX_E_ARG;
    }
    return ret(launch_compact_indices(d_mask, d_out, n, reinterpret_cast<unsigned long long*>(d_count),
                                      STREAM(stream)));
}
int abmx_cuda_match_first_equal_async(const int32_t* d_ra, size_t n, const int32_t* d_rb, size_t m,
                                      int32_t* d_row_out, void* stream) {
    return ret(launch_match_first_equal(d_ra, n, d_rb, m, d_row_out, STREAM(stream)));
}
int abmx_cuda_blend_i64_async(const uint8_t* d_mask, const int64_t* d_a, const int64_t* d_b, int64_t* d_out,
                              size_t n, void* stream) {
    return ret(launch_blend<int64_t>(d_mask, d_a, d_b, d_out, n, STREAM(stream)));
}
int abmx_cuda_blend_f64_async(const uint8_t* d_mask, const double* d_a, const double* d_b, double* d_out,
                              size_t n, void* stream) {
    return ret(launch_blend<unsigned long long>(d_mask, reinterpret_cast<const unsigned long long*>(d_a),
                                                reinterpret_cast<const unsigned long long*>(d_b),
                                                reinterpret_cast<unsigned long long*>(d_out), n, STREAM(stream)));
}
int abmx_cuda_blend_u8_async(const uint8_t* d_mask, const uint8_t* d_a, const uint8_t* d_b, uint8_t* d_out,
                             size_t n, void* stream) {
    return ret(launch_blend<uint8_t>(d_mask, d_a, d_b, d_out, n, STREAM(stream)));
}

// ---------------------------------------------------------------- 3. predation
struct abmx_predation {
    abmx_pred::Engine eng;
};

#define HANDLE(h)                          \
    if (!(h)) {                            \
        set_error("null predation handle"); \
        return ABMX_E_ARG;                 \
    }

int abmx_predation_create(const abmx_predation_config* cfg, const uint64_t* seeds, int32_t replicas,
                          abmx_predation** out) {
    if (!cfg || !seeds || !out) {
        set_error("null argument");
        return ABMX_E_ARG;
    }
    *out = nullptr;
    auto h = std::make_unique<abmx_predation>();
    const int rc = h->eng.create(*cfg, seeds, replicas);
    if (rc) return rc;
    *out = h.release();
    return ABMX_OK;
}
int abmx_predation_destroy(abmx_predation* h) {
    delete h;
    return ABMX_OK;
}
int abmx_predation_step(abmx_predation* h, int64_t t) {
    HANDLE(h);
    return h->eng.step(t);
}
int abmx_predation_run(abmx_predation* h, int64_t t0, int64_t steps, double* metrics_out) {
    HANDLE(h);
    int rc = h->eng.run_async(t0, steps);
    if (rc || !metrics_out) return rc;
    return h->eng.fetch_run_metrics(metrics_out);
}
int abmx_predation_sync(abmx_predation* h) {
    HANDLE(h);
    return ret(cudaStreamSynchronize(h->eng.stream));
}
int abmx_predation_metrics(abmx_predation* h, int64_t* out) {
    HANDLE(h);
    return h->eng.last_metrics(reinterpret_cast<long long*>(out));
}
int abmx_predation_last_events(abmx_predation* h, abmx_predation_events* out) {
    HANDLE(h);
    return h->eng.last_events(out);
}
int32_t abmx_predation_birth_pairs(abmx_predation* h, int32_t replica, int32_t species, int32_t* parent,
                                   int32_t* child, int32_t cap) {
    if (!h || replica < 0 || replica >= h->eng.R || species < 0 || species > 1) return -1;
    return h->eng.birth_pairs(replica, species, parent, child, cap);
}

static int check_rs(abmx_predation* h, int32_t r, int32_t s) {
    if (!h) {
        set_error("null predation handle");
        return ABMX_E_ARG;
    }
    if (r < 0 || r >= h->eng.R || s < 0 || s > 1) {
        set_error("replica or species out of range");
        return ABMX_E_DOMAIN;
    }
    return ABMX_OK;
}

int abmx_predation_export(abmx_predation* h, int32_t replica, int32_t species, uint8_t* active, int64_t* ids,
                          int64_t* types, int64_t* ages, int64_t* x, int64_t* y, double* energy,
                          int32_t* num_active, int64_t* next_id) {
    if (int rc = check_rs(h, replica, species)) return rc;
    return h->eng.export_species(replica, species, active, ids, types, ages, x, y, energy, num_active, next_id);
}
int abmx_predation_import(abmx_predation* h, int32_t replica, int32_t species, const uint8_t* active,
                          const int64_t* ids, const int64_t* ages, const int64_t* x, const int64_t* y,
                          const double* energy, int32_t num_active, int64_t next_id) {
    if (int rc = check_rs(h, replica, species)) return rc;
    return h->eng.import_species(replica, species, active, ids, ages, x, y, energy, num_active, next_id);
}
int abmx_predation_export_world(abmx_predation* h, int32_t replica, uint8_t* grass_ready, int64_t* regrow) {
    if (int rc = check_rs(h, replica, 0)) return rc;
    return h->eng.export_world(replica, grass_ready, regrow);
}
int abmx_predation_import_world(abmx_predation* h, int32_t replica, const uint8_t* grass_ready,
                                const int64_t* regrow) {
    if (int rc = check_rs(h, replica, 0)) return rc;
    return h->eng.import_world(replica, grass_ready, regrow);
}
void* abmx_predation_stream(abmx_predation* h) { return h ? h->eng.stream : nullptr; }
int abmx_predation_set_timing(abmx_predation* h, int enabled) {
    HANDLE(h);
    (void)enabled;  // per-kernel timing is taken by abmx_predation_bench(per_kernel = 1)
    for (int k = 0; k < abmx_pred::kNumKernels; ++k) {
        h->eng.kernel_ms[k] = 0.0;
        h->eng.kernel_launches[k] = 0;
    }
    return ABMX_OK;
}
int32_t abmx_predation_kernel_count(void) { return abmx_pred::kNumKernels; }
const char* abmx_predation_kernel_name(int32_t k) { return abmx_pred::kernel_name(k); }
// Phase timeline of the next launches (ABMX_PRED_TRACE builds; elsewhere the buffer stays
// zero). enable = 1 allocates [2 kernels][CTAs][8] stamps.
int abmx_predation_set_trace(abmx_predation* h, int32_t enable) {
    HANDLE(h);
    auto& E = h->eng;
    if (enable && !E.d_trace) {
        E.trace_n = static_cast<size_t>(2) * E.grid(0) * 8;
        if (cudaMalloc(&E.d_trace, E.trace_n * 8) != cudaSuccess) return ABMX_E_CUDA;
        cudaMemset(E.d_trace, 0, E.trace_n * 8);
    }
    E.params.trace = enable ? E.d_trace : nullptr;
    if (E.graph_exec) {  // graph nodes captured the old parameter block: rebuild on next use
        cudaGraphExecDestroy(E.graph_exec);
        cudaGraphDestroy(E.graph);
        E.graph_exec = nullptr;
        E.graph = nullptr;
    }
    return ABMX_OK;
}
int64_t abmx_predation_trace(abmx_predation* h, uint64_t* out, int64_t cap) {
    if (!h || !h->eng.d_trace) return 0;
    const size_t n = h->eng.trace_n < static_cast<size_t>(cap) ? h->eng.trace_n : static_cast<size_t>(cap);
    cudaStreamSynchronize(h->eng.stream);
    cudaMemcpy(out, h->eng.d_trace, n * 8, cudaMemcpyDeviceToHost);
    return static_cast<int64_t>(n);
}
int abmx_predation_kernel_times(abmx_predation* h, double* ms, int64_t* launches_out) {
    HANDLE(h);
    for (int k = 0; k < abmx_pred::kNumKernels; ++k) {
        ms[k] = h->eng.kernel_ms[k];
        launches_out[k] = h->eng.kernel_launches[k];
    }
    return ABMX_OK;
}
int abmx_predation_check_status(void) { return abmx_pred::check_status(); }
int64_t abmx_predation_device_bytes(abmx_predation* h) { return h ? h->eng.device_bytes : 0; }
int abmx_predation_bench(abmx_predation* h, int64_t t0, int64_t steps, int64_t flush_bytes, int32_t per_kernel,
                         double* step_ms) {
    HANDLE(h);
    if (!step_ms || flush_bytes < 0) {
        set_error("step_ms required; flush_bytes >= 0");
        return ABMX_E_ARG;
    }
    return h->eng.bench(t0, steps, static_cast<size_t>(flush_bytes), per_kernel != 0, step_ms);
}
int abmx_predation_fetch_metrics(abmx_predation* h, double* out) {
    HANDLE(h);
    return h->eng.fetch_run_metrics(out);
}

// ---------------------------------------------------------------- ensemble
int abmx_ensemble_smem_fits(const abmx_predation_config* cfg) {
    return cfg && abmx_ens::smem_fits(*cfg) ? 1 : 0;
}

int abmx_ensemble_replica_state(const abmx_predation_config* cfg, uint64_t master, int32_t replica_begin,
                                int32_t count, int64_t steps, int32_t replica, abmx_species_arrays* sheep,
                                abmx_species_arrays* wolves, uint8_t* grass_ready, int64_t* regrow) {
    if (!cfg || !sheep || !wolves || !grass_ready || !regrow) {
        set_error("null argument");
        return ABMX_E_ARG;
    }
    if (count < 1) {
        set_error("batch needs at least one replica");  // batch.cpp:24-25
        return ABMX_E_BATCH;
    }
    if (steps < 1 || replica < 0 || replica >= count) {
        set_error("steps must be >= 1 and replica inside the batch");
        return ABMX_E_DOMAIN;
    }
    if (!abmx_ens::smem_fits(*cfg)) {
        set_error("configuration does not fit the SMEM-resident ensemble kernel");
        return ABMX_E_DOMAIN;
    }
    std::vector<uint64_t> seeds(static_cast<size_t>(count));
    const unsigned long long root = abmx_dev::split(master, 2);  // batch.cpp:12-19
    for (int32_t k = 0; k < count; ++k)
        seeds[static_cast<size_t>(k)] = abmx_dev::split(root, static_cast<unsigned long long>(replica_begin + k));
    abmx_ens::Dump d{};
    d.replica = replica;
    abmx_species_arrays* sp[2] = {sheep, wolves};
    for (int s = 0; s < 2; ++s) {
        d.active[s] = sp[s]->active;
        d.ids[s] = sp[s]->ids;
        d.ages[s] = sp[s]->ages;
        d.x[s] = sp[s]->x;
        d.y[s] = sp[s]->y;
        d.energy[s] = sp[s]->energy;
    }
    d.grass_ready = grass_ready;
    d.regrow = regrow;
    const int rc = abmx_ens::run_smem(*cfg, seeds.data(), count, steps, nullptr, nullptr, &d);
    if (rc) return rc;
    for (int s = 0; s < 2; ++s) {
        sp[s]->num_active = d.num_active[s];
        sp[s]->next_id = d.next_id[s];
    }
    return ABMX_OK;
}

int abmx_ensemble_run(const abmx_predation_config* cfg, uint64_t master, int32_t replica_begin, int32_t count,
                      int64_t steps, int32_t path, double* metrics_out, double* kernel_ms) {
    if (!cfg) {
        set_error("null config");
        return ABMX_E_ARG;
    }
    if (count < 1) {
        set_error("batch needs at least one replica");  // batch.cpp:24-25
        return ABMX_E_BATCH;
    }
    if (steps < 1) {
        set_error("steps must be >= 1");  // batch.cpp:26-27
        return ABMX_E_DOMAIN;
    }
    std::vector<uint64_t> seeds(static_cast<size_t>(count));
    const unsigned long long root = abmx_dev::split(master, 2);
    for (int32_t k = 0; k < count; ++k)
        seeds[static_cast<size_t>(k)] = abmx_dev::split(root, static_cast<unsigned long long>(replica_begin + k));
    const bool smem = abmx_ens::smem_fits(*cfg);
    if (path == 1 && !smem) {
        set_error("configuration does not fit the SMEM-resident ensemble kernel");
        return ABMX_E_DOMAIN;
    }
    if ((path == 0 && smem) || path == 1)
        return abmx_ens::run_smem(*cfg, seeds.data(), count, steps, metrics_out, kernel_ms);
    // batched HBM engine
    abmx_pred::Engine eng;
    int rc = eng.create(*cfg, seeds.data(), count);
    if (rc) return rc;
    if (steps > 0x7FFFFFFFLL) return eng.run_async(1, steps);  // reports the domain error
    rc = eng.reserve_run(steps);  // allocate outside the timed region
    if (rc) return rc;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, eng.stream);
    rc = eng.run_async(1, steps);
    cudaEventRecord(b, eng.stream);
    if (rc) return rc;
    if (metrics_out) {
        rc = eng.fetch_run_metrics(metrics_out);
    } else {
        rc = ret(cudaStreamSynchronize(eng.stream));
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    if (kernel_ms) *kernel_ms = ms;
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return rc;
}

}  // extern "C"
