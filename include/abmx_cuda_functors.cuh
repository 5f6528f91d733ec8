// abmx_cuda_functors.cuh — header-only DEVICE functor API for nvcc users.
//
// The reference passes user code as std::function callbacks (kernels.hpp:62-106,
// lifecycle.hpp:54-86), which cannot cross a C-ABI. Here the same operations take device
// functors (any callable usable in __device__ code, e.g. an __device__ lambda with
// --extended-lambda or a struct with a __device__ operator()), instantiated in the caller's own
// translation unit. The pairing, selection and lifecycle bookkeeping run through the C-ABI of
// libabmx_cuda.so (abmx_cuda.h §4); these templates add the user code on top:
//
//   select_agents<Pred>      kernels.cpp:30-35   pred(SetView, slot) -> stable front compaction
//   set_agents_mask<Fn>      kernels.cpp:155-167 fn(StateWriter&, SlotView) where mask (reads the input)
//   set_agents_rm<Apply>     kernels.cpp:116-134 apply(w, SlotView of the INPUT, RowView, k), parallel
//   set_agents_sci<Apply>    kernels.cpp:136-153 apply(w, SlotView of the RUNNING set, RowView, k), k in order
//   step_agents<Transition>  lifecycle.cpp:87-122 fn(SlotView, shared, w); placeholders -> defaults; age++
//   spawn_agents<Apply>      lifecycle.cpp:144-195 rank-match into free slots; apply writes the state
//   create_agents(schema)    lifecycle.cpp:53-85 every FieldInit kind, the documented RNG schedule
//
// Value semantics: the reference returns a new AgentSet computed from an unchanged input. On the
// device the set is updated in place; operations whose user code may read OTHER slots (RM,
// mask, step, spawn) first snapshot the columns (stream-ordered scratch), so the functor sees
// exactly the input set. Pass `slot_local = true` when the functor reads only its own slot to
// skip the snapshot (the result is then identical and no copy is made).
//
// Fields are addressed by index: resolve names once on the host with DeviceAgents::state_index
// (etc.), which throws SchemaError for unknown names, as the reference's by-name accessors do.
// Columns: Int = int64 (8 B), Real = f64 (8 B), Bool = u8 (1 B).
#pragma once

#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "abmx_cuda.h"
#include "abmx_cuda.hpp"

namespace abmx::cuda {

constexpr int kMaxFields = 16;  // per bundle (state / extra) in a device view

enum class Kind : std::int32_t { Int = 0, Real = 1, Bool = 2 };

// ---------------------------------------------------------------- device views
struct ColumnRef {
    void* data;
    std::int32_t elem_size;
};

// Read-only view of a whole set (the reference's `const AgentSet&`, reachable from a SlotView
// through set()). extra = params, policy_state, policy_params in that order.
struct SetView {
    std::int32_t capacity;
    std::int32_t n_state, n_extra;
    const std::uint8_t* active;
    const std::int64_t* ids;
    const std::int64_t* types;
    const std::int64_t* ages;
    ColumnRef state[kMaxFields];
    ColumnRef extra[kMaxFields];

    __device__ std::int64_t state_int(int f, int slot) const { return static_cast<const std::int64_t*>(state[f].data)[slot]; }
    __device__ double state_real(int f, int slot) const { return static_cast<const double*>(state[f].data)[slot]; }
    __device__ bool state_bool(int f, int slot) const { return static_cast<const std::uint8_t*>(state[f].data)[slot] != 0; }
    __device__ std::int64_t extra_int(int f, int slot) const { return static_cast<const std::int64_t*>(extra[f].data)[slot]; }
    __device__ double extra_real(int f, int slot) const { return static_cast<const double*>(extra[f].data)[slot]; }
    __device__ bool extra_bool(int f, int slot) const { return static_cast<const std::uint8_t*>(extra[f].data)[slot] != 0; }
};

// One slot of a set (agent_set.hpp:84-110).
struct SlotView {
    const SetView* s;
    std::int32_t slot;
    __device__ const SetView& set() const { return *s; }
    __device__ std::int32_t index() const { return slot; }
    __device__ bool active() const { return s->active[slot] != 0; }
    __device__ std::int64_t id() const { return s->ids[slot]; }
    __device__ std::int64_t type() const { return s->types[slot]; }
    __device__ std::int64_t age() const { return s->ages[slot]; }
    __device__ std::int64_t state_int(int f) const { return s->state_int(f, slot); }
    __device__ double state_real(int f) const { return s->state_real(f, slot); }
    __device__ bool state_bool(int f) const { return s->state_bool(f, slot); }
    __device__ std::int64_t param_int(int f) const { return s->extra_int(f, slot); }  // extra bundle index
    __device__ double param_real(int f) const { return s->extra_real(f, slot); }
    __device__ bool param_bool(int f) const { return s->extra_bool(f, slot); }
};

// Writes the state fields of one slot (agent_set.hpp:112-130).
struct StateWriter {
    const ColumnRef* cols;
    std::int32_t slot;
    __device__ void set_int(int f, std::int64_t v) const { static_cast<std::int64_t*>(cols[f].data)[slot] = v; }
    __device__ void set_real(int f, double v) const { static_cast<double*>(cols[f].data)[slot] = v; }
    __device__ void set_bool(int f, bool v) const { static_cast<std::uint8_t*>(cols[f].data)[slot] = v ? 1 : 0; }
};

// One update row (kernels.hpp:24-36).
struct RowView {
    const ColumnRef* cols;
    std::int32_t r;
    __device__ std::int32_t row() const { return r; }
    __device__ std::int64_t get_int(int f) const { return static_cast<const std::int64_t*>(cols[f].data)[r]; }
    __device__ double get_real(int f) const { return static_cast<const double*>(cols[f].data)[r]; }
    __device__ bool get_bool(int f) const { return static_cast<const std::uint8_t*>(cols[f].data)[r] != 0; }
};

// Update rows in device memory (UpdateBatch, kernels.hpp:12-21): m rows, valid mask, columns.
struct DeviceRows {
    std::int32_t m = 0;
    const std::uint8_t* valid = nullptr;
    std::int32_t n = 0;
    ColumnRef cols[kMaxFields] = {};
};

// ---------------------------------------------------------------- host schema (lifecycle.hpp:14-55)
struct FieldInit {
    enum Op : std::int32_t { ConstInt, ConstReal, ConstBool, UniformInt, UniformReal, UniformIntAsReal };
    std::string name;
    Op op;
    std::int64_t ilo = 0, ihi = 0;  // ConstInt value / UniformInt* range [lo, hi)
    double rlo = 0.0, rhi = 0.0;    // ConstReal value / UniformReal range [lo, hi)
    static FieldInit const_int(std::string n, std::int64_t v) { return {std::move(n), ConstInt, v, 0, 0.0, 0.0}; }
    static FieldInit const_real(std::string n, double v) { return {std::move(n), ConstReal, 0, 0, v, 0.0}; }
    static FieldInit const_bool(std::string n, bool v) { return {std::move(n), ConstBool, v ? 1 : 0, 0, 0.0, 0.0}; }
    static FieldInit uniform_int(std::string n, std::int64_t lo, std::int64_t hi) { return {std::move(n), UniformInt, lo, hi, 0.0, 0.0}; }
    static FieldInit uniform_real(std::string n, double lo, double hi) { return {std::move(n), UniformReal, 0, 0, lo, hi}; }
    static FieldInit uniform_int_as_real(std::string n, std::int64_t lo, std::int64_t hi) {
        return {std::move(n), UniformIntAsReal, lo, hi, 0.0, 0.0};
    }
    Kind kind() const { return op == ConstInt || op == UniformInt ? Kind::Int : op == ConstBool ? Kind::Bool : Kind::Real; }
};

struct AgentSchema {
    std::vector<FieldInit> state, params, policy_state, policy_params;
};

namespace detail {

__device__ __forceinline__ std::uint64_t mix64(std::uint64_t z) {  // rng.cpp:12-16
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ std::uint64_t draw(std::uint64_t key, std::uint64_t c) {  // rng.cpp:22-24
    return mix64(key + 0x9E3779B97F4A7C15ULL * (c + 1));
}

// materialize (lifecycle.cpp:11-40) for every slot; reset_slot zeroes the STATE placeholders
// (agent_set.cpp:45-58), the other bundles keep their values
template <int kUnused = 0>
__global__ void k_init_field(void* col, std::int32_t op, std::int64_t ilo, std::int64_t ihi, double rlo, double rhi,
                             std::uint64_t stream, std::int32_t n, std::int32_t zero_from) {
    for (std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const bool zero = i >= zero_from;
        switch (op) {
            case FieldInit::ConstInt: static_cast<std::int64_t*>(col)[i] = zero ? 0 : ilo; break;
            case FieldInit::ConstBool: static_cast<std::uint8_t*>(col)[i] = zero ? 0 : static_cast<std::uint8_t>(ilo != 0); break;
            case FieldInit::ConstReal: static_cast<double*>(col)[i] = zero ? 0.0 : rlo; break;
            case FieldInit::UniformInt:
            case FieldInit::UniformIntAsReal: {  // rng.cpp:30-36: lo + hi64(draw * span)
                const std::uint64_t span = static_cast<std::uint64_t>(ihi - ilo);
                const std::int64_t v = ilo + static_cast<std::int64_t>(__umul64hi(draw(stream, static_cast<std::uint64_t>(i)), span));
                if (op == FieldInit::UniformInt)
                    static_cast<std::int64_t*>(col)[i] = zero ? 0 : v;
                else
                    static_cast<double*>(col)[i] = zero ? 0.0 : static_cast<double>(v);
                break;
            }
            default: {  // UniformReal: lo + (hi - lo) * u01, unfused like the reference's x86-64 build
                const double u = static_cast<double>(draw(stream, static_cast<std::uint64_t>(i)) >> 11) * 0x1.0p-53;
                static_cast<double*>(col)[i] = zero ? 0.0 : __dadd_rn(rlo, __dmul_rn(__dsub_rn(rhi, rlo), u));
            }
        }
    }
}

template <int kUnused = 0>
__global__ void k_init_lifecycle(std::uint8_t* active, std::int64_t* ids, std::int64_t* types, std::int64_t* ages,
                                 std::int64_t* counters, std::int32_t n, std::int32_t num_active, std::int64_t type) {
    for (std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        active[i] = i < num_active;
        ids[i] = i < num_active ? i : 0;
        types[i] = type;
        ages[i] = 0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        counters[0] = num_active;
        counters[1] = num_active;
        counters[2] = 0;
    }
}

template <class Pred>
__global__ void k_select_pred(SetView s, Pred pred, std::uint8_t* mask) {
    for (std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < s.capacity; i += gridDim.x * blockDim.x)
        mask[i] = pred(s, i) ? 1 : 0;
}

template <class Fn>
__global__ void k_mask_fn(SetView in, const std::uint8_t* mask, StateWriter w0, Fn fn) {
    for (std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < in.capacity; i += gridDim.x * blockDim.x) {
        if (!mask[i]) continue;
        StateWriter w = w0;
        w.slot = i;
        fn(w, SlotView{&in, i});
    }
}

// pair k: slot slots[k], row rows[k], k < npairs (device count, reduced from `result`)
template <class Apply>
__global__ void k_pairs_parallel(SetView in, DeviceRows R, const std::int32_t* slots, const std::int32_t* rows,
                                 const std::int64_t* npairs, StateWriter w0, Apply apply) {
    const std::int64_t p = *npairs;
    for (std::int64_t k = blockIdx.x * static_cast<std::int64_t>(blockDim.x) + threadIdx.x; k < p;
         k += static_cast<std::int64_t>(gridDim.x) * blockDim.x) {
        StateWriter w = w0;
        w.slot = slots[k];
        apply(w, SlotView{&in, slots[k]}, RowView{R.cols, rows[k]}, static_cast<std::int32_t>(k));
    }
}

// SCI: one thread walks the pairs in order over the RUNNING set (iteration k sees k' < k)
template <class Apply>
__global__ void k_pairs_sequential(SetView running, DeviceRows R, const std::int32_t* slots, const std::int32_t* rows,
                                   const std::int64_t* npairs, StateWriter w0, Apply apply) {
    if (blockIdx.x != 0 || threadIdx.x != 0) return;
    const std::int64_t p = *npairs;
    for (std::int64_t k = 0; k < p; ++k) {
        StateWriter w = w0;
        w.slot = slots[k];
        apply(w, SlotView{&running, slots[k]}, RowView{R.cols, rows[k]}, static_cast<std::int32_t>(k));
    }
}

template <class Fn>
__global__ void k_step(SetView in, StateWriter w0, Fn fn, const void* shared) {
    for (std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < in.capacity; i += gridDim.x * blockDim.x) {
        StateWriter w = w0;
        w.slot = i;
        fn(SlotView{&in, i}, shared, w);
    }
}

// placeholders back to defaults (the blend of lifecycle.cpp:102-115), age++ on active slots
template <int kUnused = 0>
__global__ void k_step_finish(SetView in, StateWriter w0, std::int64_t* ages, bool increment_age) {
    for (std::int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < in.capacity; i += gridDim.x * blockDim.x) {
        if (!in.active[i]) {
            for (int f = 0; f < in.n_state; ++f) {
                if (in.state[f].elem_size == 8)
                    static_cast<std::int64_t*>(w0.cols[f].data)[i] = 0;
                else if (in.state[f].elem_size == 4)
                    static_cast<std::int32_t*>(w0.cols[f].data)[i] = 0;
                else
                    static_cast<std::uint8_t*>(w0.cols[f].data)[i] = 0;
            }
        } else if (increment_age) {
            ages[i] += 1;
        }
    }
}

inline unsigned grid_for(std::int64_t n) {
    const std::int64_t g = (n + 255) / 256;
    return static_cast<unsigned>(g < 1 ? 1 : (g > 148 * 16 ? 148 * 16 : g));
}

inline void ck(cudaError_t e) {
    if (e != cudaSuccess) throw DeviceError(std::string("CUDA: ") + cudaGetErrorString(e));
}

}  // namespace detail

// ---------------------------------------------------------------- device-resident AgentSet
// Owns the lifecycle arrays and the columns of every bundle (create_agents), or wraps
// caller-owned ones. extra = params, then policy_state, then policy_params.
class DeviceAgents {
public:
    DeviceAgents() = default;
    DeviceAgents(const DeviceAgents&) = delete;
    DeviceAgents& operator=(const DeviceAgents&) = delete;
    DeviceAgents(DeviceAgents&& o) noexcept { *this = std::move(o); }
    DeviceAgents& operator=(DeviceAgents&& o) noexcept {
        std::swap(allocs_, o.allocs_);
        std::swap(raw_, o.raw_);
        std::swap(state_cols_, o.state_cols_);
        std::swap(extra_cols_, o.extra_cols_);
        std::swap(state_names_, o.state_names_);
        std::swap(extra_names_, o.extra_names_);
        std::swap(state_kinds_, o.state_kinds_);
        std::swap(extra_kinds_, o.extra_kinds_);
        raw_.state = state_cols_.data();
        raw_.extra = extra_cols_.data();
        return *this;
    }
    ~DeviceAgents() {
        for (void* p : allocs_) cudaFree(p);
    }

    const abmx_agent_set& raw() const { return raw_; }
    std::int32_t capacity() const { return raw_.capacity; }
    void set_id_recycling(bool on) { raw_.recycle_ids = on ? 1 : 0; }

    std::int32_t state_index(const std::string& name) const { return find(state_names_, name); }
    std::int32_t extra_index(const std::string& name) const { return find(extra_names_, name); }
    Kind state_kind(std::int32_t f) const { return state_kinds_.at(static_cast<std::size_t>(f)); }
    Kind extra_kind(std::int32_t f) const { return extra_kinds_.at(static_cast<std::size_t>(f)); }
    std::int32_t n_state() const { return raw_.n_state; }
    std::int32_t n_extra() const { return raw_.n_extra; }

    SetView view() const {
        SetView v{};
        v.capacity = raw_.capacity;
        v.n_state = raw_.n_state;
        v.n_extra = raw_.n_extra;
        v.active = raw_.active;
        v.ids = raw_.ids;
        v.types = raw_.types;
        v.ages = raw_.ages;
        for (int f = 0; f < raw_.n_state; ++f) v.state[f] = ColumnRef{state_cols_[f].data, state_cols_[f].elem_size};
        for (int f = 0; f < raw_.n_extra; ++f) v.extra[f] = ColumnRef{extra_cols_[f].data, extra_cols_[f].elem_size};
        return v;
    }
    StateWriter writer() const {
        StateWriter w{};
        w.cols = d_state_refs();
        w.slot = 0;
        return w;
    }
    // counters {num_active, next_id} (device -> host, synchronous)
    std::int64_t num_active(void* stream = nullptr) const { return counter(0, stream); }
    std::int64_t next_id(void* stream = nullptr) const { return counter(1, stream); }

    // internal: device-side copy of the state ColumnRefs (StateWriter reads them on the device)
    const ColumnRef* d_state_refs() const { return d_refs_; }

    friend DeviceAgents create_agents(std::int32_t, std::int32_t, const AgentSchema&, std::uint64_t, std::int64_t,
                                      cudaStream_t);

private:
    static std::int32_t find(const std::vector<std::string>& names, const std::string& n) {
        for (std::size_t i = 0; i < names.size(); ++i)
            if (names[i] == n) return static_cast<std::int32_t>(i);
        throw SchemaError("no field named " + n);
    }
    std::int64_t counter(int i, void* stream) const {
        std::int64_t v = 0;
        detail::ck(cudaMemcpyAsync(&v, raw_.counters + i, 8, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
        detail::ck(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
        return v;
    }
    void* alloc(std::size_t bytes) {
        void* p = nullptr;
        detail::ck(cudaMalloc(&p, bytes ? bytes : 16));
        allocs_.push_back(p);
        return p;
    }

    std::vector<void*> allocs_;
    abmx_agent_set raw_{};
    std::vector<abmx_column> state_cols_, extra_cols_;
    std::vector<std::string> state_names_, extra_names_;
    std::vector<Kind> state_kinds_, extra_kinds_;
    ColumnRef* d_refs_ = nullptr;
};

// create_agents (lifecycle.cpp:53-85): capacity slots, the first num_active live (ids
// 0..num_active-1, age 0, type agent_type); every field drawn from
// seed.split(CreateField = 1).split(field ordinal) with the ordinal running over state, params,
// policy_state, policy_params in declaration order; placeholder STATE fields zeroed.
inline DeviceAgents create_agents(std::int32_t capacity, std::int32_t num_active, const AgentSchema& schema,
                                  std::uint64_t seed, std::int64_t agent_type = 0, cudaStream_t stream = nullptr) {
    if (capacity < 0) throw CapacityError("negative capacity");
    if (num_active < 0 || num_active > capacity) throw CapacityError("num_active exceeds capacity");
    DeviceAgents d;
    const std::size_t n = static_cast<std::size_t>(capacity);
    d.raw_.capacity = capacity;
    d.raw_.active = static_cast<std::uint8_t*>(d.alloc(n));
    d.raw_.ids = static_cast<std::int64_t*>(d.alloc(n * 8));
    d.raw_.types = static_cast<std::int64_t*>(d.alloc(n * 8));
    d.raw_.ages = static_cast<std::int64_t*>(d.alloc(n * 8));
    d.raw_.counters = static_cast<std::int64_t*>(d.alloc(3 * 8));
    d.raw_.retired = static_cast<std::int64_t*>(d.alloc(n * 8));
    const std::uint64_t root = split(seed, 1);  // StreamTag::CreateField
    std::uint64_t ordinal = 0;
    const std::vector<FieldInit>* bundles[4] = {&schema.state, &schema.params, &schema.policy_state, &schema.policy_params};
    for (int b = 0; b < 4; ++b) {
        std::vector<std::string> seen;
        for (const FieldInit& f : *bundles[b]) {
            for (const auto& s : seen)
                if (s == f.name) throw SchemaError("duplicate field " + f.name);  // FieldBundle::add
            seen.push_back(f.name);
            if ((f.op == FieldInit::UniformInt || f.op == FieldInit::UniformIntAsReal) && !(f.ilo < f.ihi) && capacity > 0)
                throw DomainError("uniform_int: empty range");  // rng.cpp:30-36
            const Kind k = f.kind();
            const std::int32_t es = k == Kind::Bool ? 1 : 8;
            void* col = d.alloc(n * static_cast<std::size_t>(es));
            if (capacity > 0) {
                detail::k_init_field<0><<<detail::grid_for(capacity), 256, 0, stream>>>(
                    col, f.op, f.ilo, f.ihi, f.rlo, f.rhi, split(root, ordinal), capacity, b == 0 ? num_active : capacity);
                detail::ck(cudaGetLastError());
            }
            ++ordinal;
            (b == 0 ? d.state_cols_ : d.extra_cols_).push_back(abmx_column{col, es, 0});
            (b == 0 ? d.state_names_ : d.extra_names_).push_back(f.name);
            (b == 0 ? d.state_kinds_ : d.extra_kinds_).push_back(k);
        }
    }
    if (d.state_cols_.size() > static_cast<std::size_t>(kMaxFields) || d.extra_cols_.size() > static_cast<std::size_t>(kMaxFields))
        throw SchemaError("more than 16 fields in a bundle of a device functor set");
    d.raw_.n_state = static_cast<std::int32_t>(d.state_cols_.size());
    d.raw_.n_extra = static_cast<std::int32_t>(d.extra_cols_.size());
    d.raw_.state = d.state_cols_.data();
    d.raw_.extra = d.extra_cols_.data();
    detail::k_init_lifecycle<0><<<detail::grid_for(capacity), 256, 0, stream>>>(d.raw_.active, d.raw_.ids, d.raw_.types, d.raw_.ages,
                                                                             d.raw_.counters, capacity, num_active, agent_type);
    detail::ck(cudaGetLastError());
    d.d_refs_ = static_cast<ColumnRef*>(d.alloc(sizeof(ColumnRef) * kMaxFields));
    ColumnRef h[kMaxFields] = {};
    for (int f = 0; f < d.raw_.n_state; ++f) h[f] = ColumnRef{d.state_cols_[f].data, d.state_cols_[f].elem_size};
    detail::ck(cudaMemcpyAsync(d.d_refs_, h, sizeof h, cudaMemcpyHostToDevice, stream));
    detail::ck(cudaStreamSynchronize(stream));  // h is a stack array
    return d;
}

namespace detail {

// Stream-ordered copy of the lifecycle arrays and all columns: the functor's read view of the
// INPUT set while the real columns are written.
class Snapshot {
public:
    Snapshot(const DeviceAgents& d, cudaStream_t st) : st_(st) {
        view_ = d.view();
        const std::size_t n = static_cast<std::size_t>(d.capacity());
        view_.active = static_cast<const std::uint8_t*>(copy(d.raw().active, n));
        view_.ids = static_cast<const std::int64_t*>(copy(d.raw().ids, n * 8));
        view_.types = static_cast<const std::int64_t*>(copy(d.raw().types, n * 8));
        view_.ages = static_cast<const std::int64_t*>(copy(d.raw().ages, n * 8));
        for (int f = 0; f < view_.n_state; ++f)
            view_.state[f].data = copy(view_.state[f].data, n * static_cast<std::size_t>(view_.state[f].elem_size));
        // params / policy columns are never written by these operations: no copy needed
    }
    ~Snapshot() {
        for (void* p : bufs_) cudaFreeAsync(p, st_);
    }
    const SetView& view() const { return view_; }

private:
    void* copy(const void* src, std::size_t bytes) {
        void* p = nullptr;
        ck(cudaMallocAsync(&p, bytes ? bytes : 16, st_));
        bufs_.push_back(p);
        if (bytes) ck(cudaMemcpyAsync(p, src, bytes, cudaMemcpyDeviceToDevice, st_));
        return p;
    }
    cudaStream_t st_;
    SetView view_{};
    std::vector<void*> bufs_;
};

struct PairScratch {
    std::int32_t* slots = nullptr;
    std::int32_t* rows = nullptr;
    std::int64_t* result = nullptr;  // {pairs, valid rows} (set_rm) / {spawned, dropped} (spawn)
    cudaStream_t st;
    PairScratch(std::int64_t cap, std::int64_t m, cudaStream_t s) : st(s) {
        ck(cudaMallocAsync(reinterpret_cast<void**>(&slots), static_cast<std::size_t>(cap > 0 ? cap : 1) * 4, st));
        ck(cudaMallocAsync(reinterpret_cast<void**>(&rows), static_cast<std::size_t>(m > 0 ? m : 1) * 4, st));
        ck(cudaMallocAsync(reinterpret_cast<void**>(&result), 16, st));
    }
    ~PairScratch() {
        cudaFreeAsync(slots, st);
        cudaFreeAsync(rows, st);
        cudaFreeAsync(result, st);
    }
};

// the pairing of set_agents_rm / spawn_agents without any column copy (NULL row columns)
inline std::vector<abmx_column> no_copy(const DeviceAgents& d) {
    return std::vector<abmx_column>(static_cast<std::size_t>(d.n_state() > 0 ? d.n_state() : 1), abmx_column{nullptr, 8, 0});
}

}  // namespace detail

// ---------------------------------------------------------------- operations
// select_agents (kernels.cpp:30-35): indices[0, count) = slots where pred(set, slot) holds,
// ascending, then the others ascending. d_indices: capacity int32, d_count: device int64.
template <class Pred>
void select_agents(const DeviceAgents& d, Pred pred, std::int32_t* d_indices, std::int64_t* d_count,
                   cudaStream_t stream = nullptr) {
    std::uint8_t* mask = nullptr;
    detail::ck(cudaMallocAsync(reinterpret_cast<void**>(&mask), static_cast<std::size_t>(d.capacity() > 0 ? d.capacity() : 1), stream));
    detail::k_select_pred<<<detail::grid_for(d.capacity()), 256, 0, stream>>>(d.view(), pred, mask);
    detail::ck(cudaGetLastError());
    check(abmx_agents_select(mask, d.capacity(), d_indices, d_count, stream));
    detail::ck(cudaFreeAsync(mask, stream));
}

// set_agents_mask (kernels.cpp:155-167): fn(writer of slot i, view of the INPUT slot i) where mask[i]
template <class Fn>
void set_agents_mask(const DeviceAgents& d, const std::uint8_t* d_mask, Fn fn, cudaStream_t stream = nullptr,
                     bool slot_local = false) {
    if (slot_local) {
        detail::k_mask_fn<<<detail::grid_for(d.capacity()), 256, 0, stream>>>(d.view(), d_mask, d.writer(), fn);
        detail::ck(cudaGetLastError());
        return;
    }
    detail::Snapshot in(d, stream);
    detail::k_mask_fn<<<detail::grid_for(d.capacity()), 256, 0, stream>>>(in.view(), d_mask, d.writer(), fn);
    detail::ck(cudaGetLastError());
}

// set_agents_rm (kernels.cpp:116-134): the k-th target slot gets the k-th valid row through
// apply(w, view of the INPUT slot, row, k); every pair runs in parallel
template <class Apply>
void set_agents_rm(const DeviceAgents& d, const std::uint8_t* d_target, const DeviceRows& rows, Apply apply,
                   cudaStream_t stream = nullptr, bool slot_local = false) {
    detail::PairScratch P(d.capacity(), rows.m, stream);
    const auto none = detail::no_copy(d);
    // pairing first: it copies no column, so the snapshot (if any) still equals the input
    check(abmx_agents_set_rm(&d.raw(), d_target, rows.m, rows.valid, none.data(), P.slots, P.rows, P.result, stream));
    const unsigned g = detail::grid_for(d.capacity() < rows.m ? d.capacity() : rows.m);
    if (slot_local) {
        detail::k_pairs_parallel<<<g, 256, 0, stream>>>(d.view(), rows, P.slots, P.rows, P.result, d.writer(), apply);
    } else {
        detail::Snapshot in(d, stream);
        detail::k_pairs_parallel<<<g, 256, 0, stream>>>(in.view(), rows, P.slots, P.rows, P.result, d.writer(), apply);
    }
    detail::ck(cudaGetLastError());
}

// set_agents_sci (kernels.cpp:136-153): r = min(p, q) iterations IN ORDER, iteration k reading the
// running set (it sees the effects of iterations < k). Sequential by definition: one device
// thread walks the pairs (the pairing itself is the parallel selection of the C-ABI).
template <class Apply>
void set_agents_sci(const DeviceAgents& d, const std::uint8_t* d_target, const DeviceRows& rows, Apply apply,
                    cudaStream_t stream = nullptr) {
    detail::PairScratch P(d.capacity(), rows.m, stream);
    const auto none = detail::no_copy(d);
    check(abmx_agents_set_sci(&d.raw(), d_target, rows.m, rows.valid, none.data(), P.slots, P.rows, P.result, stream));
    detail::k_pairs_sequential<<<1, 32, 0, stream>>>(d.view(), rows, P.slots, P.rows, P.result, d.writer(), apply);
    detail::ck(cudaGetLastError());
}

// step_agents (lifecycle.cpp:87-122): fn(view of the INPUT slot, shared, writer) on every slot;
// then placeholder slots' state back to defaults and age += 1 on active slots
template <class Fn>
void step_agents(const DeviceAgents& d, Fn fn, const void* d_shared = nullptr, bool increment_age = true,
                 cudaStream_t stream = nullptr, bool slot_local = false) {
    if (slot_local) {
        detail::k_step<<<detail::grid_for(d.capacity()), 256, 0, stream>>>(d.view(), d.writer(), fn, d_shared);
    } else {
        detail::Snapshot in(d, stream);
        detail::k_step<<<detail::grid_for(d.capacity()), 256, 0, stream>>>(in.view(), d.writer(), fn, d_shared);
    }
    detail::ck(cudaGetLastError());
    detail::k_step_finish<0><<<detail::grid_for(d.capacity()), 256, 0, stream>>>(d.view(), d.writer(), d.raw().ages, increment_age);
    detail::ck(cudaGetLastError());
}

// spawn_agents (lifecycle.cpp:144-195): the k-th free slot receives the k-th valid row; active,
// id (retired stack first when recycling, then next_id++), age 0 and type are set by the C-ABI,
// apply(w, view of the INPUT slot, row, k) writes the state. d_result (nullable, device
// int64[2]) = {spawned, dropped}; d_slots / d_rows (nullable) = pair k.
template <class Apply>
void spawn_agents(const DeviceAgents& d, const DeviceRows& rows, Apply apply, bool set_type = false,
                  std::int64_t agent_type = 0, std::int64_t* d_result = nullptr, cudaStream_t stream = nullptr) {
    detail::PairScratch P(d.capacity(), rows.m, stream);
    const auto none = detail::no_copy(d);
    detail::Snapshot in(d, stream);  // the input view (placeholders) before the lifecycle fields change
    check(abmx_agents_spawn(&d.raw(), rows.m, rows.valid, none.data(), set_type ? 1 : 0, agent_type, P.slots, P.rows,
                            P.result, stream));
    const unsigned g = detail::grid_for(d.capacity() < rows.m ? d.capacity() : rows.m);
    detail::k_pairs_parallel<<<g, 256, 0, stream>>>(in.view(), rows, P.slots, P.rows, P.result, d.writer(), apply);
    detail::ck(cudaGetLastError());
    if (d_result) detail::ck(cudaMemcpyAsync(d_result, P.result, 16, cudaMemcpyDeviceToDevice, stream));
}

// pinned_keys (kernels.cpp:37-50): keys of active slots, +inf / -inf on placeholders
inline void pinned_keys(const DeviceAgents& d, const double* d_keys, bool descending, double* d_out,
                        cudaStream_t stream = nullptr) {
    check(abmx_agents_pinned_keys(d_keys, d.raw().active, d.capacity(), descending ? 1 : 0, d_out, stream));
}

// remove_agents (lifecycle.cpp:124-142) needs no user code: the C-ABI entry, for completeness
inline void remove_agents(const DeviceAgents& d, const std::uint8_t* d_kill, std::int64_t* d_killed = nullptr,
                          cudaStream_t stream = nullptr) {
    check(abmx_agents_remove(&d.raw(), d_kill, d_killed, stream));
}

}  // namespace abmx::cuda
