// Test library: the device functor API (include/abmx_cuda_functors.cuh) on fixed scenarios that
// oracle/ref_functor_cases.cpp runs through the reference's std::function API. The pytest suite
// (tests/test_functors_gpu.py) compares the two bit for bit. Built by `make functor_cases`
// (nvcc, -fmad=false: the reference's x86-64 double math is unfused) into
// build/libabmx_functor_cases.so. TEST INFRASTRUCTURE: not part of the product library.
#include <cstdint>
#include <cstring>
#include <vector>

#include "abmx_cuda_functors.cuh"

using namespace abmx::cuda;

namespace {

// the schema every scenario starts from (ordinal order: state, params, policy_state, policy_params)
AgentSchema rich_schema() {
    AgentSchema s;
    s.state = {FieldInit::const_int("a", 7),           FieldInit::const_real("b", 2.5),
               FieldInit::const_bool("c", true),       FieldInit::uniform_int("d", -5, 9),
               FieldInit::uniform_real("e", 1.5, 4.0), FieldInit::uniform_int_as_real("f", 0, 100)};
    s.params = {FieldInit::uniform_real("p", 0.0, 1.0)};
    s.policy_state = {FieldInit::const_int("ps", 3)};
    s.policy_params = {FieldInit::uniform_int("pp", 0, 1000)};
    return s;
}
enum { A, B, C, D, E, F };  // state field indices
enum { P, PS, PP };          // extra field indices

template <class T>
void dl(T* host, const void* dev, int32_t n) {
    cudaMemcpy(host, dev, static_cast<size_t>(n) * sizeof(T), cudaMemcpyDeviceToHost);
}

// ints [a, d, ps, pp][cap], reals [b, e, f, p][cap], bools c[cap], counters {num_active, next_id}
void export_rich(const DeviceAgents& d, uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages, int64_t* ints,
                 double* reals, uint8_t* bools, int64_t* counters) {
    cudaDeviceSynchronize();
    const int32_t n = d.capacity();
    const abmx_agent_set& r = d.raw();
    dl(active, r.active, n);
    dl(ids, r.ids, n);
    dl(types, r.types, n);
    dl(ages, r.ages, n);
    dl(ints, r.state[A].data, n);
    dl(ints + n, r.state[D].data, n);
    dl(ints + 2 * n, r.extra[PS].data, n);
    dl(ints + 3 * n, r.extra[PP].data, n);
    dl(reals, r.state[B].data, n);
    dl(reals + n, r.state[E].data, n);
    dl(reals + 2 * n, r.state[F].data, n);
    dl(reals + 3 * n, r.extra[P].data, n);
    dl(bools, r.state[C].data, n);
    counters[0] = d.num_active();
    counters[1] = d.next_id();
}

// lifecycle.hpp TransitionFn of the step scenario: reads a NEIGHBOUR slot of the input set, a
// param, the shared input, its age
struct Transition {
    __device__ void operator()(const SlotView& v, const void* shared, const StateWriter& w) const {
        const int i = v.index(), cap = v.set().capacity;
        w.set_int(D, v.state_int(D) + v.set().state_int(D, (i + 1) % cap));
        w.set_real(E, v.state_real(E) * 0.5 + static_cast<const double*>(shared)[0]);
        w.set_real(B, v.state_real(B) + v.param_real(P));
        if (v.active() && v.age() % 2 == 1) w.set_bool(C, !v.state_bool(C));
    }
};

// ApplyFn of test_kernels.cpp:203-217: reads slot 0 of whatever set the kernel exposes
struct PeekFirst {
    __device__ void operator()(const StateWriter& w, const SlotView& v, const RowView& r, int32_t) const {
        w.set_int(0, r.get_int(0) + v.set().state_int(0, 0));
    }
};

// order-dependent apply: reads slot (slot + 7) % cap and the pair index
struct Shifted {
    __device__ void operator()(const StateWriter& w, const SlotView& v, const RowView& r, int32_t k) const {
        w.set_int(0, r.get_int(0) + v.set().state_int(0, (v.index() + 7) % v.set().capacity) + k);
    }
};

struct Positive {  // select_agents predicate
    __device__ bool operator()(const SetView& s, int32_t i) const { return s.active[i] && s.state_int(D, i) > 0; }
};

struct MaskFn {  // set_agents_mask SlotUpdateFn
    __device__ void operator()(const StateWriter& w, const SlotView& v) const {
        w.set_int(D, v.state_int(D) + 10 + v.set().state_int(D, (v.index() + 3) % v.set().capacity));
        w.set_real(E, v.state_real(E) * 2.0);
    }
};

struct Newborn {  // spawn_agents ApplyFn
    __device__ void operator()(const StateWriter& w, const SlotView& v, const RowView& r, int32_t k) const {
        w.set_int(D, r.get_int(0) * 2 + k);
        w.set_real(E, v.state_real(E) + 1.0 + static_cast<double>(v.age()));
    }
};

// a set with one int state column "value" holding `values`, every slot live
DeviceAgents value_set(int32_t cap, const int64_t* values) {
    AgentSchema s;
    s.state = {FieldInit::const_int("value", 0)};
    DeviceAgents d = create_agents(cap, cap, s, 1);
    cudaMemcpy(d.raw().state[0].data, values, static_cast<size_t>(cap) * 8, cudaMemcpyHostToDevice);
    return d;
}

struct Rows {
    DeviceRows r;
    void* buf[2] = {nullptr, nullptr};
    Rows(int32_t m, const int64_t* v, const uint8_t* valid) {
        cudaMalloc(&buf[0], static_cast<size_t>(m > 0 ? m : 1) * 8);
        cudaMalloc(&buf[1], static_cast<size_t>(m > 0 ? m : 1));
        cudaMemcpy(buf[0], v, static_cast<size_t>(m) * 8, cudaMemcpyHostToDevice);
        cudaMemcpy(buf[1], valid, static_cast<size_t>(m), cudaMemcpyHostToDevice);
        r.m = m;
        r.valid = static_cast<const uint8_t*>(buf[1]);
        r.n = 1;
        r.cols[0] = ColumnRef{buf[0], 8};
    }
    ~Rows() {
        cudaFree(buf[0]);
        cudaFree(buf[1]);
    }
};

uint8_t* upload_mask(const uint8_t* h, int32_t n) {
    uint8_t* d = nullptr;
    cudaMalloc(&d, static_cast<size_t>(n > 0 ? n : 1));
    cudaMemcpy(d, h, static_cast<size_t>(n), cudaMemcpyHostToDevice);
    return d;
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return cudaDeviceSynchronize() == cudaSuccess ? 0 : 3;
    } catch (const abmx::cuda::CapacityError&) {
        return 11;
    } catch (const abmx::cuda::DomainError&) {
        return 12;
    } catch (const abmx::cuda::SchemaError&) {
        return 13;
    } catch (...) {
        return 1;
    }
}

}  // namespace

extern "C" {

// create_agents with every FieldInit kind (test_core.cpp:37-82)
int fc_create(int32_t cap, int32_t num_active, uint64_t seed, int64_t type, uint8_t* active, int64_t* ids,
              int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools, int64_t* counters) {
    return guarded([&] {
        DeviceAgents d = create_agents(cap, num_active, rich_schema(), seed, type);
        export_rich(d, active, ids, types, ages, ints, reals, bools, counters);
    });
}

// create, then `steps` x step_agents(Transition, shared = {g}) (test_core.cpp:84-133)
int fc_step(int32_t cap, int32_t num_active, uint64_t seed, int64_t type, int32_t steps, double g, int32_t slot_local,
            uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools,
            int64_t* counters) {
    return guarded([&] {
        DeviceAgents d = create_agents(cap, num_active, rich_schema(), seed, type);
        double* sh = nullptr;
        cudaMalloc(&sh, 8);
        cudaMemcpy(sh, &g, 8, cudaMemcpyHostToDevice);
        for (int t = 0; t < steps; ++t) step_agents(d, Transition{}, sh, true, nullptr, slot_local != 0);
        export_rich(d, active, ids, types, ages, ints, reals, bools, counters);
        cudaFree(sh);
    });
}

// test_kernels.cpp:203-217: out = {sci slot 0, sci slot 1, rm slot 0, rm slot 1}
int fc_peek_first(int64_t* out) {
    return guarded([&] {
        const int64_t vals[2] = {2, 4}, rv[2] = {100, 1000};
        const uint8_t both[2] = {1, 1};
        uint8_t* target = upload_mask(both, 2);
        Rows rows(2, rv, both);
        DeviceAgents s1 = value_set(2, vals), s2 = value_set(2, vals);
        set_agents_sci(s1, target, rows.r, PeekFirst{});
        set_agents_rm(s2, target, rows.r, PeekFirst{});
        cudaDeviceSynchronize();
        dl(out, s1.raw().state[0].data, 2);
        dl(out + 2, s2.raw().state[0].data, 2);
        cudaFree(target);
    });
}

// set_agents_rm (mode 0) / set_agents_sci (mode 1) with the order-dependent Shifted apply
int fc_rm_sci(int32_t mode, int32_t cap, const int64_t* values, const uint8_t* target, int32_t m, const int64_t* rv,
              const uint8_t* valid, int64_t* out) {
    return guarded([&] {
        DeviceAgents s = value_set(cap, values);
        uint8_t* t = upload_mask(target, cap);
        Rows rows(m, rv, valid);
        if (mode == 0)
            set_agents_rm(s, t, rows.r, Shifted{});
        else
            set_agents_sci(s, t, rows.r, Shifted{});
        cudaDeviceSynchronize();
        dl(out, s.raw().state[0].data, cap);
        cudaFree(t);
    });
}

// select_agents(active && d > 0) on the created set; returns the count (or -errors)
int32_t fc_select(int32_t cap, int32_t num_active, uint64_t seed, int32_t* indices) {
    int64_t count = -1;
    const int rc = guarded([&] {
        DeviceAgents d = create_agents(cap, num_active, rich_schema(), seed, 0);
        int32_t* di = nullptr;
        int64_t* dc = nullptr;
        cudaMalloc(&di, static_cast<size_t>(cap > 0 ? cap : 1) * 4);
        cudaMalloc(&dc, 8);
        select_agents(d, Positive{}, di, dc);
        cudaDeviceSynchronize();
        dl(indices, di, cap);
        dl(&count, dc, 1);
        cudaFree(di);
        cudaFree(dc);
    });
    return rc ? -rc : static_cast<int32_t>(count);
}

// set_agents_mask(MaskFn) on the created set
int fc_mask(int32_t cap, int32_t num_active, uint64_t seed, const uint8_t* mask, uint8_t* active, int64_t* ids,
            int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools, int64_t* counters) {
    return guarded([&] {
        DeviceAgents d = create_agents(cap, num_active, rich_schema(), seed, 0);
        uint8_t* dm = upload_mask(mask, cap);
        set_agents_mask(d, dm, MaskFn{});
        export_rich(d, active, ids, types, ages, ints, reals, bools, counters);
        cudaFree(dm);
    });
}

// create, one step, remove_agents(kill), spawn_agents(rows, Newborn) with optional recycling and
// type; spawned_dropped = {spawned, dropped}
int fc_spawn(int32_t cap, int32_t num_active, uint64_t seed, const uint8_t* kill, int32_t m, const int64_t* rv,
             const uint8_t* valid, int32_t recycle, int32_t set_type, int64_t type, uint8_t* active, int64_t* ids,
             int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools, int64_t* counters,
             int64_t* spawned_dropped) {
    return guarded([&] {
        DeviceAgents d = create_agents(cap, num_active, rich_schema(), seed, 1);
        d.set_id_recycling(recycle != 0);
        double* sh = nullptr;
        cudaMalloc(&sh, 8);
        const double g = 0.25;
        cudaMemcpy(sh, &g, 8, cudaMemcpyHostToDevice);
        step_agents(d, Transition{}, sh);
        uint8_t* dk = upload_mask(kill, cap);
        remove_agents(d, dk);
        Rows rows(m, rv, valid);
        int64_t* res = nullptr;
        cudaMalloc(&res, 16);
        spawn_agents(d, rows.r, Newborn{}, set_type != 0, type, res);
        export_rich(d, active, ids, types, ages, ints, reals, bools, counters);
        dl(spawned_dropped, res, 2);
        cudaFree(res);
        cudaFree(dk);
        cudaFree(sh);
    });
}

}  // extern "C"
