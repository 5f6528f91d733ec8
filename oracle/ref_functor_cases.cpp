// TEST INFRASTRUCTURE ONLY: the functor-API scenarios of tests/cpp/functor_cases.cu run through
// the UNMODIFIED reference's own std::function API (lifecycle.hpp:54-86, kernels.hpp:62-106),
// linked into oracle/_ref/libabmx_ref.so by oracle/Makefile. Same scenarios, same outputs, so
// tests/test_functors_gpu.py compares the device functors with the reference bit for bit.
#include <cstdint>
#include <cstring>
#include <exception>
#include <vector>

#include "abmx/agent_set.hpp"
#include "abmx/errors.hpp"
#include "abmx/kernels.hpp"
#include "abmx/lifecycle.hpp"
#include "abmx/rng.hpp"

using namespace abmx;

namespace {

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

template <class T>
void put(T* dst, std::span<const T> src) {
    std::memcpy(dst, src.data(), src.size() * sizeof(T));
}

void export_rich(const AgentSet& s, uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages, int64_t* ints,
                 double* reals, uint8_t* bools, int64_t* counters) {
    const size_t n = static_cast<size_t>(s.capacity());
    put(active, s.active());
    put(ids, s.ids());
    put(types, s.types());
    put(ages, s.ages());
    put(ints, s.state().ints("a"));
    put(ints + n, s.state().ints("d"));
    put(ints + 2 * n, s.policy_state().ints("ps"));
    put(ints + 3 * n, s.policy_params().ints("pp"));
    put(reals, s.state().reals("b"));
    put(reals + n, s.state().reals("e"));
    put(reals + 2 * n, s.state().reals("f"));
    put(reals + 3 * n, s.params().reals("p"));
    put(bools, s.state().bools("c"));
    counters[0] = s.num_active();
    counters[1] = s.next_id();
}

const TransitionFn transition = [](const SlotView& v, const FieldBundle* shared, StateWriter& w) {
    const Index i = v.slot(), cap = v.set().capacity();
    w.set_int("d", v.state_int("d") + v.set().state().ints("d")[static_cast<size_t>((i + 1) % cap)]);
    w.set_real("e", v.state_real("e") * 0.5 + shared->reals("g")[0]);
    w.set_real("b", v.state_real("b") + v.param_real("p"));
    if (v.is_active() && v.age() % 2 == 1) w.set_bool("c", !v.state_bool("c"));
};

AgentSet value_set(int32_t cap, const int64_t* values) {
    FieldBundle st(static_cast<size_t>(cap));
    st.add("value", Column::of(std::vector<int64_t>(values, values + cap)));
    AgentSet s(cap, std::move(st), FieldBundle(static_cast<size_t>(cap)));
    for (int32_t i = 0; i < cap; ++i) {
        s.active_mut()[static_cast<size_t>(i)] = 1;
        s.ids_mut()[static_cast<size_t>(i)] = i;
    }
    s.set_num_active(cap);
    s.set_next_id(cap);
    return s;
}

UpdateBatch value_rows(int32_t m, const int64_t* rv, const uint8_t* valid) {
    FieldBundle v(static_cast<size_t>(m));
    v.add("value", Column::of(std::vector<int64_t>(rv, rv + m)));
    return UpdateBatch(std::move(v), Mask(valid, valid + m));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const CapacityError&) {
        return 11;
    } catch (const DomainError&) {
        return 12;
    } catch (const SchemaError&) {
        return 13;
    } catch (const std::exception&) {
        return 1;
    }
}

}  // namespace

extern "C" {

int ref_fc_create(int32_t cap, int32_t num_active, uint64_t seed, int64_t type, uint8_t* active, int64_t* ids,
                  int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools, int64_t* counters) {
    return guarded([&] {
        const AgentSet s = create_agents(cap, num_active, rich_schema(), RngState{seed}, type);
        export_rich(s, active, ids, types, ages, ints, reals, bools, counters);
    });
}

int ref_fc_step(int32_t cap, int32_t num_active, uint64_t seed, int64_t type, int32_t steps, double g, int32_t,
                uint8_t* active, int64_t* ids, int64_t* types, int64_t* ages, int64_t* ints, double* reals,
                uint8_t* bools, int64_t* counters) {
    return guarded([&] {
        AgentSet s = create_agents(cap, num_active, rich_schema(), RngState{seed}, type);
        FieldBundle shared(1);
        shared.add_real("g", g);
        for (int t = 0; t < steps; ++t) s = step_agents(s, transition, &shared);
        export_rich(s, active, ids, types, ages, ints, reals, bools, counters);
    });
}

int ref_fc_peek_first(int64_t* out) {
    return guarded([&] {
        const int64_t vals[2] = {2, 4}, rv[2] = {100, 1000};
        const uint8_t both[2] = {1, 1};
        const AgentSet a = value_set(2, vals);
        const UpdateBatch b = value_rows(2, rv, both);
        const ApplyFn peek_first = [](StateWriter& w, const SlotView& v, const RowView& r, Index) {
            w.set_int("value", r.get_int("value") + v.set().state().ints("value")[0]);
        };
        const AgentSet sci = set_agents_sci(a, std::span<const uint8_t>(both, 2), b, peek_first);
        const AgentSet rm = set_agents_rm(a, std::span<const uint8_t>(both, 2), b, peek_first);
        out[0] = sci.state().ints("value")[0];
        out[1] = sci.state().ints("value")[1];
        out[2] = rm.state().ints("value")[0];
        out[3] = rm.state().ints("value")[1];
    });
}

int ref_fc_rm_sci(int32_t mode, int32_t cap, const int64_t* values, const uint8_t* target, int32_t m,
                  const int64_t* rv, const uint8_t* valid, int64_t* out) {
    return guarded([&] {
        const AgentSet a = value_set(cap, values);
        const UpdateBatch b = value_rows(m, rv, valid);
        const ApplyFn shifted = [](StateWriter& w, const SlotView& v, const RowView& r, Index k) {
            const auto cap2 = v.set().capacity();
            w.set_int("value", r.get_int("value") +
                                   v.set().state().ints("value")[static_cast<size_t>((v.slot() + 7) % cap2)] + k);
        };
        const std::span<const uint8_t> t(target, static_cast<size_t>(cap));
        const AgentSet o = mode == 0 ? set_agents_rm(a, t, b, shifted) : set_agents_sci(a, t, b, shifted);
        put(out, o.state().ints("value"));
    });
}

int32_t ref_fc_select(int32_t cap, int32_t num_active, uint64_t seed, int32_t* indices) {
    int32_t count = -1;
    const int rc = guarded([&] {
        const AgentSet s = create_agents(cap, num_active, rich_schema(), RngState{seed}, 0);
        const SelectionResult r = select_agents(s, [](const AgentSet& set, Index i) {
            return set.active()[static_cast<size_t>(i)] && set.state().ints("d")[static_cast<size_t>(i)] > 0;
        });
        std::memcpy(indices, r.indices.data(), r.indices.size() * 4);
        count = r.count;
    });
    return rc ? -rc : count;
}

int ref_fc_mask(int32_t cap, int32_t num_active, uint64_t seed, const uint8_t* mask, uint8_t* active, int64_t* ids,
                int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools, int64_t* counters) {
    return guarded([&] {
        const AgentSet s = create_agents(cap, num_active, rich_schema(), RngState{seed}, 0);
        const SlotUpdateFn fn = [](StateWriter& w, const SlotView& v) {
            const auto c2 = v.set().capacity();
            w.set_int("d", v.state_int("d") + 10 + v.set().state().ints("d")[static_cast<size_t>((v.slot() + 3) % c2)]);
            w.set_real("e", v.state_real("e") * 2.0);
        };
        const AgentSet o = set_agents_mask(s, std::span<const uint8_t>(mask, static_cast<size_t>(cap)), fn);
        export_rich(o, active, ids, types, ages, ints, reals, bools, counters);
    });
}

int ref_fc_spawn(int32_t cap, int32_t num_active, uint64_t seed, const uint8_t* kill, int32_t m, const int64_t* rv,
                 const uint8_t* valid, int32_t recycle, int32_t set_type, int64_t type, uint8_t* active, int64_t* ids,
                 int64_t* types, int64_t* ages, int64_t* ints, double* reals, uint8_t* bools, int64_t* counters,
                 int64_t* spawned_dropped) {
    return guarded([&] {
        AgentSet s = create_agents(cap, num_active, rich_schema(), RngState{seed}, 1);
        s.set_id_recycling(recycle != 0);
        FieldBundle shared(1);
        shared.add_real("g", 0.25);
        s = step_agents(s, transition, &shared);
        s = remove_agents(s, std::span<const uint8_t>(kill, static_cast<size_t>(cap)));
        FieldBundle v(static_cast<size_t>(m));
        v.add("v", Column::of(std::vector<int64_t>(rv, rv + m)));
        const UpdateBatch b(std::move(v), Mask(valid, valid + m));
        const ApplyFn newborn = [](StateWriter& w, const SlotView& sv, const RowView& r, Index k) {
            w.set_int("d", r.get_int("v") * 2 + k);
            w.set_real("e", sv.state_real("e") + 1.0 + static_cast<double>(sv.age()));
        };
        SpawnOutcome o = set_type ? spawn_agents(s, b, newborn, type) : spawn_agents(s, b, newborn);
        export_rich(o.set, active, ids, types, ages, ints, reals, bools, counters);
        spawned_dropped[0] = o.spawned;
        spawned_dropped[1] = o.dropped;
    });
}

// pinned_keys (kernels.cpp:37-50) on a set whose active mask is given
int ref_pinned_keys(int32_t cap, const uint8_t* active, const double* keys, int32_t descending, double* out) {
    return guarded([&] {
        FieldBundle st(static_cast<size_t>(cap));
        AgentSet s(cap, std::move(st), FieldBundle(static_cast<size_t>(cap)));
        int32_t live = 0;
        for (int32_t i = 0; i < cap; ++i) live += (s.active_mut()[static_cast<size_t>(i)] = active[i] ? 1 : 0);
        s.set_num_active(live);
        const std::vector<double> k = pinned_keys(s, std::span<const double>(keys, static_cast<size_t>(cap)),
                                                  descending ? SortDirection::Descending : SortDirection::Ascending);
        std::memcpy(out, k.data(), k.size() * 8);
    });
}

}  // extern "C"
