"""Predation step on the B200 vs the CPU oracle: bit-exact state after every step.

Mirrors tests/test_predation.cpp and the survey's C1/C2 parity runs."""
import numpy as np
import pytest

from helpers import c1, species_equal, state_hash, tiny

pytestmark = pytest.mark.gpu


def make_pair(abmx, oracle, cfgd, seed):
    cfg = abmx.PredationConfig(**cfgd)
    return abmx.PredationModel(cfg, seed), oracle.pred(cfgd, seed)


def assert_same_state(gpu, orc, what):
    for s in (0, 1):
        species_equal(gpu.export_species(s), orc.export_species(s), f"{what} species {s}")
    gr, gg = gpu.export_world()
    orr, org = orc.export_world()
    assert np.array_equal(gr, orr), what
    assert np.array_equal(gg, org), what


def assert_same_events(ge, oe, what):
    assert ge.grass_eaten == oe["grass_eaten"], what
    assert ge.sheep_eaten_by_wolves == oe["sheep_eaten_by_wolves"], what
    for name in ("sheep", "wolves"):
        g, o = getattr(ge, name), oe[name]
        for k in ("metabolized", "deaths", "births", "births_dropped"):
            assert getattr(g, k) == o[k], (what, name, k, getattr(g, k), o[k])
        for k in ("energy_removed_deaths", "energy_dropped_births"):
            assert getattr(g, k) == o[k], (what, name, k, getattr(g, k), o[k])


def test_init_matches_oracle(abmx, oracle):
    seed = abmx.replica_seeds(7, 1)[0]
    gpu, orc = make_pair(abmx, oracle, c1(), seed)
    assert_same_state(gpu, orc, "init")
    assert state_hash(gpu) == orc.hash(True)


def test_c1_trajectory_bitexact_every_step(abmx, oracle):
    seed = abmx.replica_seeds(7, 1)[0]
    gpu, orc = make_pair(abmx, oracle, c1(), seed)
    for t in range(1, 101):
        gpu.step(t)
        oe = orc.step(t)
        m = gpu.collect_metrics()[0].tolist()
        assert m == orc.metrics(), (t, m, orc.metrics())
        assert_same_events(gpu.last_events(), oe, f"t={t}")
        if t % 10 == 0 or t < 5:
            assert_same_state(gpu, orc, f"t={t}")
    # SURVEY §8c known answers at t=100
    assert gpu.collect_metrics()[0].tolist()[:3] == [715, 61, 4613]


def test_c1_run_metrics_match_survey_known_answers(abmx):
    seed = abmx.replica_seeds(7, 1)[0]
    gpu = abmx.PredationModel(abmx.PredationConfig(**c1()), seed)
    m = gpu.run(1, 100)[0]
    for t, want in ((1, (589, 408, 9414)), (2, (591, 422, 8884)), (3, (589, 433, 8447)),
                    (50, (429, 203, 5891)), (100, (715, 61, 4613))):
        assert tuple(int(v) for v in m[t - 1, :3]) == want, t


def test_run_equals_step_loop(abmx):
    cfg = abmx.PredationConfig(**tiny())
    a = abmx.PredationModel(cfg, 10)
    b = abmx.PredationModel(cfg, 10)
    ma = a.run(1, 40)[0]
    for t in range(1, 41):
        b.step(t)
        assert b.collect_metrics()[0].tolist() == ma[t - 1].astype(np.int64).tolist()
    assert state_hash(a) == state_hash(b)


@pytest.mark.parametrize("seed", [1, 2, 10, 12, 99])
def test_tiny_configs_bitexact(abmx, oracle, seed):
    gpu, orc = make_pair(abmx, oracle, tiny(), seed)
    for t in range(1, 41):
        gpu.step(t)
        oe = orc.step(t)
        assert_same_events(gpu.last_events(), oe, f"seed {seed} t={t}")
        assert_same_state(gpu, orc, f"seed {seed} t={t}")


def test_birth_pairs_match_reference(abmx, reference):
    cfgd = tiny(reproduce_prob_sheep=0.9, reproduce_prob_wolf=0.9)
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfgd), 8)
    ref = reference.pred(cfgd, 8)
    for t in range(1, 7):
        gpu.step(t)
        ref.step(t)
        for s in (0, 1):
            assert gpu.birth_pairs(s) == ref.birth_pairs(s), (t, s)
            st = gpu.export_species(s)
            for parent, child in gpu.birth_pairs(s):
                assert st["x"][child] == st["x"][parent] and st["y"][child] == st["y"][parent]
                assert st["ages"][child] == 0


@pytest.mark.parametrize("case", ["one_cell_two_sheep", "wolf_and_sheep", "two_wolves_one_sheep",
                                  "overflow", "starve", "regrow_zero", "regrow_negative",
                                  "crowded_cell", "empty_world", "no_wolf_capacity",
                                  "no_sheep_capacity", "one_row", "one_column", "full_at_start",
                                  "crowded_multi_tile"])
def test_unit_cases_vs_reference(abmx, reference, case):
    """tests/test_predation.cpp:89-224 setups, compared field-by-field with the reference."""
    cfgd = tiny()
    seed = 5
    if case == "one_cell_two_sheep":
        cfgd = tiny(width=1, height=1, n_sheep0=2, n_wolves0=0, reproduce_prob_sheep=0.0)
    elif case == "wolf_and_sheep":
        cfgd = tiny(width=1, height=1, n_sheep0=1, n_wolves0=1, reproduce_prob_sheep=0.0,
                    reproduce_prob_wolf=0.0)
    elif case == "two_wolves_one_sheep":
        cfgd = tiny(width=1, height=1, n_sheep0=1, n_wolves0=2, reproduce_prob_wolf=0.0)
    elif case == "overflow":
        cfgd = tiny(n_sheep0=8, sheep_capacity=8, n_wolves0=0, reproduce_prob_sheep=1.0)
    elif case == "starve":
        cfgd = tiny(n_sheep0=1, n_wolves0=0, metabolism=2.0)
    elif case == "regrow_zero":
        cfgd = tiny(regrow_delay=0)
    elif case == "regrow_negative":
        cfgd = tiny(regrow_delay=-3)
    elif case == "crowded_cell":
        # long per-cell lists: exercises the pool + heap-sort pairing path
        cfgd = tiny(width=2, height=1, n_sheep0=300, n_wolves0=40, sheep_capacity=400,
                    wolf_capacity=400)
    elif case == "empty_world":  # test_predation.cpp:63-72, 89-103
        cfgd = tiny(n_sheep0=0, n_wolves0=0)
    elif case == "no_wolf_capacity":
        cfgd = tiny(n_wolves0=0, wolf_capacity=0)
    elif case == "no_sheep_capacity":
        cfgd = tiny(n_sheep0=0, sheep_capacity=0)
    elif case == "one_row":
        cfgd = tiny(width=64, height=1, n_sheep0=40, n_wolves0=10)
    elif case == "one_column":
        cfgd = tiny(width=1, height=64, n_sheep0=40, n_wolves0=10)
    elif case == "full_at_start":
        cfgd = tiny(n_sheep0=400, n_wolves0=400, sheep_capacity=400, wolf_capacity=400)
    elif case == "crowded_multi_tile":
        # more slots than cells over several 1024-slot tiles: the sort-based k_cells pairing
        cfgd = tiny(width=30, height=30, n_sheep0=1500, n_wolves0=500, sheep_capacity=2500,
                    wolf_capacity=2500)
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfgd), seed)
    ref = reference.pred(cfgd, seed)
    if case == "overflow":
        for m in (gpu, ref):
            d = m.export_species(0)
            d["energy"] = np.where(d["active"] > 0, 10.0, 0.0)
            m.import_species(0, d)
    if case == "starve":
        for m in (gpu, ref):
            d = m.export_species(0)
            d["energy"][0] = 1.0
            m.import_species(0, d)
            c = cfgd["width"] * cfgd["height"]
            m.import_world(np.zeros(c, np.uint8), np.full(c, 5, np.int64))
    for t in range(1, 16):
        gpu.step(t)
        oe = ref.step(t)
        assert_same_events(gpu.last_events(), oe, f"{case} t={t}")
        assert_same_state(gpu, ref, f"{case} t={t}")


def test_energy_ledger_balances_exactly(abmx):
    """test_predation.cpp:226-239: delta(E) == eats*gain - metab - removed - dropped."""
    cfgd = tiny()
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfgd), 10)
    before = [gpu.export_species(s)["energy"].sum() for s in (0, 1)]
    for t in range(1, 41):
        gpu.step(t)
        ev = gpu.last_events()
        after = [gpu.export_species(s)["energy"].sum() for s in (0, 1)]
        eats = (ev.grass_eaten, ev.sheep_eaten_by_wolves)
        gains = (cfgd["energy_gain_sheep"], cfgd["energy_gain_wolf"])
        for s, sp in enumerate((ev.sheep, ev.wolves)):
            rhs = eats[s] * gains[s] - sp.metabolized * cfgd["metabolism"] - \
                sp.energy_removed_deaths - sp.energy_dropped_births
            assert after[s] - before[s] == rhs, (t, s)
        before = after


def test_capacity_invariance(abmx):
    """C1 with caps 1024 and caps 20000 give identical trajectories."""
    seed = abmx.replica_seeds(7, 1)[0]
    a = abmx.PredationModel(abmx.PredationConfig(**c1()), seed).run(1, 100)
    b = abmx.PredationModel(abmx.PredationConfig(**c1(sheep_capacity=20000, wolf_capacity=20000)),
                            seed).run(1, 100)
    assert np.array_equal(a, b)


def test_batched_replicas_equal_solo_runs(abmx):
    """test_batch.cpp:72-90: a batch of R replicas == R solo models, bitwise."""
    cfg = abmx.PredationConfig(**tiny(width=16, height=16, sheep_capacity=600, wolf_capacity=600))
    seeds = abmx.replica_seeds(3, 6)
    batch = abmx.PredationModel(cfg, seeds).run(1, 15)
    for r, s in enumerate(seeds):
        solo = abmx.PredationModel(cfg, s).run(1, 15)[0]
        assert np.array_equal(batch[r], solo), r


def test_c2_scale_first_steps_bitexact(abmx, oracle):
    """C2 (1M-slot capacity, 2048^2 cells): full state bit-exact after 3 steps."""
    cfgd = c1(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
              sheep_capacity=524288, wolf_capacity=524288)
    seed = abmx.replica_seeds(7, 1)[0]
    gpu, orc = make_pair(abmx, oracle, cfgd, seed)
    for t in range(1, 4):
        gpu.step(t)
        oe = orc.step(t)
        assert gpu.collect_metrics()[0].tolist() == orc.metrics()
        assert_same_events(gpu.last_events(), oe, f"C2 t={t}")
    assert_same_state(gpu, orc, "C2 t=3")


def test_import_rejects_bad_state(abmx):
    m = abmx.PredationModel(abmx.PredationConfig(**tiny()), 1)
    d = m.export_species(0)
    d["num_active"] += 1
    with pytest.raises(abmx.CapacityError):
        m.import_species(0, d)
    d = m.export_species(0)
    d["x"][0] = 99
    with pytest.raises(abmx.DomainError):
        m.import_species(0, d)


def test_create_errors(abmx):
    with pytest.raises(abmx.CapacityError):
        abmx.PredationModel(abmx.PredationConfig(**tiny(n_sheep0=500)), 1)
    with pytest.raises(abmx.DomainError):
        abmx.PredationModel(abmx.PredationConfig(**tiny(regrow_delay=1 << 25)), 1)


# ---------------------------------------------------------------------- golden fixtures
def _golden(name):
    import json
    import os
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name)) as f:
        return json.load(f)


def _run_golden(abmx, tr):
    m = abmx.PredationModel(abmx.PredationConfig(**tr["config"]), tr["seed"])
    assert state_hash(m) == tr["hashes"]["0"]
    for t in range(1, tr["steps"] + 1):
        m.step(t)
        assert m.collect_metrics()[0].tolist() == tr["metrics"][t - 1], t
        ev = m.last_events()
        want = tr["events"][t - 1]
        assert ev.grass_eaten == want["grass_eaten"] and ev.sheep_eaten_by_wolves == want["sheep_eaten_by_wolves"]
        if str(t) in tr["hashes"]:
            assert state_hash(m) == tr["hashes"][str(t)], t


@pytest.mark.parametrize("name", ["c1", "c1_caps20000", "tiny_regrow0", "one_cell", "overflow"])
def test_golden_trajectories_from_reference(abmx, name):
    """Fixtures generated from the unmodified reference (oracle/gen_golden.py)."""
    _run_golden(abmx, _golden("predation.json")[name])


def test_golden_tiny_from_reference(abmx):
    for tr in _golden("predation.json")["tiny"]:
        _run_golden(abmx, tr)


def test_golden_c2_from_reference(abmx):
    _run_golden(abmx, _golden("predation_c2.json")["c2"])


def test_golden_run_batch_from_reference(abmx):
    g = _golden("batch.json")
    for path in (1, 2):
        got, _ = abmx.run_batch(abmx.PredationConfig(**g["config"]), g["master"], g["replicas"],
                                g["steps"], path=path)
        assert np.array_equal(got, np.array(g["metrics"])), path


@pytest.mark.parametrize("cfgname", ["sparse", "crowded"])
def test_timed_per_kernel_path_identical(abmx, oracle, cfgname):
    """bench(per_kernel) launches the kernels directly (not the graph): same states; both the
    list-walk pairing (sparse grid) and the sort-based pairing kernel (crowded grid)."""
    cfgd = tiny(width=40, height=40, n_sheep0=200, n_wolves0=60) if cfgname == "sparse" else tiny()
    seed = abmx.replica_seeds(7, 1)[0]
    gpu, orc = make_pair(abmx, oracle, cfgd, seed)
    ms, got = gpu.bench(1, 30, flush_bytes=0, per_kernel=True)
    for t in range(1, 31):
        orc.step(t)
        assert got[0, t - 1].astype(np.int64).tolist() == orc.metrics(), t
    assert_same_state(gpu, orc, cfgname)
    assert (ms > 0).all()


@pytest.mark.parametrize("delay", [1, 2, 300])
def test_regrow_delays_including_long_ones(abmx, reference, delay):
    """Lazy regrow (due epochs) vs the reference countdown, incl. delays beyond a byte."""
    cfgd = tiny(regrow_delay=delay, width=6, height=6, n_sheep0=40)
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfgd), 17)
    ref = reference.pred(cfgd, 17)
    for t in range(1, 25):
        gpu.step(t)
        ref.step(t)
        assert gpu.collect_metrics()[0].tolist() == ref.metrics(), t
        assert_same_state(gpu, ref, f"delay {delay} t={t}")


def test_world_import_mid_run(abmx, reference):
    """Import a hand-made world after some steps (due epochs rebuilt from counters)."""
    cfgd = tiny()
    gpu = abmx.PredationModel(abmx.PredationConfig(**cfgd), 21)
    ref = reference.pred(cfgd, 21)
    for t in range(1, 6):
        gpu.step(t)
        ref.step(t)
    c = cfgd["width"] * cfgd["height"]
    rng = np.random.default_rng(1)
    regrow = rng.integers(0, 8, c).astype(np.int64)
    ready = (regrow == 0).astype(np.uint8)
    for m in (gpu, ref):
        m.import_world(ready, regrow)
    for t in range(6, 20):
        gpu.step(t)
        ref.step(t)
        assert_same_state(gpu, ref, f"t={t}")
        assert gpu.collect_metrics()[0].tolist() == ref.metrics(), t


def test_per_call_step_paths_agree(abmx):
    """The per-call path (step + collect_metrics: one graph whose k_book publishes the rows and
    a sequence word to mapped memory) agrees with run() for a batch of replicas, including
    switches between the two paths and state reads in between."""
    cfg = abmx.PredationConfig(**tiny(width=16, height=16, sheep_capacity=600, wolf_capacity=600))
    seeds = abmx.replica_seeds(5, 4)
    want = abmx.PredationModel(cfg, seeds).run(1, 30)
    m = abmx.PredationModel(cfg, seeds)
    for t in range(1, 11):
        m.step(t)
        assert np.array_equal(m.collect_metrics(), want[:, t - 1].astype(np.int64)), t
    rows = m.run(11, 10)
    assert np.array_equal(rows, want[:, 10:20])
    assert np.array_equal(m.collect_metrics(), want[:, 19].astype(np.int64))
    for t in range(21, 31):
        m.step(t)
        if t == 25:
            m.export_species(0, replica=2)  # a state read applies the pending births
        assert np.array_equal(m.collect_metrics(), want[:, t - 1].astype(np.int64)), t


@pytest.mark.parametrize("cfgname", ["tiny", "tiny_delay300", "c1", "crowded"])
def test_long_runs_cross_epoch_wraparounds(abmx, oracle, cfgname):
    """700 steps: the 8-bit list tags wrap (255), the cell words are cleared every 128 steps,
    the lowest-slot tags cycle (128) and, with delay 300, due epochs span several clears. Every
    metrics row and the final state equal the oracle; a per-call tail after a run() segment."""
    cfgd = {"tiny": tiny(), "tiny_delay300": tiny(regrow_delay=300),
            "c1": c1(), "crowded": tiny(width=10, height=10, n_sheep0=150, n_wolves0=60,
                                        sheep_capacity=400, wolf_capacity=400)}[cfgname]
    seed = abmx.replica_seeds(9, 1)[0]
    gpu, orc = make_pair(abmx, oracle, cfgd, seed)
    rows = gpu.run(1, 650)[0]
    for t in range(1, 651):
        orc.step(t)
        assert rows[t - 1].astype(np.int64).tolist() == orc.metrics(), (cfgname, t)
    for t in range(651, 701):
        gpu.step(t)
        orc.step(t)
        assert gpu.collect_metrics()[0].tolist() == orc.metrics(), (cfgname, t)
    assert_same_state(gpu, orc, f"{cfgname} t=700")


def test_c1_soak_10000_steps(abmx, oracle):
    """C1 for 10,000 steps in chunks of run() (the cell words cleared 78 times, the 8-bit list
    and lowest-slot tags wrapping dozens of times, the due ring cycling): every metrics row
    and the final state equal the oracle."""
    seed = abmx.replica_seeds(13, 1)[0]
    gpu, orc = make_pair(abmx, oracle, c1(), seed)
    t = 1
    for chunk in (1000, 2500, 37, 3463, 3000):
        rows = gpu.run(t, chunk)[0]
        for q in range(chunk):
            orc.step(t + q)
            assert rows[q].astype(np.int64).tolist() == orc.metrics(), t + q
        t += chunk
    assert t == 10001
    assert_same_state(gpu, orc, "c1 t=10000")


def test_c2_scale_100_steps_both_paths(abmx, oracle):
    """C2 at full size for its 100 steps: 10 per-call steps (events every step),
    then 90 steps in one run(); metrics every step and the full state at the end."""
    cfgd = c1(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
              sheep_capacity=524288, wolf_capacity=524288)
    seed = abmx.replica_seeds(7, 1)[0]
    gpu, orc = make_pair(abmx, oracle, cfgd, seed)
    for t in range(1, 11):
        gpu.step(t)
        oe = orc.step(t)
        assert gpu.collect_metrics()[0].tolist() == orc.metrics(), t
        assert_same_events(gpu.last_events(), oe, f"C2 t={t}")
    rows = gpu.run(11, 90)[0]
    for t in range(11, 101):
        orc.step(t)
        assert rows[t - 11].astype(np.int64).tolist() == orc.metrics(), t
    assert_same_state(gpu, orc, "C2 t=100")


def test_small_engine_after_large_keeps_the_large_one_runnable(abmx):
    """the dynamic shared-memory limit is one setting per kernel; creating a smaller
    engine after a larger one must not lower it below what the larger one launches with."""
    # 7M sheep slots: k_move's tile-count prefix needs ~55 KB of dynamic shared memory, above
    # the 48 KB default; the tiny model needs ~1 KB
    big_cfg = abmx.PredationConfig(**c1(width=1024, height=1024, n_sheep0=200000, n_wolves0=20000,
                                        sheep_capacity=7000000, wolf_capacity=300000))
    big = abmx.PredationModel(big_cfg, 5)
    big.step(1)
    small = abmx.PredationModel(abmx.PredationConfig(**tiny()), 6)
    small.step(1)
    for t in range(2, 5):
        big.step(t)  # would fail with an invalid-argument launch if the limit had shrunk
    fresh = abmx.PredationModel(big_cfg, 5)
    for t in range(1, 5):
        fresh.step(t)
    assert big.collect_metrics().tolist() == fresh.collect_metrics().tolist()
    assert state_hash(big) == state_hash(fresh)
