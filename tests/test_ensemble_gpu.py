"""Ensemble runner (run_batch) on the B200: SMEM-resident CTA-per-replica kernel and the
batched HBM engine vs the oracle's run_batch, bitwise on every metrics row."""
import numpy as np
import pytest

from helpers import c1, tiny

pytestmark = pytest.mark.gpu


def test_smem_path_fits_c1(abmx):
    assert abmx.smem_fits(abmx.PredationConfig(**c1()))


@pytest.mark.parametrize("path", [1, 2])
def test_c1_ensemble_matches_oracle(abmx, oracle, path):
    K, T = 24, 100
    got, ms = abmx.run_batch(abmx.PredationConfig(**c1()), 7, K, T, path=path)
    want = oracle.run_batch(c1(), 7, K, T)
    assert np.array_equal(got, want)
    assert ms > 0


def test_c1_ensemble_matches_reference_run_batch(abmx, reference):
    K, T = 16, 50
    got, _ = abmx.run_batch(abmx.PredationConfig(**c1()), 99, K, T)
    want, _ = reference.run_batch(c1(), 99, K, T, threads=4)
    assert np.array_equal(got, want)


def test_replica_offsets_shard_cleanly(abmx, oracle):
    """Replica r's seed depends only on (master, r): shards [0,8) + [8,16) == [0,16)."""
    cfg = abmx.PredationConfig(**c1())
    full, _ = abmx.run_batch(cfg, 5, 16, 30)
    a, _ = abmx.run_batch(cfg, 5, 8, 30, begin=0)
    b, _ = abmx.run_batch(cfg, 5, 8, 30, begin=8)
    assert np.array_equal(np.concatenate([a, b]), full)


@pytest.mark.parametrize("cfgd", [
    tiny(), tiny(width=1, height=1, n_sheep0=2, n_wolves0=3), tiny(regrow_delay=0),
    tiny(n_sheep0=8, sheep_capacity=8, reproduce_prob_sheep=1.0),
    c1(sheep_capacity=2000, wolf_capacity=600),
    c1(width=30, height=7, n_sheep0=200, n_wolves0=150, sheep_capacity=3000, wolf_capacity=4000),
    tiny(n_sheep0=0, n_wolves0=0), tiny(n_wolves0=0, wolf_capacity=0),
    tiny(n_sheep0=0, sheep_capacity=0), tiny(width=64, height=1, n_sheep0=40, n_wolves0=10),
    tiny(width=1, height=64, n_sheep0=40, n_wolves0=10), tiny(regrow_delay=-2),
    tiny(regrow_delay=254), tiny(n_sheep0=400, n_wolves0=400, sheep_capacity=400, wolf_capacity=400),
])
def test_smem_path_edge_configs(abmx, oracle, cfgd):
    got, _ = abmx.run_batch(abmx.PredationConfig(**cfgd), 11, 6, 40, path=1)
    want = oracle.run_batch(cfgd, 11, 6, 40)
    assert np.array_equal(got, want)


def test_run_batch_errors(abmx):
    with pytest.raises(abmx.BatchError):
        abmx.run_batch(abmx.PredationConfig(**c1()), 1, 0, 5)
    with pytest.raises(abmx.DomainError):
        abmx.run_batch(abmx.PredationConfig(**c1()), 1, 2, 0)


def test_long_ensemble_run(abmx, oracle):
    """700 steps of C1 replicas in the on-chip kernel (grass countdowns and per-step list
    clears over a long run)."""
    got, _ = abmx.run_batch(abmx.PredationConfig(**c1()), 19, 6, 700, path=1)
    assert np.array_equal(got, oracle.run_batch(c1(), 19, 6, 700))


@pytest.mark.parametrize("delay,gain", [(1, 4.0), (30, 4.0), (60, 8.0), (120, 16.0)])
def test_ensemble_lazy_regrow_past_renormalisation(abmx, oracle, delay, gain):
    """8500 steps of small grids, past the grass-word renormalisation at step 8192
    (ensemble.cu kRenorm): the per-step grass count and populations stay bit-exact."""
    cfg = c1(width=24, height=24, n_sheep0=60, n_wolves0=6, sheep_capacity=512, wolf_capacity=64,
             regrow_delay=delay, energy_gain_sheep=gain)
    got, _ = abmx.run_batch(abmx.PredationConfig(**cfg), 23, 3, 8500, path=1)
    want = oracle.run_batch(cfg, 23, 3, 8500)
    assert want[:, -1, 0].sum() > 0  # sheep survive, so grazing continues to the end
    assert np.array_equal(got, want)


@pytest.mark.parametrize("cfgd,steps,replica", [(c1(), 100, 3), (tiny(), 60, 0),
                                                (c1(regrow_delay=0), 40, 1), (c1(regrow_delay=-2), 40, 2),
                                                (c1(width=24, height=24, n_sheep0=60, n_wolves0=6,
                                                    sheep_capacity=512, wolf_capacity=64,
                                                    energy_gain_sheep=8.0, regrow_delay=60), 8300, 1)])
def test_ensemble_final_state_vs_oracle(abmx, oracle, cfgd, steps, replica):
    """The on-chip kernel's final state of one batch member -- every agent column, next_id,
    num_active, grass_ready and the regrow countdowns (lazy regrow converted back, incl. after
    the renormalisation at step 8192) -- against the oracle's PredationModel of that replica."""
    from helpers import species_equal
    master, count = 31, 4
    sh, wo, ready, regrow = abmx.ensemble_replica_state(abmx.PredationConfig(**cfgd), master, count,
                                                         steps, replica)
    orc = oracle.pred(cfgd, oracle.replica_seed(master, replica))
    for t in range(1, steps + 1):
        orc.step(t)
    for s, got in ((0, sh), (1, wo)):
        want = orc.export_species(s)
        species_equal({k: v for k, v in got.items()}, want, f"species {s}")
    wr, wg = orc.export_world()
    assert np.array_equal(ready, wr) and np.array_equal(regrow, wg)
