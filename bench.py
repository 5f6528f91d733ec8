#!/usr/bin/env python
"""bench.py — predation hot path on B200: agent-steps/sec and % of the HBM roofline.

Workload (BASELINE.json configs[1], SURVEY §8d "C2"): ONE predation model at 1M-agent
capacity per GPU — 2048 x 2048 cells, 300,000 sheep + 30,000 wolves initially, capacities
524,288 + 524,288 — heavy birth/death churn every step. A "step" is one full
step_predation (move, graze, predation, metabolise, starve, reproduce + spawn, regrow).
Under torchrun each rank runs its own replica (seed master.split(2).split(rank)): weak
scaling, no data-path collective; the per-rank summary rows are gathered with NCCL.
The line also carries the C3 ensemble (4096 x C1 replicas, sharded over the ranks).

  value      capacity slot-steps/s over all ranks, device-timed (CUDA events per step,
             L2 flushed before every timed step: an untimed 256 MiB write, then a 256 MiB read
             so L2 holds clean lines), max over ranks
  e2e        the same metric through the C-ABI call a user makes: abmx_predation_step(t)
             (H2D of t) + abmx_predation_metrics (D2H of the metrics row), host wall clock
  roofline   dominant kernel: SURVEY §8d algorithmic bytes apportioned to that kernel
             / its CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs; plus
             random_access_cost: the step's random cell-word atomics / reads alone and the
             bare launch shape, event-timed (the bound; profiles/r02_c2_cost_model.md), and
             step_dram_bytes_in_step: one ncu range over k_move + k_update (profiles/)
  cpu_baseline  the reference's own C++ step_predation (oracle/_ref, -O3) on this host
  ensemble / traffic / finance   secondary sections: device times of
             the C3 ensemble, the C4 road and roads variant, the C5 markets (and the one-market
             reading), each with the reference's own CPU run on a bounded sample
  agents     the generic lifecycle (remove_agents + spawn_agents) on a
             C2-sized set, bit-compared with the reference's own remove/spawn on the same inputs
  kernel_table  the KernelTable device entries (rank_scan, count_true, compact_indices,
             match_first_equal, blend_i64) on 2^26 elements, L2 flushed, event-timed

`--impl reference` times the reference CPU implementation (oracle/_ref) on the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MASTER_SEED = 7
C2 = dict(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000, sheep_capacity=524288,
          wolf_capacity=524288, energy_gain_sheep=4.0, energy_gain_wolf=20.0, metabolism=1.0,
          reproduce_prob_sheep=0.04, reproduce_prob_wolf=0.05, reproduce_energy_frac=0.5,
          regrow_delay=30)
C1 = dict(C2, width=100, height=100, n_sheep0=600, n_wolves0=400, sheep_capacity=1024,
          wolf_capacity=1024)
ENSEMBLE_REPLICAS = 4096
ENSEMBLE_STEPS = 100
FLUSH_BYTES = 256 << 20  # > 126 MB L2 (written, then a second buffer read: L2 left clean)
METRIC = "agent-steps/sec"
UNIT = "slot-steps/s"
WORKLOAD = ("C2 predation: 2048x2048 cells, 300k sheep + 30k wolves, capacity 524288 + 524288 "
            "(1,048,576 slots) per GPU; one model per rank")


def capacity(cfg):
    return cfg["sheep_capacity"] + cfg["wolf_capacity"]


def hbm_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = str(gpu_index)
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", self.gpu, f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        time.sleep(0.2)
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() in ("active", "1"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------- reference arm
def bench_config():
    """The `config` of BOTH arms' JSON lines (identical, so the driver can pair them)."""
    return {"workload": WORKLOAD, "replicas_per_gpu": 1, "seed": MASTER_SEED,
            "l2": "GPU arm: L2 flushed before every timed step (untimed 256 MiB write, then 256 MiB "
                  "read); reference arm: host CPU, no flush"}


def reference_arm(args, world):
    """The reference's own CPU implementation (oracle/_ref: the unmodified abmx sources,
    -O3) on this host, same metric/config; rank 0 only."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import pyoracle
    if not os.path.exists(pyoracle.REF_SO):
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libabmx_ref.so not built"}))
        return
    ref = pyoracle.Reference()
    cores = os.cpu_count() or 1
    K, W = args.steps, args.warmup
    if world == 1:
        # one model: the reference steps a single model on one thread by design
        seed = ref.replica_seed(MASTER_SEED, 0)
        m = ref.pred(C2, seed)
        m.run(1, W)
        ms = m.run(W + 1, K)
        threads = 1
        sample = f"C2 model, steps {W + 1}..{W + K} after {W} warm-up steps, 1 thread"
    else:
        # N replicas (one per rank in our arm) on run_batch threads; warmup-subtraction protocol
        threads = min(world, cores)
        _, a = ref.run_batch(C2, MASTER_SEED, world, W + K, threads=threads)
        _, b = ref.run_batch(C2, MASTER_SEED, world, W, threads=threads)
        ms = a - b
        sample = (f"{world} C2 replicas via run_batch on {threads} threads, wall({W + K} steps) - "
                  f"wall({W} steps)")
    value = world * capacity(C2) * K / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": K, "warmup": W, "ms_per_step": ms / K, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64+int", "data": "synthetic",
            "config": bench_config(),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))



# ---------------------------------------------------------------------- traffic (§8f rank 1)
TRAFFIC_L = 349_526          # C4: one road, capacity 3L = 1,048,578 slots
ROADS, ROADS_L, ROADS_STEPS = 3496, 100, 1000  # C4 roads variant (paper Table 3 shape)


def golden_fnv(name):
    """FNV-1a of the reference's own rows for a sharded workload (tests/golden/bench.json,
    written by oracle/gen_bench_golden.py from the unmodified reference)."""
    with open(os.path.join(ROOT, "tests", "golden", "bench.json")) as f:
        return json.load(f)[name]["rows_fnv"]


def gather_check(name, rows, rank, dist, device):
    """one all-gather of the per-replica metrics rows (sharding.gather_rows, replica
    order), then rank 0 checks the FNV-1a of the whole gathered block against the reference's
    (single-process run: the local rows are the whole block). Returns (rows gathered, ok)."""
    from paper_2508_16508_b200.sharding import gather_rows, rows_fnv
    full = gather_rows(rows, dist, device=device) if dist is not None else rows
    ok = None
    if rank == 0:
        ok = rows_fnv([full]) == golden_fnv(name)
        if not ok:
            raise RuntimeError(f"{name}: gathered rows differ from the reference's (FNV)")
    return int(full.shape[0]), ok


def traffic_roads(args, rank, world, allreduce, dist):
    """C4 roads variant (3496 x L=100, 1000 steps) sharded by contiguous road blocks; one
    all-gather of the metrics rows, checked on rank 0 against the reference's FNV."""
    from paper_2508_16508_b200 import traffic as T
    from paper_2508_16508_b200.sharding import shard_range
    begin, count = shard_range(ROADS, world, rank)
    T.run_batch(T.TrafficConfig(ROADS_L, 10, 0.5), MASTER_SEED, count, ROADS_STEPS, begin=begin)
    rows_r, rk = T.run_batch(T.TrafficConfig(ROADS_L, 10, 0.5), MASTER_SEED, count, ROADS_STEPS,
                             begin=begin)
    gathered, fnv_ok = gather_check("C4_roads", rows_r, rank, dist, args.gather_device)
    rk = allreduce(rk, dist.ReduceOp.MAX if dist else None)
    return {"workload": f"{ROADS} roads x L={ROADS_L}, {ROADS_STEPS} steps (run_batch)",
            "rows_gathered": gathered, "rows_match_reference": fnv_ok,
            "value": ROADS * 3 * ROADS_L * ROADS_STEPS / (rk / 1e3), "unit": UNIT,
            "device_ms": rk}


def traffic_section(args, rank, world, allreduce, dist):
    """C4 on the device: one long road per rank (device-timed steps, L2 flushed), the roads
    variant sharded by contiguous road blocks, and the reference CPU on bounded samples."""
    import numpy as np
    import paper_2508_16508_b200 as abmx
    from paper_2508_16508_b200 import traffic as T
    K, W = args.steps, args.warmup
    seed = abmx.replica_seeds(MASTER_SEED, world)[rank]
    m = T.TrafficModel(T.TrafficConfig(TRAFFIC_L, 10, 0.5), seed)
    m.bench(1, W, FLUSH_BYTES)
    step_ms = m.bench(W + 1, K, FLUSH_BYTES)
    tot = allreduce(float(np.sum(step_ms)), dist.ReduceOp.MAX if dist else None)
    m.bench(W + K + 1, max(3, min(K, 10)), FLUSH_BYTES, per_kernel=True)
    kt = {k: v[0] / max(v[1], 1) for k, v in m.kernel_times().items()}
    m.close()
    cap = 3 * TRAFFIC_L
    alg = 26 * cap  # 2N(lane 4 + cell 4 + active 1) + 2(3L)(occupancy 4)
    roads = traffic_roads(args, rank, world, allreduce, dist)
    out = {"workload": f"C4: one road L={TRAFFIC_L} (capacity {cap} slots) per GPU, period 10, "
                       f"green 0.5, seed {MASTER_SEED}",
           "value": world * cap * K / (tot / 1e3), "unit": UNIT, "ms_per_step": tot / K,
           "per_kernel_ms": kt,
           "step_effective_gbs": alg / (tot / K / 1e3) / 1e9,
           "roads": roads}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        if os.path.exists(pyoracle.REF_SO):
            ref = pyoracle.Reference()
            r = ref.traffic(TRAFFIC_L, 10, 0.5, seed)
            n = 20
            wall = r.run(1, n)
            out["cpu_baseline"] = {"value": cap * n / (wall / 1e3), "unit": UNIT, "cores": 1,
                                   "kind": "reference",
                                   "sample": f"reference TrafficModel::step, C4 steps 1..{n}, "
                                             f"1 thread ({wall / 1e3:.1f} s)"}
            threads = os.cpu_count() or 1
            ns = 300
            _, wall_b = ref.traffic_run_batch(ROADS_L, 10, 0.5, MASTER_SEED, ROADS, ns,
                                              threads=threads)
            out["roads"]["cpu_baseline"] = {
                "value": ROADS * 3 * ROADS_L * ns / (wall_b / 1e3), "unit": UNIT, "cores": threads,
                "kind": "reference",
                "sample": f"reference run_batch(TrafficModel), {ROADS} roads x {ns} steps, "
                          f"{threads} threads ({wall_b / 1e3:.1f} s)"}
    return out


# ---------------------------------------------------------------------- finance (§8f rank 2)
MARKETS, FIN_STEPS = 1024, 100  # C5: 1024 markets x default FinanceConfig, 100 steps


def finance_section(args, rank, world, allreduce, dist):
    """C5 on the device (markets sharded by contiguous blocks over the ranks) and the reference
    run_batch on the host for a bounded sample."""
    from paper_2508_16508_b200 import finance as F
    cfg = F.FinanceConfig()
    from paper_2508_16508_b200.sharding import shard_range
    begin, count = shard_range(MARKETS, world, rank)
    for _ in range(2):  # full-size warm-up runs (clocks, allocator, shared-memory carve-out)
        F.run_batch(cfg, MASTER_SEED, count, FIN_STEPS, begin=begin)
    res = [F.run_batch(cfg, MASTER_SEED, count, FIN_STEPS, begin=begin) for _ in range(3)]
    ms = allreduce(statistics.median([r[1] for r in res]), dist.ReduceOp.MAX if dist else None)
    r0 = res[0][0]
    gathered, fnv_ok = gather_check("C5", r0.reshape(r0.shape[0], r0.shape[1], -1), rank, dist,
                                    args.gather_device)
    slots = MARKETS * cfg.books * cfg.book_capacity
    out = {"workload": f"C5: {MARKETS} markets x FinanceConfig defaults (5 books x 1000 capacity, "
                       f"10 traders), {FIN_STEPS} steps (run_batch)",
           "value": slots * FIN_STEPS / (ms / 1e3), "unit": UNIT, "device_ms": ms,
           "timing": "median of 3 device-timed run_batch launches after 2 full-size warm-ups", "markets_gathered": gathered,
           "rows_match_reference": fnv_ok,
           "market_steps_per_s": MARKETS * FIN_STEPS / (ms / 1e3)}
    # SURVEY §8d C5, the alternative reading: ONE market of 1024 books (one CTA per book; the
    # books share the traders, whose cash the books fold in with exact dyadic atomics). Not
    # sharded: every rank runs its own copy.
    one = F.FinanceConfig(books=MARKETS)
    F.run_batch(one, MASTER_SEED, 1, FIN_STEPS)
    one_ms = statistics.median([F.run_batch(one, MASTER_SEED, 1, FIN_STEPS)[1] for _ in range(3)])
    out["one_market"] = {"workload": f"C5 alternative: 1 market x {MARKETS} books (1000 capacity, 10 traders), "
                                     f"{FIN_STEPS} steps",
                         "value": MARKETS * one.book_capacity * FIN_STEPS / (one_ms / 1e3), "unit": UNIT,
                         "device_ms": one_ms}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        if os.path.exists(pyoracle.REF_SO):
            ref = pyoracle.Reference()
            ns1 = 20  # a single market steps its books on one thread (finance.cpp:203-247)
            _, wall1 = ref.fin_run_batch(MASTER_SEED, 1, ns1, threads=1, books=MARKETS)
            out["one_market"]["cpu_baseline"] = {
                "value": MARKETS * one.book_capacity * ns1 / (wall1 / 1e3), "unit": UNIT, "cores": 1,
                "kind": "reference",
                "sample": f"reference FinanceModel, 1 market x {MARKETS} books x {ns1} steps, 1 thread "
                          f"({wall1 / 1e3:.2f} s)"}
            threads = os.cpu_count() or 1
            nm, ns = MARKETS, FIN_STEPS  # the full C5 workload (~1 s on the host)
            _, wall = ref.fin_run_batch(MASTER_SEED, nm, ns, threads=threads)
            out["cpu_baseline"] = {
                "value": nm * cfg.books * cfg.book_capacity * ns / (wall / 1e3), "unit": UNIT,
                "cores": threads, "kind": "reference",
                "sample": f"reference run_batch(FinanceModel), {nm} markets x {ns} steps, "
                          f"{threads} threads ({wall / 1e3:.2f} s)"}
    return out

# ---------------------------------------------------------------------- agent sets (§8 a9/a12/a17)
AGENT_CAP, AGENT_CYCLES, AGENT_CHURN = 524_288, 20, 14_000  # one C2 species, its per-step churn


def kernel_table_section(args):
    """The KernelTable entries (include/abmx/simd/kernels.hpp:15-43) on their
    stream-ordered device-pointer variants, 2^26 elements (every buffer >= 64 MiB), L2 flushed
    before each rep; event-timed median of 10 reps (the memset of the entry's workspace and its
    launches included); achieved = algorithmic bytes / that time vs the measured HBM peak."""
    import ctypes as C
    import torch
    import paper_2508_16508_b200 as abmx
    lib = abmx.lib
    n = 1 << 26
    g = torch.Generator(device="cuda").manual_seed(1)
    mask = (torch.rand(n, device="cuda", generator=g) < 0.5).to(torch.uint8)
    ranks = torch.empty(n, dtype=torch.int32, device="cuda")
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    a64 = torch.randint(-2**40, 2**40, (n,), dtype=torch.int64, device="cuda", generator=g)
    b64 = torch.randint(-2**40, 2**40, (n,), dtype=torch.int64, device="cuda", generator=g)
    o64 = torch.empty_like(a64)
    s = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    vp = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    abmx._check(lib.abmx_cuda_rank_scan_async(vp(mask), vp(ranks), C.c_size_t(n), s))
    ops = {  # name: (call, algorithmic bytes)
        "rank_scan": (lambda: lib.abmx_cuda_rank_scan_async(vp(mask), vp(ranks), C.c_size_t(n), s), 5 * n),
        "count_true": (lambda: lib.abmx_cuda_count_true_async(vp(mask), C.c_size_t(n), vp(cnt), s), n),
        "compact_indices": (lambda: lib.abmx_cuda_compact_indices_async(vp(mask), vp(out), C.c_size_t(n), vp(cnt), s),
                            2 * n + 4 * n),
        "match_first_equal": (lambda: lib.abmx_cuda_match_first_equal_async(vp(ranks), C.c_size_t(n), vp(ranks),
                                                                             C.c_size_t(n // 2), vp(out), s),
                              4 * n + 4 * (n // 2) + 4 * n),
        "blend_i64": (lambda: lib.abmx_cuda_blend_i64_async(vp(mask), vp(a64), vp(b64), vp(o64), C.c_size_t(n), s),
                      n + 8 * n * 3),
    }
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    flush2 = torch.ones(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    peak, _ = hbm_peak()
    res = {}
    for name, (f, nbytes) in ops.items():
        abmx._check(f())
        ts = []
        for r in range(10):
            flush.fill_(r)
            flush2.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            abmx._check(f())
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        us = statistics.median(ts) * 1e3
        gbs = nbytes / (us / 1e6) / 1e9
        res[name] = {"us": us, "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peak}
    del flush, flush2
    return {"workload": "KernelTable entries, 2^26 elements (mask 50% true; match: rb = the first 2^25 ranks), "
                        "L2 flushed before each rep, event-timed median of 10",
            "entries": res}


def agents_section(args, rank):
    """The generic lifecycle on a C2-sized set: K x (remove_agents(kill), spawn_agents(rows,
    valid, copy apply)) through the C-ABI on device buffers, L2 flushed before each cycle;
    the reference's own remove_agents / spawn_agents (oracle/_ref) on the same inputs beside it,
    and the two final sets compared bit for bit."""
    import ctypes as C
    import numpy as np
    import torch
    import paper_2508_16508_b200 as abmx
    from paper_2508_16508_b200 import agents as A

    rng = np.random.default_rng(11)
    cap, K = AGENT_CAP, AGENT_CYCLES
    act = (rng.random(cap) < 0.7).astype(np.uint8)
    st = {"active": act, "ids": np.where(act, np.arange(cap), 0).astype(np.int64),
          "ages": np.where(act, rng.integers(0, 100, cap), 0).astype(np.int64),
          "types": np.zeros(cap, np.int64),
          "e": np.where(act, rng.integers(0, 1000, cap), 0).astype(np.int64),
          "w": np.where(act, rng.random(cap), 0.0), "f": act.copy()}
    kills = np.zeros((K + 3, cap), np.uint8)
    valids = np.zeros((K + 3, cap), np.uint8)
    for k in range(K + 3):
        kills[k, rng.choice(cap, AGENT_CHURN, replace=False)] = 1
        valids[k, rng.choice(cap, AGENT_CHURN, replace=False)] = 1
    rows = {"e": rng.integers(0, 1000, cap).astype(np.int64), "w": rng.random(cap),
            "f": np.ones(cap, np.uint8)}
    dk = torch.from_numpy(kills).cuda()
    dv = torch.from_numpy(valids).cuda()
    out = torch.zeros(1, dtype=torch.int64, device="cuda")
    slots = torch.empty(cap, dtype=torch.int32, device="cuda")
    rws = torch.empty(cap, dtype=torch.int32, device="cuda")
    res = torch.zeros(2, dtype=torch.int64, device="cuda")

    def make():
        s = A.DeviceAgentSet.from_numpy(st, ["e", "w", "f"], next_id=cap)
        arr, keep = s._rows({k: torch.from_numpy(v).cuda() for k, v in rows.items()}, cap)
        return s, arr, keep

    def cycle(s, arr, k):  # abmx_agents_lifecycle: remove + spawn fused into one cooperative kernel
        stream = s._stream()
        abmx._check(abmx.lib.abmx_agents_lifecycle(C.byref(s._c), dk[k].data_ptr(), cap, dv[k].data_ptr(), arr, 0, 0,
                                                   out.data_ptr(), res.data_ptr(), stream))

    def cycle_two_calls(s, arr, k):  # the same cycle as abmx_agents_remove + abmx_agents_spawn
        stream = s._stream()
        abmx._check(abmx.lib.abmx_agents_remove(C.byref(s._c), dk[k].data_ptr(), out.data_ptr(), stream))
        abmx._check(abmx.lib.abmx_agents_spawn(C.byref(s._c), cap, dv[k].data_ptr(), arr, 0, 0,
                                               slots.data_ptr(), rws.data_ptr(), res.data_ptr(), stream))

    w, warr, wkeep = make()
    for k in range(3):  # warm-up on a throw-away set
        cycle(w, warr, K + k)
    s, arr, keep = make()
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    flush2 = torch.ones(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        flush.fill_(k)
        flush2.sum()
        ev[k][0].record()
        cycle(s, arr, k)
        ev[k][1].record()
    torch.cuda.synchronize()
    import statistics
    cyc = [a.elapsed_time(b) for a, b in ev]
    ms, ms_mean = statistics.median(cyc), sum(cyc) / K
    w2, warr2, wkeep2 = make()
    for k in range(3):  # warm-up of the two-call path too (its own scratch sizes, first launches)
        cycle_two_calls(w2, warr2, K + k)
    s2, arr2, keep2 = make()  # the unfused two-call cycle on the same inputs, for comparison
    ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for k in range(K):
        flush.fill_(k)
        flush2.sum()
        ev2[k][0].record()
        cycle_two_calls(s2, arr2, k)
        ev2[k][1].record()
    torch.cuda.synchronize()
    cyc2 = [a.elapsed_time(b) for a, b in ev2]
    ms_two, ms_two_mean = statistics.median(cyc2), sum(cyc2) / K
    same = all(np.array_equal(a, b) for a, b in zip(s.to_numpy().values(), s2.to_numpy().values()))
    out_d = {"workload": f"lifecycle cycles on a {cap}-slot set (e:i64, w:f64, f:u8; 70% live): "
                         f"remove_agents of {AGENT_CHURN} random slots + spawn_agents of {cap} rows with "
                         f"{AGENT_CHURN} valid, copy apply (fused: abmx_agents_lifecycle); {K} cycles, "
                         f"L2 flushed before each",
             "value": cap / (ms / 1e3), "unit": "slot-cycles/s", "ms_per_cycle": ms, "ms_per_cycle_mean": ms_mean,
             "timing": "event-timed per cycle on the set's stream, median of the cycles (a cycle's events also "
                       "see any host submission delay, ~14 us of API calls per cycle; the mean is beside it)",
             "launches_per_cycle": "1 memset + 1 cooperative kernel (abmx_agents_lifecycle, k_life_coop)",
             "two_call_ms_per_cycle": ms_two, "two_call_ms_per_cycle_mean": ms_two_mean,
             "two_call_launches_per_cycle": "2 x (1 memset + 1 cooperative kernel): abmx_agents_remove and "
                                            "abmx_agents_spawn, each one k_life_coop",
             "fused_equals_two_calls": bool(same)}
    if rank == 0 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        if os.path.exists(pyoracle.REF_SO):
            ref = pyoracle.Reference()
            ewf = pyoracle.new_ewf_state(st["active"], st["ids"], st["ages"], st["types"], st["e"],
                                         st["w"], st["f"], cap)
            fin, rms = ref.lifecycle_bench(ewf, kills[:K], rows, valids[:K])
            got = s.to_numpy()
            exact = all(np.array_equal(got[k], fin[k]) for k in ("active", "ids", "ages", "e", "f")) and \
                np.array_equal(got["w"].view(np.uint64), fin["w"].view(np.uint64))
            out_d["bit_exact_vs_reference"] = bool(exact)
            out_d["cpu_baseline"] = {"value": cap / (rms / 1e3), "unit": "slot-cycles/s", "cores": 1,
                                     "kind": "reference",
                                     "sample": f"reference remove_agents + spawn_agents (oracle/_ref), the same "
                                               f"{K} cycles, 1 thread ({rms:.2f} ms per cycle)"}
    del flush, flush2
    return out_d


# ---------------------------------------------------------------------- our arm
def kernel_bytes(cfg, births, deaths):
    """SURVEY §8d algorithmic bytes per step, B = 42*N_tot + 2*C + 8*(births+deaths),
    apportioned to the kernel that owns each column. The 2*C regrow term is
    not given to any kernel: the lazy regrow never sweeps the cells (it stays in the step
    total, `step_effective_gbs`)."""
    n = capacity(cfg)
    return {"k_move": 25 * n + 8 * births,   # x,y,age read+write (2*(4+4+4)) + active read; newborn ids
            "k_cells": 0,                    # crowded grids only (pairing scratch)
            "k_update": 17 * n + 8 * deaths}  # energy read+write (2*8) + active write; zeroed ids


def ensemble_section(args, rank, world, allreduce, barrier, dist):
    """C3: 4096 x C1 replicas sharded by contiguous blocks over the ranks (sharding.shard_range);
    one all-gather of the metrics rows, checked on rank 0 against the reference's FNV."""
    import paper_2508_16508_b200 as abmx
    from paper_2508_16508_b200.sharding import shard_range
    begin, count = shard_range(ENSEMBLE_REPLICAS, world, rank)
    c1 = abmx.PredationConfig(**C1)
    abmx.run_batch(c1, MASTER_SEED, min(count, 296), 5, begin=begin, path=1)  # warm-up
    barrier()
    rows, kms = abmx.run_batch(c1, MASTER_SEED, count, ENSEMBLE_STEPS, begin=begin, path=1)
    kmax = allreduce(kms, dist.ReduceOp.MAX if dist else None)
    gathered, fnv_ok = gather_check("C3", rows, rank, dist, args.gather_device)
    slots = ENSEMBLE_REPLICAS * capacity(C1) * ENSEMBLE_STEPS
    c3_bytes = ENSEMBLE_REPLICAS * ENSEMBLE_STEPS * (42 * capacity(C1) + 2 * 100 * 100)
    ens = {"workload": "C3: 4096 x C1 replicas (100x100, 600+400, caps 1024+1024), 100 steps, "
                       "SMEM/register-resident CTA per replica",
           "value": slots / (kmax / 1e3), "unit": UNIT, "kernel_ms": kmax,
           "replicas_gathered": gathered, "rows_match_reference": fnv_ok, "scaling": "strong",
           "effective_gbs": c3_bytes / (kmax / 1e3) / 1e9,
           "note": "state stays on chip for all steps; effective GB/s uses SURVEY §8d bytes "
                   "and may exceed HBM peak"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        if os.path.exists(pyoracle.REF_SO):
            ref = pyoracle.Reference()
            threads = os.cpu_count() or 1
            nrep = 512  # a bounded sample of C3 (same C1 replicas, all host threads)
            _, wall = ref.run_batch(C1, MASTER_SEED, nrep, ENSEMBLE_STEPS, threads=threads)
            ens["cpu_baseline"] = {
                "value": nrep * capacity(C1) * ENSEMBLE_STEPS / (wall / 1e3), "unit": UNIT,
                "cores": threads, "kind": "reference",
                "sample": f"reference run_batch(PredationModel), {nrep} C1 replicas x "
                          f"{ENSEMBLE_STEPS} steps, {threads} threads ({wall / 1e3:.2f} s)"}
    return ens


def our_arm(args, rank, world, local_rank, dist):
    import numpy as np
    import torch
    import paper_2508_16508_b200 as abmx

    torch.cuda.set_device(local_rank % max(torch.cuda.device_count(), 1))
    K, W = args.steps, args.warmup

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()

    def allreduce(x, op):
        if dist is None:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=args.gather_device)
        dist.all_reduce(t, op=op)
        return float(t.item())

    if args.sharded_only:  # the sharded workloads and their gather checks only
        out = {"n_ranks": world, "backend": args.dist_backend if dist is not None else None,
               "C3": ensemble_section(args, rank, world, allreduce, barrier, dist),
               "C4_roads": traffic_roads(args, rank, world, allreduce, dist),
               "C5": finance_section(args, rank, world, allreduce, dist)}
        if rank == 0:
            print(json.dumps({"sharded_check": out}))
        return

    cfg = abmx.PredationConfig(**C2)
    seed = abmx.replica_seeds(MASTER_SEED, world)[rank]
    model = abmx.PredationModel(cfg, seed)

    # warm-up (also builds and instantiates the CUDA graph)
    model.bench(1, W, FLUSH_BYTES)
    t_next = W + 1
    barrier()
    launches0 = abmx.launch_count()
    with ClockSampler(local_rank) as clk:
        step_ms, met = model.bench(t_next, K, FLUSH_BYTES)
    launches = abmx.launch_count() - launches0
    t_next += K
    barrier()
    total_ms = float(np.sum(step_ms))
    max_ms = allreduce(total_ms, dist.ReduceOp.MAX if dist else None)
    live = float(met[0, :, 0].sum() + met[0, :, 1].sum())
    live_all = allreduce(live, dist.ReduceOp.SUM if dist else None)
    value = world * capacity(C2) * K / (max_ms / 1e3)

    # per-kernel durations (events around each kernel, graph off) for the roofline
    model.set_timing(True)
    model.set_timing(False)
    kt_steps = max(3, min(K, 10))
    model.bench(t_next, kt_steps, FLUSH_BYTES, per_kernel=True)
    t_next += kt_steps
    times = model.kernel_times()
    ev = model.last_events()
    births = ev.sheep.births + ev.wolves.births
    deaths = ev.sheep.deaths + ev.wolves.deaths
    bd = births + deaths
    kb = kernel_bytes(C2, births, deaths)
    avg = {k: ms / n for k, (ms, n) in times.items() if n}
    step_sum = sum(avg.values())
    dom = max(avg, key=avg.get)
    peak, peak_src = hbm_peak()
    achieved = kb[dom] / (avg[dom] / 1e3) / 1e9
    traffic, in_step = None, None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            traffic = tj.get(dom)
            in_step = tj.get("_in_step")
        except Exception:
            traffic = None
    step_bytes = 42 * capacity(C2) + 2 * C2["width"] * C2["height"] + 8 * bd
    # the step's random cell-word accesses alone, in the same launch shape and live fractions, L2
    # flushed, event-timed: their cost, not a bound (each includes the ~6 us launch + event floor;
    # profiles/r02_c2_cost_model.md has the per-class measurements and the ncu evidence)
    n_tiles = capacity(C2) // 2 // 1024
    ls = float(met[0, :, 0].mean()) / C2["sheep_capacity"]
    lw = float(met[0, :, 1].mean()) / C2["wolf_capacity"]
    atom_us, _ = abmx.diag_random_access(C2["width"] * C2["height"], n_tiles, n_tiles, ls, lw, 0, True)
    read_us, _ = abmx.diag_random_access(C2["width"] * C2["height"], n_tiles, n_tiles, ls, lw, 1, True)
    none_us, _ = abmx.diag_random_access(C2["width"] * C2["height"], n_tiles, n_tiles, ls, lw, 2, True)
    access = {"unit": "us", "launch_shape_alone": none_us,
              "k_move_random_atomics_alone": atom_us, "k_move": avg["k_move"] * 1e3,
              "k_update_random_reads_alone": read_us, "k_update": avg["k_update"] * 1e3,
              "note": "event-timed kernels doing ONLY the step's random cell-word atomicExch+atomicMax "
                      "(k_move) / 16-byte reads (k_update) / nothing (launch shape and hashing), same "
                      "grid and live fractions, L2 flushed clean; the random-access ceiling and the "
                      "sum-of-floors accounting are in profiles/r02_c2_cost_model.md §6"}
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes": kb[dom], "avg_launch_ms": avg[dom],
                "kernel_share": avg[dom] / step_sum,
                "per_kernel_ms": avg,
                "step_effective_gbs": step_bytes / (total_ms / K / 1e3) / 1e9,
                "random_access_cost": access,
                "step_dram_bytes_in_step": in_step.get("step_dram_bytes") if in_step else None,
                "step_algorithmic_bytes": kb["k_move"] + kb["k_update"]}

    # warm back-to-back figure beside the flushed headline: run() of K steps, no flush between
    stream = torch.cuda.ExternalStream(model.stream)
    model.run(t_next, K, metrics=False)
    t_next += K
    w0, w1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w0.record(stream)
    model.run(t_next, K, metrics=False)
    w1.record(stream)
    w1.synchronize()
    t_next += K
    warm_ms = allreduce(w0.elapsed_time(w1), dist.ReduceOp.MAX if dist else None)
    warm = {"value": world * capacity(C2) * K / (warm_ms / 1e3), "unit": UNIT, "ms_per_step": warm_ms / K,
            "note": f"run() of {K} steps back to back on the engine stream (CUDA graph per step, "
                    "the final births included), L2 NOT flushed between steps: not the headline"}

    # e2e through the C-ABI: step(t) [H2D t] + collect_metrics [D2H row], L2 flushed between
    flush = torch.empty(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    flush2 = torch.ones(FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    for _ in range(max(W, 3)):  # warm the per-call path (step graph, pinned staging)
        model.step(t_next)
        model.collect_metrics()
        t_next += 1
    e2e_s = 0.0
    for q in range(K):
        flush.fill_(q)
        flush2.sum()  # leave L2 holding clean lines (see Engine::bench)
        torch.cuda.synchronize()
        a = time.perf_counter()
        model.step(t_next)
        model.collect_metrics()
        e2e_s += time.perf_counter() - a
        t_next += 1
    e2e_max = allreduce(e2e_s, dist.ReduceOp.MAX if dist else None)
    e2e = {"value": world * capacity(C2) * K / e2e_max, "unit": UNIT, "h2d_bytes_per_step": 8,
           "d2h_bytes_per_step": 32}
    del flush, flush2
    model.close()

    ens = None if args.no_ensemble else ensemble_section(args, rank, world, allreduce, barrier, dist)

    traffic = None if args.no_traffic else traffic_section(args, rank, world, allreduce, dist)
    finance = None if args.no_finance else finance_section(args, rank, world, allreduce, dist)
    agents = None if args.no_agents else agents_section(args, rank)
    ktab = None if args.no_kernel_table else kernel_table_section(args)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import pyoracle
        if os.path.exists(pyoracle.REF_SO):
            ref = pyoracle.Reference()
            m = ref.pred(C2, abmx.replica_seeds(MASTER_SEED, 1)[0])
            m.run(1, 2)
            n_cpu = args.cpu_steps
            ms = m.run(3, n_cpu)
            cpu = {"value": capacity(C2) * n_cpu / (ms / 1e3), "unit": UNIT, "cores": 1,
                   "kind": "reference",
                   "sample": f"reference step_predation (oracle/_ref, -O3), C2 steps 3..{2 + n_cpu}, "
                             f"1 thread ({ms / 1e3:.1f} s)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
                "warmup": W, "ms_per_step": max_ms / K, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64+int", "data": "synthetic",
                "config": bench_config(),
                "timing": "CUDA events per step on the engine stream (the last step's births, "
                          "applied by k_finalize, inside its bracket); max over ranks",
                "live_agent_steps_per_s": live_all / (max_ms / 1e3),
                "e2e": e2e, "warm_run": warm, "gpu_launches": int(launches), "clocks": clk.summary(),
                "roofline": roofline, "cpu_baseline": cpu, "ensemble": ens, "traffic": traffic,
                "finance": finance, "agents": agents, "kernel_table": ktab}
        print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=40)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ensemble", action="store_true")
    ap.add_argument("--no-traffic", action="store_true")
    ap.add_argument("--no-finance", action="store_true")
    ap.add_argument("--no-agents", action="store_true")
    ap.add_argument("--no-kernel-table", action="store_true")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: CPU collectives, for tests)")
    ap.add_argument("--sharded-only", action="store_true",
                    help="run only the sharded workloads (C3, C4 roads, C5) and print their "
                         "gather checks; used by tests/test_bench_sharded_gpu.py")
    args = ap.parse_args()
    args.gather_device = "cuda" if args.dist_backend == "nccl" else "cpu"
    if args.warmup < 3:
        args.warmup = 3  # timing rules: >= 3 warm-up steps
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            reference_arm(args, world)
        return
    dist = None
    if world > 1:
        import torch
        import torch.distributed as D
        dev = local_rank % max(torch.cuda.device_count(), 1)
        torch.cuda.set_device(dev)
        if args.dist_backend == "nccl":
            D.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            D.init_process_group("gloo")
        dist = D
    try:
        our_arm(args, rank, world, local_rank, dist)
    finally:
        if dist is not None:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
