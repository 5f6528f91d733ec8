"""GPU: the header-only C++ mirror (include/abmx_cuda.hpp) compiled against libabmx_cuda.so and
run like a reference user's program; its metrics rows must equal the oracle's."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_mirror_models(abmx, oracle, tmp_path):
    exe = str(tmp_path / "hpp_models")
    libdir = os.path.join(ROOT, "paper_2508_16508_b200")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "hpp_models.cpp"), "-L", libdir,
                    "-labmx_cuda", f"-Wl,-rpath,{libdir}", "-o", exe], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout.splitlines()
    rows = {}
    for line in out:
        tag, *vals = line.split()
        rows.setdefault(tag, []).append(vals)
    seed = abmx.replica_seeds(7, 1)[0]
    cfg = dict(width=100, height=100, n_sheep0=600, n_wolves0=400, sheep_capacity=1024,
               wolf_capacity=1024, energy_gain_sheep=4.0, energy_gain_wolf=20.0, metabolism=1.0,
               reproduce_prob_sheep=0.04, reproduce_prob_wolf=0.05, reproduce_energy_frac=0.5,
               regrow_delay=30)
    p = oracle.pred(cfg, seed)
    for t in range(20):
        p.step(t + 1)
        assert [int(float(x)) for x in rows["P"][t]] == list(p.metrics()), t
    tm = oracle.traffic(30, 10, 0.5, seed)
    for t in range(40):
        tm.step(t + 1)
        assert [float(x) for x in rows["T"][t]] == tm.metrics().tolist(), t
    assert [int(x) for x in rows["TT"][0]] == [tm.m.spawned_total, tm.m.exited_total]
    fm = oracle.fin(seed, book_capacity=64)
    for t in range(10):
        fm.step(t + 1)
        got = np.array([[float(x) for x in r] for r in rows["F"][5 * t:5 * t + 5]])
        assert np.array_equal(got, fm.metrics()), t
    assert rows["E"][0] == ["DomainError"]
