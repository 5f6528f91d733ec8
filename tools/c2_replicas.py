import os, sys, statistics
sys.path.insert(0, os.getcwd())
import paper_2508_16508_b200 as abmx
cfg = abmx.PredationConfig(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
                           sheep_capacity=524288, wolf_capacity=524288)
for R in (1, 2, 4, 8):
    m = abmx.PredationModel(cfg, abmx.replica_seeds(7, R))
    m.bench(1, 5, 256 << 20)
    ms, _ = m.bench(6, 20, 256 << 20)
    med = statistics.median(ms)
    print(R, "replicas: step ms", round(med, 4), "slot-steps/s %.3e" % (R * 1048576 / (med / 1e3)))
    m.close()
