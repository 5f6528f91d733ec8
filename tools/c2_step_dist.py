"""Per-step device time distribution of C2 (bench path: graph steps, L2 flushed between steps),
with the step's births and deaths, to look for structure in the spread."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402

cfg = abmx.PredationConfig(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
                           sheep_capacity=524288, wolf_capacity=524288)
m = abmx.PredationModel(cfg, abmx.replica_seeds(7, 1)[0])
m.bench(1, 5)
ms, met = m.bench(6, 300)
us = ms * 1e3
print("steps 6..305: mean %.2f median %.2f min %.2f p90 %.2f max %.2f" % (us.mean(), np.median(us), us.min(),
                                                                         np.percentile(us, 90), us.max()))
print("by step mod 8:", [round(float(us[(np.arange(300) + 6) % 8 == k].mean()), 2) for k in range(8)])
print("by step mod 2:", [round(float(us[(np.arange(300) + 6) % 2 == k].mean()), 2) for k in range(2)])
print("first 60:", " ".join("%.1f" % x for x in us[:60]))
ns = met[0, :, 0]
print("corr(time, n_sheep) = %.3f" % np.corrcoef(us, ns)[0, 1])
fast = us < np.median(us)
print("fast steps mean n_sheep %.0f, slow %.0f" % (ns[fast].mean(), ns[~fast].mean()))
# flush variants
for fb in (0, 64 << 20, 512 << 20):
    ms2, _ = m.bench(400 + fb % 7, 100, fb)
    print("flush %4d MiB: mean %.2f median %.2f min %.2f" % (fb >> 20, ms2.mean() * 1e3, np.median(ms2) * 1e3,
                                                           ms2.min() * 1e3))
