"""ncu range target: ONE C2 step (k_move + k_update, graph launch) between cudaProfilerStart and
cudaProfilerStop, after an untimed L2 flush, as in bench.py. Under
  ncu --replay-mode app-range --profile-from-start off --cache-control none --metrics ...
the two kernels are measured as one workload: in-step DRAM bytes, with k_update reading the
cell words k_move left in L2 (no cache flush between the kernels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2508_16508_b200 as abmx  # noqa: E402

cfg = abmx.PredationConfig(width=2048, height=2048, n_sheep0=300000, n_wolves0=30000,
                           sheep_capacity=524288, wolf_capacity=524288)
m = abmx.PredationModel(cfg, abmx.replica_seeds(7, 1)[0])
m.bench(1, 6, 256 << 20)  # warm-up, leaves births pending like a run
flush = torch.empty((256 << 20) // 4, dtype=torch.int32, device="cuda")
flush2 = torch.ones((256 << 20) // 4, dtype=torch.int32, device="cuda")
flush.fill_(1)
flush2.sum()
torch.cuda.synchronize()
torch.cuda.profiler.start()
m.run(7, 1, metrics=False)  # one step: k_move + k_update (+ k_finalize for its births)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("range ok")
