#!/bin/bash
# Regenerate the committed profiles/ summaries from the captures in gpurun_out/ (after
# tools/profile_round.sh r01, tools/profile_models.sh r01 and the C3 capture c3_final).
set -e
cp gpurun_out/bench_r01.json profiles/r01_bench.json
{ echo "# ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv python bench.py (tools/profile_round.sh); mean per launch";
  python tools/ncu_launches.py gpurun_out/launches_r01.csv; } > profiles/r01_launches.txt
python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep | grep '^{' > /tmp/c2.jsonl
python tools/ncu_summary.py gpurun_out/c3_final.ncu-rep | grep '^{' | tail -1 > /tmp/c3.jsonl
{ for f in trf_c4_r01 trf_ens_r01 fin_r01 agents_r01 table_r01; do python tools/ncu_summary.py gpurun_out/$f.ncu-rep; done; } | grep '^{' > /tmp/models.jsonl
python - <<'PY'
import json, statistics
def agg(rows):
    by = {}
    for r in rows:
        by.setdefault(r["kernel"], []).append(r)
    out = []
    for k, rs in by.items():
        m = {"kernel": k, "launches": len(rs)}
        for key in rs[0]:
            if key != "kernel":
                m[key] = statistics.mean(r[key] for r in rs)
        out.append(m)
    return out
c2 = agg([json.loads(l) for l in open("/tmp/c2.jsonl")])
c3 = json.loads(open("/tmp/c3.jsonl").read())
c3["note"] = "C3: 4096 x C1 x 100 steps, one launch (tools/prof_c3.py)"
open("profiles/r01_ncu_full.jsonl", "w").write("\n".join(json.dumps(x) for x in c2 + [c3]) + "\n")
d = {x["kernel"]: x["dram_bytes"] for x in c2}
d["_source"] = ("ncu --set full --clock-control none (cold L2, ncu cache control), tools/prof_c2.py on C2; "
                "dram__bytes_read.sum + dram__bytes_write.sum per launch, mean of the captured launches "
                "(profiles/r01_ncu_full.jsonl)")
open("profiles/ncu_traffic.json", "w").write(json.dumps(d, indent=1) + "\n")
models = agg([json.loads(l) for l in open("/tmp/models.jsonl")])
open("profiles/r01_models_ncu.jsonl", "w").write("\n".join(json.dumps(x) for x in models) + "\n")
for x in c2 + [c3] + models:
    print(x["kernel"], round(x["ms"], 4))
PY
{ echo "== k_move"; python tools/ncu_stalls.py gpurun_out/prof_r01.ncu-rep k_move 10;
  echo "== k_update"; python tools/ncu_stalls.py gpurun_out/prof_r01.ncu-rep k_update 10;
  echo "== k_ensemble (C3)"; python tools/ncu_stalls.py gpurun_out/c3_final.ncu-rep k_ensemble 10; } > profiles/r01_stalls.txt
{ echo "== k_traffic_ens"; python tools/ncu_lines.py gpurun_out/trf_ens_r01.ncu-rep k_traffic_ens 10;
  echo "== k_fin"; python tools/ncu_lines.py gpurun_out/fin_r01.ncu-rep k_fin 15;
  echo "== k_ensemble"; python tools/ncu_lines.py gpurun_out/c3_final.ncu-rep k_ensemble 15; } > profiles/r01_models_lines.txt
