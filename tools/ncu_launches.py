"""Average per-kernel metrics from an `ncu --csv --log-file` launch list."""
import collections
import csv
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
hdr = rows[0]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
agg = collections.defaultdict(list)
for r in rows[1:]:
    try:
        agg[(r[ki].split("(")[0], r[mi], r[ui])].append(float(r[vi].replace(",", "")))
    except (ValueError, IndexError):
        pass
for (k, m, u), v in sorted(agg.items()):
    print(f"{k:16s} {m:32s} {sum(v) / len(v):14.2f} {u:8s} n={len(v)}")
