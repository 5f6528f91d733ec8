"""Summarise an ncu --metrics gpu__time_duration.sum,dram__bytes_*.sum --csv launch list:
one line per launch (kernel, us, DRAM MB read / written)."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hd = rows[h]
ki, mi, vi = hd.index("Kernel Name"), hd.index("Metric Name"), hd.index("Metric Value")
cur = {}
for r in rows[h + 1:]:
    if len(r) > vi:
        cur.setdefault((int(r[0]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
skip = sys.argv[2] if len(sys.argv) > 2 else None
for (i, k), d in cur.items():
    if skip and skip in k:
        continue
    print(f"{i:4d} {k[:70]:70s} {d.get('gpu__time_duration.sum', 0) / 1e3:9.1f} us  "
          f"R {d.get('dram__bytes_read.sum', 0) / 1e6:8.1f} MB  W {d.get('dram__bytes_write.sum', 0) / 1e6:8.1f} MB")
