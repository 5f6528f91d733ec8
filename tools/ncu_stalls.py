"""Top stall reasons and hottest SASS lines of one kernel in an ncu report."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 14
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", kern, "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
data = []
for row in rows[2:]:  # first kernel instance only
    if row and row[0] == "Kernel Name":
        break
    if len(row) == len(hdr):
        data.append(row)
si = hdr.index("Warp Stall Sampling (All Samples)")
val = lambda r: int(r[si]) if r[si].isdigit() else 0
print("total samples", sum(val(r) for r in data))
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
agg = {hdr[i]: sum(int(r[i]) if r[i].isdigit() else 0 for r in data) for i in cols}
print(sorted(agg.items(), key=lambda x: -x[1])[:8])
for k in sorted(range(len(data)), key=lambda k: -val(data[k]))[:n]:
    print(val(data[k]), data[k][1].strip()[:64], "| prev:", data[k - 1][1].strip()[:48])
