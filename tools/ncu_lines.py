"""Warp-stall samples per CUDA source line of one kernel (needs -lineinfo and
--import-source on). usage: python tools/ncu_lines.py <report> <kernel> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda",
                      "-k", kern], capture_output=True, text=True).stdout
fname, rows, seen_fn = "?", [], set()
hdr = None
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if (fname, r[1]) in seen_fn:  # later instances of the same kernel: stop
            break
        seen_fn.add((fname, r[1]))
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0].isdigit() and len(r) > 4 and r[4].isdigit():
        rows.append((int(r[4]), fname, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
print("total samples", tot)
for s, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{s:6d} {100 * s / tot:5.1f}%  {f}:{ln:<5d} {src}")
