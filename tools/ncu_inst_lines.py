"""Executed warp instructions per CUDA source line of one kernel (needs -lineinfo and
--import-source on). usage: python tools/ncu_inst_lines.py <report> <kernel> [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda", "-k", kern],
                     capture_output=True, text=True).stdout
hdr, rows, fname, seen = None, [], "?", set()
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if (fname, r[1]) in seen:
            break
        seen.add((fname, r[1]))
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0].isdigit():
        d = dict(zip(hdr, r))
        ie = d.get("Instructions Executed", "0")
        if ie.isdigit() and int(ie) > 0:
            rows.append((int(ie), fname, int(r[0]), r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
print("total warp instructions", tot)
for n, f, ln, src in sorted(rows, reverse=True)[:top]:
    print(f"{n:>11d} {100 * n / tot:5.1f}%  {f}:{ln:<5d} {src}")
