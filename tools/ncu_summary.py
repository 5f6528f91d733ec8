"""Summarise an ncu report (raw page) per kernel: duration, DRAM bytes, throughput, occupancy."""
import csv
import io
import json
import subprocess
import sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]


def summarise(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")].split("(")[0]}
        for w in WANT:
            if w in hdr:
                v = r[hdr.index(w)]
                u = units[hdr.index(w)]
                try:
                    x = float(v.replace(",", ""))
                    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1, "us": 1e-3, "ms": 1, "ns": 1e-6}.get(u)
                    if w.startswith("dram__bytes") or w == "lts__t_bytes.sum":
                        x = x * (scale or 1)
                        d[w] = x
                    elif w == "gpu__time_duration.sum":
                        d["ms"] = x * (scale or 1)
                    else:
                        d[w] = x
                except ValueError:
                    d[w] = v
        if "dram__bytes_read.sum" in d:
            d["dram_bytes"] = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0)
            d["dram_gbs"] = d["dram_bytes"] / (d["ms"] / 1e3) / 1e9
        res.append(d)
    return res


if __name__ == "__main__":
    for d in summarise(sys.argv[1]):
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items()}))
