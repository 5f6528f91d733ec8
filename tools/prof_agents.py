"""Lifecycle cycles on a C2-sized device agent set (bench.py agents section), for ncu / timing."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import argparse  # noqa: E402
import bench  # noqa: E402

ap = argparse.Namespace(no_cpu_baseline=True)
r = bench.agents_section(ap, 0)
print("ms per cycle", r["ms_per_cycle"])
