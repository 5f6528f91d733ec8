"""Run pytest selections against the loaded libabmx_cuda.so, then report the device bounds
checks of a -DABMX_CHECKED build (abmx_predation_check_status; tools/sanitize_smoke.py).
usage: ABMX_CUDA_LIB=build/variants/checked/libabmx_cuda.so python tools/checked_pytest.py <pytest args>"""
import ctypes as C
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
rc = pytest.main(sys.argv[1:])
import paper_2508_16508_b200 as abmx  # noqa: E402
abmx.lib.abmx_predation_check_status.restype = C.c_int
chk = abmx.lib.abmx_predation_check_status()
print(f"pytest rc {int(rc)}; device bounds checks: {chk} (0 = on, none failed; -1 = not a checked build)")
sys.exit(int(rc) or (chk not in (0,)))
