"""GPU: the Python snippets of INTEGRATION.md run as written (the ctypes one with the library's
in-tree path) and give what their comments promise."""
import os
import re

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def snippets():
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    return re.findall(r"```python\n(.*?)```", text, re.S)


def test_python_api_snippet(abmx):
    ns = {}
    exec(snippets()[0], ns)  # noqa: S102 - our own documentation
    assert ns["rows"].shape == (4096, 100, 4)
    assert ns["m"].collect_metrics().shape == (1, 4)
    assert ns["ranks"].tolist() == [1, 0, 2, 3]


def test_ctypes_snippet(abmx):
    src = snippets()[1].replace('"libabmx_cuda.so"', repr(abmx.library_path))
    ns = {}
    exec(src, ns)  # noqa: S102
    lib = ns["lib"]
    m = np.array([1, 0, 1, 1], np.uint8)
    out = np.zeros(4, np.int32)
    import ctypes as C
    lib.abmx_cuda_rank_scan(m.ctypes.data_as(C.POINTER(C.c_uint8)), out.ctypes.data_as(C.POINTER(C.c_int32)), 4)
    assert out.tolist() == [1, 0, 2, 3]
