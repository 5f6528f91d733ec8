"""CPU: the in-situ recipe's Backend::Cuda patch (oracle/patch_cuda_backend.py) applies cleanly to a
copy of the reference tree and makes exactly the edits INTEGRATION.md section 1 describes."""
import os
import shutil
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"


@pytest.mark.skipif(not os.path.exists(os.path.join(REF, "src", "simd", "dispatch.cpp")),
                    reason="reference sources absent")
def test_backend_cuda_patch_applies(tmp_path):
    tree = tmp_path / "tree"
    tree.mkdir()
    shutil.copytree(os.path.join(REF, "include"), tree / "include")
    shutil.copytree(os.path.join(REF, "src"), tree / "src")
    subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "patch_cuda_backend.py"), str(tree)], check=True)
    hdr = (tree / "include/abmx/simd/kernels.hpp").read_text()
    disp = (tree / "src/simd/dispatch.cpp").read_text()
    assert "enum class Backend { Auto, Scalar, Avx2, Cuda };" in hdr
    assert '#include "abmx_cuda.h"' in disp
    assert "case Backend::Cuda:\n        return cuda_table();" in disp
    assert 'std::strcmp(env, "cuda") == 0' in disp
    # idempotent
    subprocess.run([sys.executable, os.path.join(ROOT, "oracle", "patch_cuda_backend.py"), str(tree)], check=True)
    assert (tree / "src/simd/dispatch.cpp").read_text() == disp
