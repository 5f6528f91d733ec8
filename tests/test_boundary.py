"""CPU: the C-ABI boundary — the shared library loads and exports every symbol that
include/abmx_cuda.h declares (no compute calls: there is no GPU here), the KernelTable struct
has the reference layout, and the Python/C++ host mirrors match the reference interface."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "abmx_cuda.h")
LIB = os.path.join(ROOT, "paper_2508_16508_b200", "libabmx_cuda.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^[\w\s\*]+?\b(abmx_\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if not n.endswith("_t")))


def test_library_built_for_sm100a():
    assert os.path.exists(LIB), "build with `make` (no CPU fallback exists)"
    out = subprocess.run(["cuobjdump", "--list-elf", LIB], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(LIB)
    names = declared_functions()
    assert len(names) >= 40, names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_kernel_table_layout_matches_reference():
    """abmx_kernel_table == abmx::simd::KernelTable: name + 7 function pointers
    (include/abmx/simd/kernels.hpp:15-43)."""
    import paper_2508_16508_b200 as m
    t = m.kernel_table()
    assert t.name == b"cuda"
    assert C.sizeof(m._KernelTableC) == 8 * 8
    for f in ("rank_scan", "count_true", "compact_indices", "match_first_equal", "blend_i64",
              "blend_f64", "blend_u8"):
        assert getattr(t, f), f


def test_kernel_table_layout_against_reference_build(reference):
    import paper_2508_16508_b200 as m
    ref_tab = reference.table(0)
    assert ref_tab.struct.name == b"scalar"
    assert C.sizeof(type(ref_tab.struct)) == C.sizeof(m._KernelTableC)


def test_python_mirror_defaults_match_reference_config():
    """PredationConfig defaults (predation.hpp:13-27)."""
    import paper_2508_16508_b200 as m
    c = m.PredationConfig()
    assert (c.width, c.height, c.n_sheep0, c.n_wolves0) == (100, 100, 600, 400)
    assert (c.sheep_capacity, c.wolf_capacity) == (20000, 20000)
    assert (c.energy_gain_sheep, c.energy_gain_wolf, c.metabolism) == (4.0, 20.0, 1.0)
    assert (c.reproduce_prob_sheep, c.reproduce_prob_wolf, c.reproduce_energy_frac) == (0.04, 0.05, 0.5)
    assert c.regrow_delay == 30
    with pytest.raises(m.SchemaError):
        m.PredationConfig(no_such_field=1)


def test_host_seed_plumbing_matches_oracle(oracle):
    import paper_2508_16508_b200 as m
    assert m.replica_seeds(7, 1)[0] == 0x2e80eb5276648836
    for r, s in enumerate(m.replica_seeds(123, 9)):
        assert s == oracle.replica_seed(123, r)


def test_error_taxonomy():
    import paper_2508_16508_b200 as m
    for e in (m.SchemaError, m.CapacityError, m.DomainError, m.BatchError, m.CudaError,
              m.ContractError):
        assert issubclass(e, m.AbmxError)
    assert m._ERRORS[7] is m.ContractError
    assert m._ERRORS[1] is m.DomainError and m._ERRORS[2] is m.CapacityError


@pytest.mark.parametrize("hdr", ["abmx_cuda.h", "abmx_cuda.hpp"])
def test_headers_compile_standalone(hdr, tmp_path):
    """Each public header is self-contained (C11 for the ABI, C++20 for the host mirror)."""
    is_c = hdr.endswith(".h")
    tu = tmp_path / ("tu.c" if is_c else "tu.cpp")
    tu.write_text(f'#include "{hdr}"\nint main(void) {{ return 0; }}\n')
    cmd = ["gcc" if is_c else "g++", "-fsyntax-only", "-std=c11" if is_c else "-std=c++20", "-Wall",
           "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"), str(tu)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_oracle_is_not_linked_into_the_product():
    """The product library must not depend on or embed the checker."""
    out = subprocess.run(["nm", "-D", LIB], capture_output=True, text=True).stdout
    assert "orc_" not in out and "ref_pred" not in out
    ldd = subprocess.run(["ldd", LIB], capture_output=True, text=True).stdout
    assert "oracle" not in ldd and "abmx_ref" not in ldd


def test_integration_snippets_compile(tmp_path):
    """The C++ in INTEGRATION.md compiles against this repo's headers and, for the reference-side
    bindings, the reference's own public headers (skipped where /root/reference is absent)."""
    import re
    import shutil
    import subprocess
    ref_inc = "/root/reference/proj/include"
    if not os.path.isdir(ref_inc) or not shutil.which("g++"):
        pytest.skip("reference headers or g++ not available")
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```cpp\n(.*?)```", text, re.S)
    assert len(blocks) >= 5
    pre = ('#include <cstdint>\n#include <vector>\n#include "abmx/simd/kernels.hpp"\n#include "abmx/batch.hpp"\n'
           '#include "abmx/models/predation.hpp"\n#include "abmx/models/traffic.hpp"\n#include "abmx_cuda.hpp"\n')
    fragments = {  # statement-level snippets: the names the prose around them provides
        1: "void f1() {\n%s}\n",
        3: ("void f3() {\nstruct { bool id_recycling() const { return false; } } set;\n"
            "int32_t cap = 0, m = 0; int64_t species = 0; void* stream = nullptr;\n"
            "void *d_e = nullptr, *d_w = nullptr, *d_f = nullptr;\n"
            "uint8_t *d_active = nullptr, *d_kill = nullptr, *d_valid = nullptr;\n"
            "int64_t *d_ids = nullptr, *d_types = nullptr, *d_ages = nullptr, *d_counters = nullptr,"
            " *d_retired = nullptr, *d_res = nullptr;\n"
            "int32_t *d_slots = nullptr, *d_rows = nullptr; abmx_column* rows = nullptr;\n%s}\n"),
    }
    body = []
    for i, b in enumerate(blocks):
        b = re.sub(r'#include "abmx_cuda\.hp?p?"\n', "", b)
        body.append(fragments[i] % b if i in fragments else b)
    src = tmp_path / "integration.cpp"
    src.write_text(pre + "namespace abmx::models {\n" + "\n".join(body[2:]) + "\n}\n" +
                   body[0] + "\n" + body[1])
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), "-I", ref_inc,
                        "-I", "/usr/local/cuda/include", str(src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[:2000]


def test_integration_functor_snippet_compiles(tmp_path):
    """The device-functor example in INTEGRATION.md compiles with nvcc against include/."""
    import re
    import shutil
    import subprocess
    if not shutil.which("nvcc"):
        pytest.skip("nvcc not available")
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    blocks = re.findall(r"```cuda\n(.*?)```", text, re.S)
    assert blocks
    src = tmp_path / "functors.cu"
    src.write_text(blocks[0])
    r = subprocess.run(["nvcc", "-std=c++17", "-fmad=false", "-gencode", "arch=compute_100a,code=sm_100a", "-c",
                        "-I", os.path.join(ROOT, "include"), str(src), "-o", str(tmp_path / "functors.o")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[:2000]
