"""TEST INFRASTRUCTURE ONLY: apply INTEGRATION.md section 1's Backend::Cuda patch to a COPY of
the reference tree (oracle/Makefile `ref_cuda` makes the copy under /tmp, outside the
repository; only the built library lands in oracle/_ref_cuda/, which is git-ignored).

  * include/abmx/simd/kernels.hpp:45   enum class Backend gains `Cuda`
  * src/simd/dispatch.cpp:16-58        resolve() returns the CUDA table for Backend::Cuda and
                                       ABMX_SIMD=cuda selects it in initial_table()

usage: python oracle/patch_cuda_backend.py <tree>"""
import sys
from pathlib import Path


def edit(path: Path, old: str, new: str) -> None:
    s = path.read_text()
    if new in s:
        return  # already patched
    if old not in s:
        raise SystemExit(f"{path}: anchor not found: {old!r}")
    path.write_text(s.replace(old, new, 1))


tree = Path(sys.argv[1])
edit(tree / "include/abmx/simd/kernels.hpp", "enum class Backend { Auto, Scalar, Avx2 };",
     "enum class Backend { Auto, Scalar, Avx2, Cuda };")
disp = tree / "src/simd/dispatch.cpp"
edit(disp, '#include "abmx/errors.hpp"\n',
     '#include "abmx/errors.hpp"\n#include "abmx_cuda.h"  // the B200 engine (libabmx_cuda.so)\n')
edit(disp, "namespace {\n\nconst KernelTable* resolve(Backend b) {",
     "namespace {\n\n"
     "static_assert(sizeof(KernelTable) == sizeof(abmx_kernel_table), \"KernelTable layout\");\n"
     "const KernelTable* cuda_table() {\n"
     "    return reinterpret_cast<const KernelTable*>(abmx_cuda_kernel_table());\n"
     "}\n\n"
     "const KernelTable* resolve(Backend b) {")
edit(disp, "    case Backend::Avx2:\n        return avx2_table();\n",
     "    case Backend::Avx2:\n        return avx2_table();\n    case Backend::Cuda:\n        return cuda_table();\n")
edit(disp, '        else if (std::strcmp(env, "avx2") == 0)\n            b = Backend::Avx2;\n',
     '        else if (std::strcmp(env, "avx2") == 0)\n            b = Backend::Avx2;\n'
     '        else if (std::strcmp(env, "cuda") == 0)\n            b = Backend::Cuda;\n')
print("patched", tree)
