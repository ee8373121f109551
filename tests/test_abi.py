"""The C-ABI library loads without a GPU and exports every declared symbol."""

import ctypes
import os
import re

import numpy as np

from _util import ROOT

HEADER = os.path.join(ROOT, "include", "sph_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int32_t|size_t|long long|const char\*)\s+(sph_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_builds_and_exports_every_declared_symbol():
    from paper_2603_11868_b200 import _native, build
    build.build_library()
    lib = _native.load()
    syms = declared_symbols()
    assert len(syms) >= 35
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.EXPORTED)
    assert lib.sph_abi_version() == _native.ABI_VERSION == 16


def test_struct_layouts_match_header(tmp_path):
    """Every ctypes mirror has the C compiler's size and field offsets for
    the header's structs (gcc on include/sph_b200.h, no GPU needed)."""
    import subprocess
    from paper_2603_11868_b200 import _native
    structs = {"SphSweepArgs_f32": _native.SphSweepArgs_f32,
               "SphSweepArgs_f64": _native.SphSweepArgs_f64,
               "SphStepStats": _native.SphStepStats, "SphEngine": _native.SphEngine,
               "SphHaloPlan": _native.SphHaloPlan, "SphRows": _native.SphRows,
               "SphSlabGeom": _native.SphSlabGeom}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "sph_b200.h"',
             'int main(void) {']
    for name, cls in structs.items():
        lines.append(f'printf("{name} size %zu\\n", sizeof({name}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{name} {f} %zu\\n", offsetof({name}, {f}));')
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                    str(src), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout
    for line in out.splitlines():
        name, field, value = line.split()
        cls = structs[name]
        got = ctypes.sizeof(cls) if field == "size" else getattr(cls, field).offset
        assert got == int(value), (name, field)


def test_workspace_queries_need_no_gpu():
    from paper_2603_11868_b200 import _native
    lib = _native.load()
    assert lib.sph_sweep_workspace_bytes(1000) >= 32 * 256 * 4
    assert lib.sph_sort_workspace_bytes(1 << 20) > (1 << 20) * 16
    assert lib.sph_cll_workspace_bytes(1000, 5000) > 0
    assert lib.sph_engine_workspace_bytes(1000, 5000, 0) > 0


def test_product_path_refuses_cpu_fallback():
    import pytest
    import torch
    from paper_2603_11868_b200 import _native, ExecutionPolicy
    from paper_2603_11868_b200.sorting import radix_sort_permutation
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(_native.NativeUnavailable):
        radix_sort_permutation(ExecutionPolicy.cuda(), np.arange(5))


def test_sass_is_sm100a():
    """The shipped library carries sm_100a SASS (not just PTX)."""
    import shutil
    import subprocess
    import pytest
    from paper_2603_11868_b200 import build
    exe = shutil.which("cuobjdump")
    if exe is None:
        pytest.skip("cuobjdump missing")
    out = subprocess.run([exe, "--list-elf", build.LIB], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
