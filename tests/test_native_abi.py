"""CPU-side checks of the C ABI: the library loads and exports every entry
point include/rlfc_b200.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re

from conftest import ROOT


def declared_functions():
    text = open(os.path.join(ROOT, "include", "rlfc_b200.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|uint64_t)\s+(rlfc_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1805_06019_b200 import _build, _native
    _build.build_cuda()
    lib = _native.load_library()
    names = declared_functions()
    assert len(names) >= 9
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(_native.EXPORTS)
    buf = ctypes.create_string_buffer(64)
    lib.rlfc_version(buf, 64)
    assert b"sm_100a" in buf.value


def test_cubin_targets_sm100a():
    import subprocess
    from paper_1805_06019_b200 import _build
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          _build.CUDA_LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_field_struct_layout():
    from paper_1805_06019_b200 import _native
    # 18 int32 + 3*32 int32 + 3 ptr + 3 ptr + 3 u64 + 1 ptr
    assert ctypes.sizeof(_native.RlfcField) == 18 * 4 + 96 * 4 + 10 * 8
