"""C-ABI checks that run without a GPU: the library loads, exports every
symbol include/omnitrack.h declares, and the ctypes records match the C
layout.  No compute calls (there is no device here)."""
import ctypes as C
import os
import re

import pytest

from paper_1910_06017_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "omnitrack.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(?:int|const char \*)\s*(ft_\w+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(_lib.LIB_PATH):
        from paper_1910_06017_b200 import build
        build.build()
    return _lib.load()


def test_header_declares_the_path():
    syms = declared_symbols()
    for need in ["ft_build_pyramid", "ft_structure_texture", "ft_compute_flow", "ft_predict",
                 "ft_match", "ft_hungarian", "ft_update", "ft_tracker_step"]:
        assert need in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
        assert name in _lib.SIGNATURES, f"{name} missing from the ctypes table"


def test_struct_layouts():
    assert C.sizeof(_lib.ft_flow_params) == 40
    assert C.sizeof(_lib.ft_det) == 48
    assert C.sizeof(_lib.ft_track) == 72
    assert C.sizeof(_lib.ft_tracker_config) == 24 + 40 + 40 + 16  # + motion, klt_grid, prefetch, pad


def test_host_scalars_without_gpu(lib):
    out = C.c_int()
    for (w, h), lvl in [((720, 576), 0), ((2560, 1280), 1), ((4096, 2048), 2),
                        ((1920, 1080), 1), ((3840, 2160), 2)]:
        _lib.check(lib.ft_select_level(w, h, C.byref(out)))
        assert out.value == lvl
    _lib.check(lib.ft_auto_scales(720, 576, C.byref(out)))
    assert out.value == 6
    _lib.check(lib.ft_auto_scales(960, 540, C.byref(out)))
    assert out.value == 6
    with pytest.raises(ValueError):
        _lib.check(lib.ft_select_level(1, 5, C.byref(out)))


def test_error_mapping(lib):
    with pytest.raises(ValueError, match="at least 2x2"):
        _lib.check(lib.ft_select_level(1, 1, C.byref(C.c_int())))


def test_kernels_are_sm100a(lib):
    # the shared object carries sm_100a SASS (cuobjdump lists the ELF arch)
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
