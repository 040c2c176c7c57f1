"""The C-ABI library loads and exports every entry point include/se2ot.h declares (no GPU needed:
no compute call is made here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "se2ot.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^[A-Za-z_][\w \*]*?\b(se2_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib():
    from paper_2402_15322_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_the_north_star_entry_points():
    names = declared_functions()
    for n in ("se2_kernel_build", "se2_conv", "se2_sinkhorn", "se2_barycenter", "se2_marginal_error"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    names = declared_functions()
    assert len(names) >= 15
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    from paper_2402_15322_b200 import _lib
    assert sorted(_lib.EXPORTED) == names


def test_abi_version_and_no_internal_symbols(lib):
    lib.se2_abi_version.restype = ctypes.c_int32
    assert lib.se2_abi_version() == 1
    # internal launchers are hidden (-fvisibility=hidden): only the C ABI is exported
    assert not hasattr(lib, "_ZN3se218launch_conv_linearEPK12se2_kernel_sPKfiRKNS_8EpilogueEP11CUstream_stPi")


def test_invalid_arguments_fail_without_gpu(lib):
    """Argument validation happens before any CUDA call: null pointers -> SE2_EINVAL (1)."""
    lib.se2_kernel_build.restype = ctypes.c_int
    assert lib.se2_kernel_build(None, None, ctypes.c_double(0.1), 3, 1, 0, None) == 1
    lib.se2_last_error.restype = ctypes.c_char_p
    assert b"null" in lib.se2_last_error()
    lib.se2_conv.restype = ctypes.c_int
    assert lib.se2_conv(None, None, None, 1, 0, None) == 1
