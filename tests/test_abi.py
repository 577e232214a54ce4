"""CPU: the native libraries load and export every symbol their C headers
declare (no compute calls -- there is no GPU here)."""
import ctypes
import os
import re

import pytest

from paper_1709_07781_b200 import _build, ndx

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header: str, prefix: str) -> list[str]:
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"\w+)\s*\(", src)))


def test_libndx_exports_every_declared_symbol():
    lib = ctypes.CDLL(ndx.lib_path())
    names = declared("ndx.h", "ndx_")
    assert len(names) >= 35
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    names = set(declared("ndx.h", "ndx_"))
    bound = {s[0] for s in ndx.SIGNATURES}
    assert names == bound, (names - bound, bound - names)


def test_libndactor_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(_build.LIB, "libndactor.so"))
    names = declared("ndactor_c.h", "ndactor_")
    assert names
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_error_strings_and_sizes_without_gpu():
    lib = ndx.load()
    assert lib.ndx_abi_version() == 1
    assert b"invalid" in lib.ndx_error_string(10001)
    assert b"2^31" in lib.ndx_error_string(10002)
    assert lib.ndx_wah_ctl_bytes() % 256 == 0
    # one u64 status per (tile, digit) of the pass with the most: the wide
    # pass has 16384-pair tiles x 2048 digits, the byte passes 8192 x 256
    n = 1 << 20
    assert lib.ndx_wah_status_bytes(n) >= 256 + max((n // 16384) * 2048, (n // 8192) * 256) * 8
    assert lib.ndx_wah_emit_scratch_bytes(1 << 20) > 0
    assert lib.ndx_scan_scratch_bytes(5000) > 0


def test_launchers_validate_arguments_without_gpu():
    lib = ndx.load()
    # null pointers are rejected before any CUDA call
    assert lib.ndx_wah_plan(None, 10, None, None, None) == 10001
    assert lib.ndx_wah_emit(None, 10, None, None, None, None, None, None) == 10001
    assert lib.ndx_compact_count(None, 5, None, None) == 10001


def test_kernels_are_sm100a_cubins():
    """The fat binary carries sm_100a SASS (no PTX-only fallback)."""
    import shutil
    import subprocess

    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(cuobjdump):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([cuobjdump, "--list-elf", ndx.lib_path()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
