"""The C-ABI library loads, exports every symbol include/sgp4b.h declares,
and rejects bad arguments with status codes (host-side validation only: no
kernel is launched, so these run without a GPU)."""

import ctypes
import re
import subprocess

import numpy as np
import pytest

from paper_2603_27830_b200 import _native
from tests.conftest import ROOT

HEADER = ROOT / "include" / "sgp4b.h"


def declared_symbols():
    text = HEADER.read_text()
    return re.findall(r"^\s*(?:int|const char\*)\s+(sgp4b_\w+)\s*\(", text, flags=re.M)


def test_header_matches_binding():
    assert tuple(declared_symbols()) == _native.EXPORTED_SYMBOLS


def test_library_exports_every_symbol():
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.library_path())],
                         capture_output=True, text=True, check=True).stdout
    for name in declared_symbols():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name


def test_abi_constants():
    lib = _native.load()
    assert lib.sgp4b_abi_version() == _native.ABI_VERSION
    text = HEADER.read_text()
    assert f"#define SGP4B_SATREC_FIELDS {_native.SATREC_FIELDS}" in text
    assert f"#define SGP4B_RECORD_SLOTS {_native.RECORD_SLOTS}" in text


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.library_path())],
                         capture_output=True, text=True, check=True).stdout
    assert "sm_100a" in out


GRAV = np.zeros(8)


@pytest.mark.parametrize("call", [
    lambda L: L.sgp4b_init(1, 0, GRAV.ctypes.data, 64, 1, 1, 1, 1, None),       # n = 0
    lambda L: L.sgp4b_init(1, 4, GRAV.ctypes.data, 16, 1, 1, 1, 1, None),       # precision
    lambda L: L.sgp4b_init(None, 4, GRAV.ctypes.data, 64, 1, 1, 1, 1, None),   # null
    lambda L: L.sgp4b_pack(1, 1, 1, 4, None, 64, 1, None),                      # null grav
    lambda L: L.sgp4b_propagate_grid(1, 4, 1, None, 0, 1.0, 32, GRAV.ctypes.data, 1, 0, 0, 1, 0, None),
    lambda L: L.sgp4b_propagate_grid(1, 4, 1, None, 8, 1.0, 32, GRAV.ctypes.data, 1, 8, 4, 1, 8, None),
    lambda L: L.sgp4b_propagate_grid(1, 1, 1, None, (1 << 30) + 1, 1.0, 32, GRAV.ctypes.data, 1,
                                     (1 << 31), (1 << 31), 1, (1 << 31), None),  # m > 2^30
    lambda L: L.sgp4b_propagate_pairs(1, 1, 1, None, 0, 1.0, 64, GRAV.ctypes.data, 1, 1, None),
    lambda L: L.sgp4b_solve_kepler(1, 1, 1, 4, 8, 1, None),
    lambda L: L.sgp4b_drift_percentiles(1, 1, 0, 4, 1, 1, 1, None),            # n = 0
    lambda L: L.sgp4b_drift_percentiles(1, None, 4, 4, 1, 1, 1, None),         # null
    lambda L: L.sgp4b_tle_columns(1, 100, 1, 1, 0, 1, 1, 1, None),              # n = 0
    lambda L: L.sgp4b_tle_columns(None, 100, 1, 1, 4, 1, 1, 1, None),           # null
    lambda L: L.sgp4b_code_rows(1, 0, 4, 4, 1, None),                           # n = 0
    lambda L: L.sgp4b_code_rows(1, 4, 8, 4, 1, None),                           # stride < m
    lambda L: L.sgp4b_code_rows(None, 4, 4, 4, 1, None),                        # null
])
def test_invalid_arguments_rejected(call):
    lib = _native.load()
    assert call(lib) == -1
    assert lib.sgp4b_last_error()  # message recorded


def _sass(function_pattern: str) -> str:
    """SASS of the library's functions whose mangled name matches."""
    import shutil
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", str(_native.library_path())], capture_output=True,
                         text=True, check=True).stdout
    blocks = re.split(r"\n\s*Function : ", out)
    return "\n".join(b for b in blocks if re.match(function_pattern, b))


def test_fp32_grid_kernel_sass_is_the_designed_one():
    """The shipped fp32 grid kernel is compiled for sm_100a with packed
    dual-fp32 arithmetic (FFMA2/FMUL2), SFU transcendentals (MUFU),
    evict-first 128-bit streaming stores, and no local-memory spills
    (DESIGN.md §3-4): a regression guard that needs no GPU."""
    sass = _sass(r"\S*grid_kernelIfLb1ELb0E")
    assert sass, "grid_kernel<float, true, false> not found"
    for op in ("FFMA2", "FMUL2", "MUFU.SIN", "MUFU.RSQ", "STG.E.EF.128"):
        assert op in sass, op
    assert "STL" not in sass and "LDL" not in sass
    # one satellite record load per row: 10 x 128-bit broadcast loads
    assert len(re.findall(r"LDG\.E\.128\.CONSTANT", sass)) >= 10
