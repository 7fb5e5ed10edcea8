"""ctypes binding of ``libsgp4b.so`` (the C ABI declared in include/sgp4b.h).

There is no CPU fallback: importing the compute entry points without the
built library, or calling them without a CUDA device, raises.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_NAME = "libsgp4b.so"
LIB_PATH = _HERE / LIB_NAME

SATREC_FIELDS = 33
RECORD_SLOTS = 40
ABI_VERSION = 7

#: every symbol include/sgp4b.h declares, in header order
EXPORTED_SYMBOLS = (
    "sgp4b_init",
    "sgp4b_pack",
    "sgp4b_propagate_grid",
    "sgp4b_propagate_pairs",
    "sgp4b_drift_norms",
    "sgp4b_drift_percentiles",
    "sgp4b_tle_columns",
    "sgp4b_code_rows",
    "sgp4b_solve_kepler",
    "sgp4b_peer_access",
    "sgp4b_host_alloc",
    "sgp4b_host_free",
    "sgp4b_last_error",
    "sgp4b_abi_version",
)

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_vp = ctypes.c_void_p

_SIGNATURES = {
    "sgp4b_init": (_c_int, [_vp, _c_i64, _vp, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "sgp4b_pack": (_c_int, [_vp, _vp, _vp, _c_i64, _vp, _c_int, _vp, _vp]),
    "sgp4b_propagate_grid": (_c_int, [_vp, _c_i64, _vp, _vp, _c_i64, ctypes.c_double, _c_int,
                                      _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _vp]),
    "sgp4b_propagate_pairs": (_c_int, [_vp, _vp, _vp, _vp, _c_i64, ctypes.c_double, _c_int,
                                       _vp, _vp, _vp, _vp]),
    "sgp4b_drift_norms": (_c_int, [_vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _vp, _vp]),
    "sgp4b_drift_percentiles": (_c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _vp, _vp, _vp]),
    "sgp4b_tle_columns": (_c_int, [_vp, _c_i64, _vp, _vp, _c_i64, _vp, _vp, _vp, _vp]),
    "sgp4b_code_rows": (_c_int, [_vp, _c_i64, _c_i64, _c_i64, _vp, _vp]),
    "sgp4b_solve_kepler": (_c_int, [_vp, _vp, _vp, _c_i64, _c_int, _vp, _vp]),
    "sgp4b_peer_access": (_c_int, [_c_int, _c_int]),
    "sgp4b_host_alloc": (_c_int, [_c_i64, ctypes.POINTER(_vp)]),
    "sgp4b_host_free": (_c_int, [_vp]),
    "sgp4b_last_error": (ctypes.c_char_p, []),
    "sgp4b_abi_version": (_c_int, []),
}


class NativeError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lib = None


def library_path() -> Path:
    override = os.environ.get("SGP4B_LIBRARY")
    return Path(override) if override else LIB_PATH


def load() -> ctypes.CDLL:
    """Load (once) and type the shared library; raise if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    path = library_path()
    if not path.exists():
        raise ImportError(
            f"{path} is not built; run `python -c 'import __graft_entry__ as g; "
            f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(str(path))
    for name, (restype, argtypes) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = restype
        fn.argtypes = argtypes
    if lib.sgp4b_abi_version() != ABI_VERSION:
        raise ImportError(f"{path}: ABI version {lib.sgp4b_abi_version()} != {ABI_VERSION}")
    _lib = lib
    return lib


def check(status: int) -> None:
    if status != 0:
        msg = load().sgp4b_last_error().decode(errors="replace")
        raise NativeError(f"sgp4b status {status}: {msg}")


def ptr(tensor) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    if tensor is None:
        return None
    return tensor.data_ptr()


def stream_handle(torch_stream) -> int:
    return torch_stream.cuda_stream
