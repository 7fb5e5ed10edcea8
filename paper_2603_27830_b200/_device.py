"""Device-side satrec state and the thin calls onto the C ABI.

PyTorch is used only as the CUDA allocator / stream provider; every number
is computed by libsgp4b.so.  Nothing here falls back to the CPU: without a
CUDA device the calls raise.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .gravity import GravityModel

SATREC_FIELDS = _native.SATREC_FIELDS
RECORD_SLOTS = _native.RECORD_SLOTS
MAX_INIT_CODE = (1 << 23) - 1        # width of the record's persistent-code field


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError(
            "paper_2603_27830_b200 needs a CUDA device (B200, sm_100a); "
            "there is no CPU fallback")
    _native.load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {device}")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


def torch_dtype(precision: int) -> torch.dtype:
    return torch.float32 if precision == 32 else torch.float64


def np_dtype(precision: int):
    return np.float32 if precision == 32 else np.float64


def precision_of(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return 32
    if dt == np.float64:
        return 64
    raise ValueError(f"dtype must be float32 or float64, got {dt}")


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


@dataclass
class DeviceSatrec:
    """All per-satellite state of one batch, resident on one GPU.

    satrec : (33, n) fp64, SatInit float fields in dataclass order.  The
             propagate path needs only the records, so batches built from
             element columns write it on first use (a second init launch over
             the kept columns, bit-identical) instead of at init time.
    codes  : (n,) int32 error_code_at_init
    isimp  : (n,) uint8
    record : (n, 40) packed propagate records at the batch precision
    """

    _satrec: torch.Tensor | None
    codes: torch.Tensor
    isimp: torch.Tensor
    record: torch.Tensor
    precision: int
    grav: GravityModel
    device: torch.device
    elements: torch.Tensor | None = None      # (7, n) fp64 init input, for the lazy satrec

    @property
    def n(self) -> int:
        return int(self.codes.shape[0])

    @property
    def satrec(self) -> torch.Tensor | None:
        if self._satrec is None and self.elements is not None:
            self._satrec = _satrec_of(self.elements, self.grav, self.device)
        return self._satrec


_GRAV_CACHE: dict = {}


def _grav_host(grav: GravityModel, device) -> np.ndarray:
    # the C ABI reads grav[8] on the host (kernel launch parameter)
    key = (grav, str(device))
    arr = _GRAV_CACHE.get(key)
    if arr is None:
        arr = grav.as_array()
        _GRAV_CACHE[key] = arr
    return arr


def _host_ptr(arr: np.ndarray) -> int:
    return arr.ctypes.data


def init_device(elements: np.ndarray, grav: GravityModel, precision: int,
                device=None) -> DeviceSatrec:
    """(7, n) fp64 element columns -> DeviceSatrec via the init kernel."""
    device = require_cuda(device)
    elements = np.ascontiguousarray(elements, dtype=np.float64)
    if not elements.flags.writeable:                  # torch.from_numpy wants writable
        elements = elements.copy()
    n = elements.shape[1]
    el = torch.from_numpy(elements).to(device, non_blocking=False)
    return init_device_tensor(el, grav, precision, device)


def init_device_tensor(el: torch.Tensor, grav: GravityModel, precision: int,
                       device=None) -> DeviceSatrec:
    """Same as :func:`init_device` for (7, n) fp64 columns already on the GPU
    (the columns are kept: the public satrec is written on first use)."""
    device = require_cuda(device if device is not None else el.device)
    n = int(el.shape[1])
    codes = torch.empty((n,), dtype=torch.int32, device=device)
    isimp = torch.empty((n,), dtype=torch.uint8, device=device)
    record = torch.empty((n, RECORD_SLOTS), dtype=torch_dtype(precision), device=device)
    g = _grav_host(grav, device)
    with torch.cuda.device(device):
        _native.check(_native.load().sgp4b_init(
            el.data_ptr(), n, _host_ptr(g), precision, None,
            codes.data_ptr(), isimp.data_ptr(), record.data_ptr(), _stream(device)))
    return DeviceSatrec(None, codes, isimp, record, precision, grav, device, elements=el)


def _satrec_of(el: torch.Tensor, grav: GravityModel, device) -> torch.Tensor:
    """The (33, n) fp64 satrec of element columns (init kernel, no records)."""
    n = int(el.shape[1])
    satrec = torch.empty((SATREC_FIELDS, n), dtype=torch.float64, device=device)
    codes = torch.empty((n,), dtype=torch.int32, device=device)
    isimp = torch.empty((n,), dtype=torch.uint8, device=device)
    g = _grav_host(grav, device)
    with torch.cuda.device(device):
        _native.check(_native.load().sgp4b_init(
            el.data_ptr(), n, _host_ptr(g), 64, satrec.data_ptr(), codes.data_ptr(),
            isimp.data_ptr(), None, _stream(device)))
    return satrec


def pack_device(satrec64: np.ndarray, codes: np.ndarray, isimp: np.ndarray,
                grav: GravityModel, precision: int, device=None) -> DeviceSatrec:
    """Host SoA fields (e.g. from a user-built SatInit) -> packed records."""
    codes_i = np.asarray(codes)
    if codes_i.size and (codes_i.min() < 0 or codes_i.max() > MAX_INIT_CODE):
        # the packed record carries the persistent code in 23 bits; the
        # reference keeps any nonzero code, so out-of-range ones are refused
        # rather than silently wrapped to another value
        raise ValueError(f"error_code_at_init must be in [0, {MAX_INIT_CODE}], got "
                         f"[{int(codes_i.min())}, {int(codes_i.max())}]")
    device = require_cuda(device)
    n = satrec64.shape[1]
    # np.array copies: the SatInit fields may be read-only views
    sr = torch.from_numpy(np.array(satrec64, dtype=np.float64, order="C")).to(device)
    cd = torch.from_numpy(np.array(codes, dtype=np.int32, order="C")).to(device)
    si = torch.from_numpy(np.array(isimp, dtype=np.uint8, order="C")).to(device)
    record = torch.empty((n, RECORD_SLOTS), dtype=torch_dtype(precision), device=device)
    g = _grav_host(grav, device)
    with torch.cuda.device(device):
        _native.check(_native.load().sgp4b_pack(
            sr.data_ptr(), cd.data_ptr(), si.data_ptr(), n, _host_ptr(g), precision,
            record.data_ptr(), _stream(device)))
    return DeviceSatrec(sr, cd, si, record, precision, grav, device)


def times_absmax(times) -> float:
    """max |t| of a time vector (host array or device tensor; a device
    tensor costs one reduction and a sync)."""
    if isinstance(times, torch.Tensor):
        return float(times.detach().abs().max().item()) if times.numel() else 0.0
    t = np.asarray(times)
    # no |t| temporary: the streamed API keeps host allocations O(1) in M
    return max(float(t.max()), -float(t.min())) if t.size else 0.0


#: longest row one grid launch takes (sgp4b.h)
MAX_STEPS_PER_LAUNCH = 1 << 30


def propagate_grid(dev: DeviceSatrec, times: torch.Tensor, planes: torch.Tensor,
                   codes: torch.Tensor, times_lo: torch.Tensor | None = None,
                   rows: tuple[int, int] | None = None, t_absmax: float | None = None) -> None:
    """Launch the grid kernel: planes (6, n, m) and codes (n, m) device
    tensors (any strides with unit column stride) receive the grid.

    ``rows=(r0, r1)`` propagates only satellites r0..r1 into row 0.. of the
    outputs (used by tiling and by the streamed API).  ``t_absmax`` is an
    upper bound on |times| (fp32 Kepler-class validity, see sgp4b.h); it is
    computed from ``times`` when not given.
    """
    if t_absmax is None:
        t_absmax = times_absmax(times) if dev.precision == 32 else float("inf")
    r0, r1 = rows if rows is not None else (0, dev.n)
    n = r1 - r0
    m = int(times.shape[0])
    if planes.stride(2) != 1 or codes.stride(1) != 1:
        raise ValueError("output columns must be contiguous")
    rec = dev.record[r0:r1]
    g = _grav_host(dev.grav, dev.device)
    # the kernels index columns with 32-bit offsets (sgp4b.h: m <= 2^30);
    # longer rows run as column blocks of the same grid
    for c0 in range(0, m, MAX_STEPS_PER_LAUNCH):
        c1 = min(m, c0 + MAX_STEPS_PER_LAUNCH)
        tl = times_lo[c0:c1] if times_lo is not None else None
        _native.check(_native.load().sgp4b_propagate_grid(
            rec.data_ptr(), n, times[c0:c1].data_ptr(), _native.ptr(tl), c1 - c0,
            float(t_absmax), dev.precision, _host_ptr(g), planes[:, :, c0:].data_ptr(),
            planes.stride(0), planes.stride(1), codes[:, c0:].data_ptr(), codes.stride(0),
            _stream(dev.device)))


def propagate_pairs(dev: DeviceSatrec, sat_idx: torch.Tensor, times: torch.Tensor,
                    rv: torch.Tensor, codes: torch.Tensor, t_absmax: float | None = None) -> None:
    p = int(times.shape[0])
    g = _grav_host(dev.grav, dev.device)
    if t_absmax is None:
        t_absmax = times_absmax(times) if dev.precision == 32 else float("inf")
    _native.check(_native.load().sgp4b_propagate_pairs(
        dev.record.data_ptr(), sat_idx.data_ptr(), times.data_ptr(), None, p, float(t_absmax),
        dev.precision, _host_ptr(g), rv.data_ptr(), codes.data_ptr(),
        _stream(dev.device)))


def solve_kepler_device(axnl: torch.Tensor, aynl: torch.Tensor, u: torch.Tensor,
                        precision: int) -> torch.Tensor:
    out = torch.empty_like(u)
    _native.check(_native.load().sgp4b_solve_kepler(
        axnl.data_ptr(), aynl.data_ptr(), u.data_ptr(), int(u.numel()), precision,
        out.data_ptr(), _stream(u.device)))
    return out


def code_rows(codes: torch.Tensor, flags: torch.Tensor) -> None:
    """flags[i] (uint8) = 1 when row i of the (n, m) int32 code plane holds
    a nonzero code (``sgp4b_code_rows``)."""
    n, m = int(codes.shape[0]), int(codes.shape[1])
    if codes.dtype != torch.int32 or codes.stride(1) != 1:
        raise ValueError("codes must be an int32 (n, m) plane with contiguous columns")
    if flags.dtype != torch.uint8 or flags.numel() < n or flags.device != codes.device:
        raise ValueError("flags must be a uint8 tensor of n entries on the codes' device")
    _native.check(_native.load().sgp4b_code_rows(
        codes.data_ptr(), n, m, codes.stride(0), flags.data_ptr(), _stream(codes.device)))
