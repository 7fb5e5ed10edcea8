"""Batch API (mirror of sgp4kit.batch, batch.py:54-269), GPU-backed.

``init_batch`` runs one init kernel over the whole catalogue and leaves the
packed satrec resident on the GPU; ``propagate_batch`` runs one grid kernel
that writes the reference's (6, N, M) planes + (N, M) int32 codes layout
directly, then copies it to pinned host memory.  ``propagate_batch_device``
is the same call with the grid left in HBM (torch tensors), the form the
multi-GPU sharding and the throughput benchmark use.
"""

from __future__ import annotations

import ctypes
import struct
import sys
from dataclasses import dataclass
from typing import Any, Callable, Sequence

import numpy as np
import torch

from . import _device, _hostmem, _native
from .gravity import WGS72, GravityModel
from .kernel import SatInit, satinit_from_device, _device_of
from .tle import MeanElements, elements_to_columns

PLANE_NAMES = ("rx", "ry", "rz", "vx", "vy", "vz")

MAGIC = b"SGB1"
_HEADER = struct.Struct("<4sQQI8s")        # magic, N, M, precision bits, tag
PLANE_ORDER_TAG = b"rrrvvve\x00"

DEFAULT_TILE_CELLS = 1 << 18


class GridAllocationError(MemoryError):
    """The output grid could not be allocated (batch.py:33-41)."""

    def __init__(self, n: int, m: int, nbytes: int):
        super().__init__(f"cannot allocate {n}x{m} output grid ({nbytes} bytes)")
        self.n = n
        self.m = m
        self.nbytes = nbytes


class StreamAborted(RuntimeError):
    """A streaming sink raised; carries the tiles already delivered."""

    def __init__(self, tiles_completed: int, cause: BaseException):
        super().__init__(f"sink failed after {tiles_completed} tiles: {cause}")
        self.tiles_completed = tiles_completed
        self.__cause__ = cause


class SatBatch:
    """Structure-of-arrays satellite batch of length ``n`` (batch.py:54-63).

    Holds the GPU-resident satrec; ``.init`` materialises the host
    :class:`SatInit` on first access.
    """

    def __init__(self, init: SatInit | None = None, n: int | None = None, *,
                 device_satrec: "_device.DeviceSatrec | None" = None):
        if device_satrec is None:
            if init is None:
                raise ValueError("SatBatch needs init or device_satrec")
            device_satrec, shape = _device_of(init)
            if len(shape) != 1:
                raise ValueError("SatBatch init fields must be 1-D")
        self._dev = device_satrec
        self._init = init
        self.n = int(n if n is not None else device_satrec.n)
        if self.n != device_satrec.n:
            raise ValueError(f"n={self.n} does not match the satrec length {device_satrec.n}")

    @property
    def device_satrec(self) -> "_device.DeviceSatrec":
        return self._dev

    @property
    def precision(self) -> int:
        return self._dev.precision

    @property
    def dtype(self):
        return _device.np_dtype(self._dev.precision)

    @property
    def init(self) -> SatInit:
        if self._init is None:
            self._init = satinit_from_device(self._dev, (self.n,))
        return self._init

    @property
    def error_codes(self) -> np.ndarray:
        return self._dev.codes.cpu().numpy().astype(np.int32)

    def __repr__(self) -> str:
        return f"SatBatch(n={self.n}, precision={self.precision}, device={self._dev.device})"


@dataclass(frozen=True)
class BatchResult:
    """Dense grid: planes (6, N, M) and error codes (N, M) (batch.py:66-81)."""

    planes: Any
    error: Any
    n: int
    m: int

    @property
    def r(self):
        return _moveaxis(self.planes[:3])

    @property
    def v(self):
        return _moveaxis(self.planes[3:])


def _moveaxis(x):
    if isinstance(x, torch.Tensor):
        return torch.movedim(x, 0, -1)
    return np.moveaxis(x, 0, -1)


def _precision(precision: int) -> int:
    if precision not in (32, 64):
        raise ValueError(f"precision must be 32 or 64, got {precision}")
    return precision


def init_batch(elements: Sequence[MeanElements], grav: GravityModel = WGS72,
               precision: int = 64, device=None) -> SatBatch:
    """Initialise many satellites at once (batch.py:92-109) on the GPU.

    ``elements`` may also be a (7, n) fp64 array in ELEMENT_COLUMNS order
    (e.g. from :func:`~paper_2603_27830_b200.tle.parse_catalog_columns`).
    Never raises on bad elements: codes land in ``.error_codes``.
    """
    if isinstance(elements, torch.Tensor):
        # (7, n) columns already on a GPU (e.g. ingest.read_catalog_columns)
        if elements.dim() != 2 or elements.shape[0] != 7:
            raise ValueError("element columns must have shape (7, n)")
        if elements.shape[1] == 0:
            raise ValueError("empty element list")
        if not elements.is_cuda:
            elements = elements.numpy()
        else:
            # a private copy: the batch keeps its columns (lazy satrec)
            el = elements.to(torch.float64).contiguous().clone()
            dev = _device.init_device_tensor(el, grav, _precision(precision), device)
            return SatBatch(device_satrec=dev)
    if isinstance(elements, np.ndarray):
        cols = np.asarray(elements, dtype=np.float64)
        if cols.ndim != 2 or cols.shape[0] != 7:
            raise ValueError("element columns must have shape (7, n)")
        if cols.shape[1] == 0:
            raise ValueError("empty element list")
    else:
        if not elements:
            raise ValueError("empty element list")
        cols = elements_to_columns(elements)
    precision = _precision(precision)
    dev = _device.init_device(cols, grav, precision, device)
    return SatBatch(device_satrec=dev)


def _times(sats: SatBatch, times) -> np.ndarray:
    # the caller's array when it already is a contiguous, writable vector of
    # the batch dtype (e.g. in pinned memory: its H2D is then a plain DMA);
    # otherwise a cast copy.  Every use completes before the call returns.
    t = np.asarray(times, dtype=sats.dtype)
    if not (t.flags.c_contiguous and t.flags.writeable):
        t = np.array(t)
    if t.ndim != 1 or t.size == 0:
        raise ValueError("times must be a non-empty 1-D array")
    return t


def _alloc_grid(n: int, m: int, precision: int, device, pin: bool = False):
    """Output grid.  On the device, rows are padded to a multiple of 4 steps
    (returned as (6, n, m) / (n, m) views) so the grid kernel always runs its
    vectorised instance — the one the scalar API shares, which keeps
    batch == scalar bit for bit."""
    tdt = _device.torch_dtype(precision)
    itemsize = 4 if precision == 32 else 8
    try:
        if device == "cpu":
            planes = torch.empty((6, n, m), dtype=tdt, pin_memory=pin)
            error = torch.empty((n, m), dtype=torch.int32, pin_memory=pin)
        else:
            m4 = -(-m // 4) * 4
            planes = torch.empty((6, n, m4), dtype=tdt, device=device)[:, :, :m]
            error = torch.empty((n, m4), dtype=torch.int32, device=device)[:, :m]
    except (torch.cuda.OutOfMemoryError, RuntimeError, MemoryError) as exc:
        if isinstance(exc, RuntimeError) and "memory" not in str(exc).lower():
            raise
        raise GridAllocationError(n, m, 6 * n * m * itemsize + 4 * n * m) from None
    return planes, error


def propagate_batch_device(sats: SatBatch, times, out: tuple | None = None,
                           times_lo=None, t_absmax: float | None = None,
                           devices=None) -> BatchResult:
    """Propagate every satellite to every time, leaving the grid in HBM.

    ``times`` is a 1-D array/tensor (cast to the batch dtype); ``out`` may
    supply preallocated (planes, error) device tensors.  ``times_lo``
    (fp32 batches only) carries the low words of fp64 times for the
    double-float secular stage.  ``t_absmax`` may give max |times| when the
    caller knows it (device-tensor times are otherwise reduced on the device,
    one sync).  ``devices`` spreads the satellites over several GPUs of this
    process; the grid still lands on the batch's device (see
    :func:`_propagate_device_multi`).  Returns a BatchResult of torch tensors.
    """
    devices = list(devices) if devices is not None else []
    if devices:
        if times_lo is not None:
            raise ValueError("times_lo is not supported with devices=")
        return _propagate_device_multi(sats, times, out, t_absmax, devices)
    dev = sats.device_satrec
    with torch.cuda.device(dev.device):
        if isinstance(times, torch.Tensor):
            t_d = times.to(device=dev.device, dtype=_device.torch_dtype(dev.precision))
            if t_d.ndim != 1 or t_d.numel() == 0:
                raise ValueError("times must be a non-empty 1-D array")
        else:
            t_h = _times(sats, times)
            if t_absmax is None:
                t_absmax = _device.times_absmax(t_h)
            t_d = torch.from_numpy(t_h).to(dev.device)
        t_d = t_d.contiguous()
        if t_d.data_ptr() % 16:              # the vector path wants 16-B aligned times
            t_d = t_d.clone()
        m = int(t_d.shape[0])
        if times_lo is not None:
            times_lo = _check_times_lo(times_lo, t_d, dev.precision)
        if out is None:
            planes, error = _alloc_grid(sats.n, m, dev.precision, dev.device)
        else:
            planes, error = _check_out(out, sats.n, m, dev.precision, dev.device)
        _device.propagate_grid(dev, t_d, planes, error, times_lo=times_lo, t_absmax=t_absmax)
    return BatchResult(planes=planes, error=error, n=sats.n, m=m)


def _propagate_device_multi(sats: SatBatch, times, out, t_absmax, devices) -> BatchResult:
    """The grid on the batch's (home) device, computed by several GPUs: each
    takes a balanced satellite range (``partition_work``'s rule), runs the
    grid kernel on its own stream, and — with NVLink peer access — stores its
    rows straight into the home device's grid (the kernel's output pointers
    are the peer's memory: no separate gather).  Without peer access a
    device computes into local memory and its rows are copied over.  Cells
    are bitwise equal to the single-device grid."""
    from .shard import shard_bounds
    dev = sats.device_satrec
    home = dev.device
    devs = _devices(devices)
    t = times.detach().cpu().numpy() if isinstance(times, torch.Tensor) else times
    t = _times(sats, t)
    n, m = sats.n, t.size
    if t_absmax is None:
        t_absmax = _device.times_absmax(t)
    lib = _native.load()
    with torch.cuda.device(home):
        if out is None:
            planes, error = _alloc_grid(n, m, dev.precision, home)
        else:
            planes, error = _check_out(out, n, m, dev.precision, home)
        home_stream = torch.cuda.current_stream(home)
        ready = torch.cuda.Event()
        ready.record(home_stream)            # records and the output exist
    jobs = []
    for g, d in enumerate(devs):
        lo, hi = shard_bounds(n, len(devs), g)
        if hi <= lo:
            continue
        direct = d == home or lib.sgp4b_peer_access(d.index, home.index) == 0
        with torch.cuda.device(d):
            stream = torch.cuda.Stream(d)
            stream.wait_event(ready)
            with torch.cuda.stream(stream):
                sub = _shard_satrec(dev, lo, hi, d)
                t_d = torch.from_numpy(t).to(d, non_blocking=True)
                if direct:
                    # rows lo..hi of the home grid, written from device d
                    _device.propagate_grid(sub, t_d, planes[:, lo:hi], error[lo:hi],
                                           t_absmax=t_absmax)
                    local = None
                else:
                    local = _alloc_grid(hi - lo, m, dev.precision, d)
                    _device.propagate_grid(sub, t_d, local[0], local[1], t_absmax=t_absmax)
                done = torch.cuda.Event()
                done.record(stream)
        jobs.append((d, stream, done, lo, hi, local, sub, t_d))
    with torch.cuda.device(home):
        for d, stream, done, lo, hi, local, *_ in jobs:
            home_stream.wait_event(done)
            if local is not None:
                planes[:, lo:hi].copy_(local[0], non_blocking=True)
                error[lo:hi].copy_(local[1], non_blocking=True)
                for x in local:                  # read by the home stream
                    x.record_stream(home_stream)
    for _, stream, *_ in jobs:
        stream.synchronize()                 # shard inputs/temporaries outlive their use
    return BatchResult(planes=planes, error=error, n=n, m=m)


def _check_out(out, n: int, m: int, precision: int, device):
    """Caller-supplied (planes, error) device tensors: shapes (6, n, m) and
    (n, m), the batch dtype and int32, on the batch's device, unit column
    stride.  Anything else would let the kernel write outside the buffers."""
    try:
        planes, error = out
    except (TypeError, ValueError):
        raise ValueError("out must be a (planes, error) pair of device tensors") from None
    if not isinstance(planes, torch.Tensor) or not isinstance(error, torch.Tensor):
        raise TypeError("out tensors must be torch tensors")
    if tuple(planes.shape) != (6, n, m) or tuple(error.shape) != (n, m):
        raise ValueError(f"out shapes {tuple(planes.shape)} / {tuple(error.shape)} do not match "
                         f"(6, {n}, {m}) / ({n}, {m})")
    if planes.dtype != _device.torch_dtype(precision) or error.dtype != torch.int32:
        raise TypeError(f"out dtypes must be {_device.torch_dtype(precision)} and int32, "
                        f"got {planes.dtype} and {error.dtype}")
    if planes.device != device or error.device != device:
        raise ValueError(f"out tensors must live on {device}")
    if planes.stride(2) != 1 or error.stride(1) != 1:
        raise ValueError("out tensors need a unit column stride")
    if min(planes.stride(0), planes.stride(1), error.stride(0)) < 0:
        raise ValueError("out tensors must not have negative strides")
    return planes, error


def _check_times_lo(times_lo, t_d: torch.Tensor, precision: int) -> torch.Tensor:
    """Low words of fp64 times for an fp32 batch: float32, same length and
    device as the times, contiguous."""
    if precision != 32:
        raise ValueError("times_lo is only meaningful for fp32 batches")
    if not isinstance(times_lo, torch.Tensor):
        times_lo = torch.as_tensor(np.asarray(times_lo, dtype=np.float32))
    if times_lo.dtype != torch.float32:
        raise TypeError(f"times_lo must be float32, got {times_lo.dtype}")
    if times_lo.ndim != 1 or times_lo.shape[0] != t_d.shape[0]:
        raise ValueError(f"times_lo must have shape ({t_d.shape[0]},), got {tuple(times_lo.shape)}")
    return times_lo.to(t_d.device).contiguous()


def split_times(times) -> tuple[np.ndarray, np.ndarray]:
    """fp64 minutes -> (hi, lo) float32 words with hi + lo == t to ~2^-48
    relative: the ``times`` / ``times_lo`` pair of an fp32 batch whose
    secular stage should see the caller's fp64 times."""
    t = np.asarray(times, dtype=np.float64)
    hi = t.astype(np.float32)
    lo = (t - hi.astype(np.float64)).astype(np.float32)
    return hi, lo


def _shard_satrec(dev: "_device.DeviceSatrec", lo: int, hi: int, device) -> "_device.DeviceSatrec":
    """Rows lo..hi of a batch's packed records on ``device`` (a peer copy
    over NVLink when it is another GPU; 160/320 bytes per satellite)."""
    rec = dev.record[lo:hi]
    codes = dev.codes[lo:hi]
    if torch.device(device) != dev.device:
        rec = rec.to(device, non_blocking=True)
        codes = codes.to(device, non_blocking=True)
    return _device.DeviceSatrec(None, codes=codes, isimp=None, record=rec,
                                precision=dev.precision, grav=dev.grav,
                                device=torch.device(device))


def _devices(devices) -> list:
    out = []
    for d in devices:
        d = torch.device("cuda", d) if isinstance(d, int) else torch.device(d)
        out.append(_device.require_cuda(d))
    if not out:
        raise ValueError("devices must name at least one CUDA device")
    return out


def propagate_batch_multi(sats: SatBatch, times, devices) -> BatchResult:
    """``propagate_batch`` over several GPUs of this process (reference
    batch.py:125-141, 193-204: the grid is partitioned into balanced
    satellite ranges, ``partition_work``'s rule, and computed concurrently).

    Each device gets its rows' packed records (peer copy), runs the grid
    kernel on its own stream, and copies its rows straight into one pinned
    host grid over its own PCIe link, so the D2H — the bound of the
    single-GPU path — runs on all links at once.  Cells are bitwise equal to
    the single-device result (no collective, satellites are independent).
    """
    t = _times(sats, times)
    dev = sats.device_satrec
    n, m = sats.n, t.size
    devs = _devices(devices)
    itemsize = 4 if dev.precision == 32 else 8
    staged = not _hostmem.worth_pinning(n * m * (6 * itemsize + 4) + n)
    planes_h, error_h, flags_h = (_host_grid_pageable if staged else _host_grid)(n, m,
                                                                                 dev.precision)
    t_abs = _device.times_absmax(t)
    src_stream = torch.cuda.current_stream(dev.device)
    ready = torch.cuda.Event()
    ready.record(src_stream)                  # the records exist on the source device
    jobs = []
    from .shard import shard_bounds
    # every device's grid kernel and code-row flags are queued first, so the
    # kernels run concurrently; the copies follow (a staged copy may block
    # the host while its ring cycles)
    for g, d in enumerate(devs):
        lo, hi = shard_bounds(n, len(devs), g)
        if hi <= lo:
            continue
        with torch.cuda.device(d):
            stream = torch.cuda.Stream(d)
            stream.wait_event(ready)
            with torch.cuda.stream(stream):
                sub = _shard_satrec(dev, lo, hi, d)
                t_d = torch.from_numpy(t).to(d, non_blocking=True)
                planes, error = _alloc_grid(hi - lo, m, dev.precision, d)
                _device.propagate_grid(sub, t_d, planes, error, t_absmax=t_abs)
                stager = _StagedD2H(stream, ring=max(4, _StagedD2H.RING // len(devs))) \
                    if staged else None
                codes = _CodesToHost(error, error_h[lo:hi], flags_h[lo:hi], stream, stager)
            jobs.append((stream, codes, stager, lo, hi, sub, t_d, planes, error))
    try:
        for stream, codes, stager, lo, hi, sub, t_d, planes, error in jobs:
            with torch.cuda.device(stream.device), torch.cuda.stream(stream):
                for p in range(6):
                    if stager is not None:
                        stager.copy(planes[p], planes_h[p, lo:hi])
                    else:
                        torch.from_numpy(planes_h[p, lo:hi]).copy_(planes[p], non_blocking=True)
        for stream, codes, *_ in jobs:
            with torch.cuda.device(stream.device), torch.cuda.stream(stream):
                codes.finish()
        for stream, codes, stager, *_ in jobs:
            if stager is not None:
                stager.join()
            stream.synchronize()
    finally:
        for _, codes, stager, *_ in jobs:
            codes.join()
            if stager is not None:
                stager.join()
    return BatchResult(planes=planes_h, error=error_h, n=n, m=m)


def propagate_batch(sats: SatBatch, times, workers: int | None = None,
                    devices=None) -> BatchResult:
    """Propagate every satellite to every time (batch.py:166-205).

    Cell (i, j) is bitwise equal to ``sgp4_propagate`` of satellite i at
    time j at the batch precision.  ``workers`` is accepted for API
    compatibility; it never affected output and the GPU needs no pool.
    Returns numpy arrays, fully materialised: the planes and the int32 code
    plane are copied from HBM into one page-locked host block (pooled at its
    exact size, see ``_hostmem``) that is released with the arrays.
    ``devices`` (e.g. ``range(torch.cuda.device_count())``) spreads the
    satellites over several GPUs of this process (``propagate_batch_multi``).
    """
    devices = list(devices) if devices is not None else []
    if devices:
        return propagate_batch_multi(sats, times, devices)
    t = _times(sats, times)
    dev = sats.device_satrec
    n, m = sats.n, t.size
    itemsize = 4 if dev.precision == 32 else 8
    staged = not _hostmem.worth_pinning(n * m * (6 * itemsize + 4) + n)
    planes_h, error_h, flags_h = (_host_grid_pageable if staged else _host_grid)(n, m,
                                                                                 dev.precision)
    with torch.cuda.device(dev.device):
        stream = torch.cuda.current_stream(dev.device)
        t_d = torch.from_numpy(t).to(dev.device, non_blocking=True)
        res = propagate_batch_device(sats, t_d, t_absmax=_device.times_absmax(t))
        stager = _StagedD2H(stream) if staged else None
        codes = _CodesToHost(res.error, error_h, flags_h, stream, stager)
        try:
            if stager is not None:
                for p in range(6):
                    stager.copy(res.planes[p], planes_h[p])
            else:
                torch.from_numpy(planes_h).copy_(res.planes, non_blocking=True)
            codes.finish()
            if stager is not None:
                stager.join()
            stream.synchronize()
        finally:
            codes.join()            # no fill may outlive the call (the block is pooled)
            if stager is not None:
                stager.join()
    _last_transfer.update(d2h_bytes=planes_h.nbytes + codes.d2h_bytes,
                          code_bytes_zero_filled=error_h.nbytes - (codes.d2h_bytes - flags_h.nbytes))
    return BatchResult(planes=planes_h, error=error_h, n=n, m=m)


_last_transfer: dict = {}


def last_transfer() -> dict:
    """Device->host bytes the last single-device ``propagate_batch`` moved
    (planes + code-row flags + flagged code rows) and the code-plane bytes it
    zero-filled on the host instead."""
    return dict(_last_transfer)


def flag_runs(flags: np.ndarray, max_runs: int) -> list[tuple[int, int]]:
    """Half-open row ranges [a, b) covering the rows whose flag is set, in
    order; the whole range [(0, n)] when there are more than ``max_runs``
    runs or more than half the rows are flagged (one copy is then cheaper)."""
    n = int(flags.shape[0])
    rows = np.flatnonzero(flags)
    if rows.size == 0:
        return []
    if rows.size * 2 > n:
        return [(0, n)]
    cut = np.flatnonzero(np.diff(rows) != 1) + 1
    if cut.size + 1 > max_runs:
        return [(0, n)]
    starts = rows[np.r_[0, cut]]
    ends = rows[np.r_[cut - 1, rows.size - 1]] + 1
    return list(zip(starts.tolist(), ends.tolist()))


class _CodesToHost:
    """D2H of an (n, m) int32 code plane that moves only the rows holding a
    nonzero code.  ``__init__`` (before the planes' D2H is queued) runs
    ``sgp4b_code_rows`` and copies the n row flags; ``finish`` waits for the
    flags (they land a few µs after the grid kernel, while the planes are
    still crossing PCIe), queues one D2H per run of flagged rows and
    zero-fills every other row in host memory on a thread pool; ``join``
    waits for the fills.  Every element of the host plane is written before
    the caller returns; with many scattered flagged rows the whole plane is
    copied instead."""

    MAX_RUNS = 64

    def __init__(self, error_d: torch.Tensor, error_h: np.ndarray, flags_h: np.ndarray, stream,
                 stager: "_StagedD2H | None" = None):
        self.error_d, self.error_h, self.flags_h, self.stream = error_d, error_h, flags_h, stream
        self.stager = stager
        self.fills = []
        n = error_d.shape[0]
        flags_d = torch.empty(n, dtype=torch.uint8, device=error_d.device)
        _device.code_rows(error_d, flags_d)
        torch.from_numpy(flags_h).copy_(flags_d, non_blocking=True)
        self.ready = torch.cuda.Event()
        self.ready.record(stream)
        self._keep = flags_d

    def finish(self) -> None:
        self.ready.synchronize()
        n = self.error_h.shape[0]
        runs = flag_runs(self.flags_h, self.MAX_RUNS)
        row_bytes = self.error_h.strides[0]
        self.d2h_bytes = self.flags_h.nbytes + sum(b - a for a, b in runs) * row_bytes
        lo = 0
        for a, b in runs:
            if self.stager is not None:
                self.stager.copy(self.error_d[a:b], self.error_h[a:b])
            else:
                torch.from_numpy(self.error_h[a:b]).copy_(self.error_d[a:b], non_blocking=True)
            self.fills += _hostmem.zero_fill_async(self.error_h, lo, a)
            lo = b
        self.fills += _hostmem.zero_fill_async(self.error_h, lo, n)

    def join(self) -> None:
        """Wait for every zero fill (all of them, even if one raised)."""
        fills, self.fills = self.fills, []
        errors = [f.exception() for f in fills]
        for e in errors:
            if e is not None:
                raise e


def _host_grid_pageable(n: int, m: int, precision: int):
    """Pageable (6, n, m) planes + (n, m) codes, as the reference allocates
    them (batch.py:177-183), for grids above the pinned pool's cache limit:
    page-locking a multi-GB block costs ~0.4 s/GB, far more than staging
    through pinned buffers.  The row flags stay pinned (tiny)."""
    try:
        planes = np.empty((6, n, m), dtype=_device.np_dtype(precision))
        error = np.empty((n, m), dtype=np.int32)
    except MemoryError:
        itemsize = 4 if precision == 32 else 8
        raise GridAllocationError(n, m, 6 * n * m * itemsize + 4 * n * m) from None
    flags = _hostmem.empty([((n,), np.uint8)])[0]
    return planes, error, flags


class _StagedD2H:
    """Device -> pageable host copies through a ring of pinned staging
    buffers: piece k crosses PCIe into buffer k mod R while worker threads
    move the earlier pieces into place (``ctypes.memmove`` releases the GIL),
    so the DMA and the host copies (page faults included) overlap.  Sources
    and destinations are C-contiguous; ``join`` waits for every piece."""

    PIECE = 32 << 20
    RING = 24

    def __init__(self, stream, ring: int | None = None):
        self.stream = stream
        self.nring = ring or self.RING
        self.ring = [np.asarray(_hostmem.alloc(self.PIECE)) for _ in range(self.nring)]
        self.events = [torch.cuda.Event() for _ in range(self.nring)]
        self.pending = [None] * self.nring
        self.k = 0

    @staticmethod
    def _drain(event, buf, dst_addr, nbytes):
        event.synchronize()
        ctypes.memmove(dst_addr, buf.ctypes.data, nbytes)

    def _piece(self, src: torch.Tensor, dst_addr: int, nbytes: int) -> None:
        """One D2H of ``src`` (any strides; ``nbytes`` of payload) into the
        next staging buffer, then an async move to ``dst_addr``."""
        k = self.k
        self.k = (k + 1) % self.nring
        if self.pending[k] is not None:
            self.pending[k].result()                # buffer k drained
        buf = self.ring[k]
        view = torch.from_numpy(buf[:nbytes]).view(src.dtype).view(src.shape)
        view.copy_(src, non_blocking=True)
        self.events[k].record(self.stream)
        self.pending[k] = _hostmem._pool().submit(self._drain, self.events[k], buf, dst_addr,
                                                  nbytes)

    def copy(self, src: torch.Tensor, dst: np.ndarray) -> None:
        """``src`` (rows, cols) on the device with unit column stride (row
        stride free: padded grids), ``dst`` the C-contiguous host rows."""
        if src.dim() != 2 or src.stride(1) != 1 or not dst.flags.c_contiguous \
                or tuple(src.shape) != dst.shape or src.element_size() != dst.itemsize:
            raise ValueError("staged copy: (rows, cols) source with unit column stride and a "
                             "C-contiguous destination of the same shape and item size")
        rows, cols = dst.shape
        row_bytes = cols * dst.itemsize
        base = dst.ctypes.data
        if row_bytes <= self.PIECE:
            step = self.PIECE // row_bytes
            for r0 in range(0, rows, step):
                r1 = min(rows, r0 + step)
                self._piece(src[r0:r1], base + r0 * row_bytes, (r1 - r0) * row_bytes)
        else:
            step = self.PIECE // dst.itemsize
            for r in range(rows):
                for c0 in range(0, cols, step):
                    c1 = min(cols, c0 + step)
                    self._piece(src[r:r + 1, c0:c1], base + r * row_bytes + c0 * dst.itemsize,
                                (c1 - c0) * dst.itemsize)

    def join(self) -> None:
        pending, self.pending = self.pending, [None] * self.nring
        errors = [f.exception() for f in pending if f is not None]
        for e in errors:
            if e is not None:
                raise e


def _host_grid(n: int, m: int, precision: int):
    """(6, n, m) planes + (n, m) int32 codes + (n,) uint8 code-row flags in
    one pinned host block."""
    try:
        return _hostmem.empty([((6, n, m), _device.np_dtype(precision)), ((n, m), np.int32),
                               ((n,), np.uint8)])
    except MemoryError:
        itemsize = 4 if precision == 32 else 8
        raise GridAllocationError(n, m, 6 * n * m * itemsize + 4 * n * m) from None


def partition_work(n: int, m: int, workers: int) -> list[tuple[int, int]]:
    """Balanced disjoint covering ranges over the flat N*M index space
    (batch.py:125-141); also the rule used to shard satellites over GPUs."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    total = n * m
    k = min(workers, total)
    if k <= 0:
        return []
    base, extra = divmod(total, k)
    bounds = np.concatenate([[0], np.cumsum([base + (i < extra) for i in range(k)])])
    return [(int(a), int(b)) for a, b in zip(bounds[:-1], bounds[1:])]


def _tile_grid(n: int, m: int, tile_rows: int, tile_cols: int):
    """Row-major (row-slice, col-slice) tiles covering N x M."""
    return list(_iter_tiles(n, m, tile_rows, tile_cols))


def _iter_tiles(n: int, m: int, tile_rows: int, tile_cols: int):
    for r in range(0, n, tile_rows):
        for c in range(0, m, tile_cols):
            yield slice(r, min(r + tile_rows, n)), slice(c, min(c + tile_cols, m))


@dataclass(frozen=True)
class StreamSummary:
    cells_emitted: int
    nonzero_error_count: int


def propagate_batch_streamed(sats: SatBatch, times, tile_rows: int, tile_cols: int,
                             sink: Callable[[slice, slice, np.ndarray, np.ndarray], Any]
                             ) -> StreamSummary:
    """Tile-by-tile propagation without a full host grid (batch.py:214-241).

    Tiles are delivered in row-major order.  The GPU computes and copies
    tile k+1 into pinned memory while the sink consumes tile k; peak host
    memory is two tiles.  A sink exception aborts with the count delivered.
    """
    if tile_rows < 1 or tile_cols < 1:
        raise ValueError("tile dimensions must be >= 1")
    # host allocations stay O(1) in N and M (the reference's memory contract,
    # test_batch.py:147-173, counts traced Python memory): times are used in
    # place when they already have the batch dtype, tiles are generated lazily
    t = np.asarray(times, dtype=sats.dtype)
    if t.ndim != 1:
        raise ValueError("times must be a 1-D array")
    dev = sats.device_satrec
    n, m = sats.n, t.size
    if n == 0 or m == 0:
        return StreamSummary(0, 0)
    cells = errors = completed = 0
    with torch.cuda.device(dev.device):
        stream = torch.cuda.current_stream(dev.device)
        t_c = np.ascontiguousarray(t)
        t_d = torch.from_numpy(t_c if t_c.flags.writeable else t_c.copy()).to(dev.device)
        t_abs = _device.times_absmax(t)

        def launch(tile):
            rows, cols = tile
            tr, tc = rows.stop - rows.start, cols.stop - cols.start
            planes_d, err_d = _alloc_grid(tr, tc, dev.precision, dev.device)
            _device.propagate_grid(dev, t_d[cols].clone(), planes_d, err_d,
                                   rows=(rows.start, rows.stop), t_absmax=t_abs)
            planes_h, err_h, _ = _host_grid(tr, tc, dev.precision)
            torch.from_numpy(planes_h).copy_(planes_d, non_blocking=True)
            torch.from_numpy(err_h).copy_(err_d, non_blocking=True)
            done = torch.cuda.Event()
            done.record(stream)
            return tile, planes_h, err_h, done, (planes_d, err_d)

        tiles = _iter_tiles(n, m, tile_rows, tile_cols)
        pending = launch(next(tiles))
        while pending is not None:
            (rows, cols), planes_np, err_np, done, keep = pending
            nxt = next(tiles, None)
            pending = launch(nxt) if nxt is not None else None
            done.synchronize()
            try:
                sink(rows, cols, planes_np, err_np)
            except Exception as exc:
                if pending is not None:
                    pending[3].synchronize()
                raise StreamAborted(completed, exc) from exc
            completed += 1
            cells += err_np.size
            errors += int(np.count_nonzero(err_np))
            del planes_np, err_np, keep
    return StreamSummary(cells_emitted=cells, nonzero_error_count=errors)


_SGB1_CHUNK = 16 << 20          # bytes per pinned staging buffer (two of them)


def write_grid_binary(result: BatchResult, stream) -> None:
    """SGB1: 32-byte little-endian header, planes rx..vz, then int32 codes
    (batch.py:244-251; reader frontend/src/sgb1.ts:89-142).

    Host results are written straight from their arrays (a C-contiguous
    (6, n, m) grid is one write, no ``tobytes`` copy).  Device results never
    form a host grid: row blocks of each plane are DMA'd into two pinned
    16 MiB staging buffers in turn, and block k is written to ``stream``
    while block k+1 crosses PCIe.
    """
    planes, error = result.planes, result.error
    if isinstance(planes, torch.Tensor) and planes.is_cuda:
        itemsize = planes.element_size()
    else:
        itemsize = np.dtype(np.asarray(planes).dtype).itemsize
    if itemsize not in (4, 8):
        raise ValueError(f"planes must be float32 or float64, got {itemsize}-byte items")
    stream.write(_HEADER.pack(MAGIC, result.n, result.m, itemsize * 8, PLANE_ORDER_TAG))
    if isinstance(planes, torch.Tensor) and planes.is_cuda:
        _write_device_grid(planes, error, stream)
        return
    planes = planes.cpu().numpy() if isinstance(planes, torch.Tensor) else planes
    error = error.cpu().numpy() if isinstance(error, torch.Tensor) else error
    le = np.dtype(f"<f{itemsize}")
    planes = np.asarray(planes)
    if planes.dtype == le and planes.flags.c_contiguous:
        stream.write(memoryview(planes.reshape(-1)).cast("B"))
    else:
        for plane in planes:
            stream.write(memoryview(np.ascontiguousarray(plane, dtype=le).reshape(-1)).cast("B"))
    codes = np.ascontiguousarray(error, dtype="<i4")
    stream.write(memoryview(codes.reshape(-1)).cast("B"))


def _write_device_grid(planes: torch.Tensor, error: torch.Tensor, stream) -> None:
    """Row blocks of the six planes and the code plane, device -> two pinned
    staging buffers (alternating) -> ``stream``."""
    n, m = int(error.shape[0]), int(error.shape[1])
    if n == 0 or m == 0:
        return
    if sys.byteorder != "little":
        raise RuntimeError("SGB1 device emission assumes a little-endian host")
    row_bytes = m * max(planes.element_size(), 4)
    rows = max(1, _SGB1_CHUNK // row_bytes)
    bufs = [np.asarray(_hostmem.alloc(rows * row_bytes)) for _ in range(2)]
    jobs = [(seg, r0, min(r0 + rows, n))
            for seg in (*planes.unbind(0), error) for r0 in range(0, n, rows)]
    with torch.cuda.device(planes.device):
        cs = torch.cuda.current_stream(planes.device)
        pending: list = [None, None]

        def issue(k: int) -> None:
            seg, r0, r1 = jobs[k]
            nb = (r1 - r0) * m * seg.element_size()
            host = torch.from_numpy(bufs[k % 2][:nb]).view(seg.dtype).view(r1 - r0, m)
            host.copy_(seg[r0:r1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(cs)
            pending[k % 2] = (ev, nb)

        issue(0)
        for k in range(len(jobs)):
            if k + 1 < len(jobs):
                issue(k + 1)            # its buffer was written out in iteration k-1
            ev, nb = pending[k % 2]
            ev.synchronize()
            stream.write(memoryview(bufs[k % 2])[:nb])


def read_grid_binary(stream) -> BatchResult:
    """Inverse of :func:`write_grid_binary`."""
    magic, n, m, bits, tag = _HEADER.unpack(stream.read(_HEADER.size))
    if magic != MAGIC:
        raise ValueError(f"bad magic: {magic!r}")
    if tag != PLANE_ORDER_TAG:
        raise ValueError(f"unknown plane order tag: {tag!r}")
    if bits not in (32, 64):
        raise ValueError(f"precision must be 32 or 64, got {bits}")
    itemsize = bits // 8
    planes = np.frombuffer(stream.read(6 * n * m * itemsize), dtype=f"<f{itemsize}")
    planes = planes.reshape(6, n, m).astype(np.float32 if bits == 32 else np.float64)
    error = np.frombuffer(stream.read(4 * n * m), dtype="<i4").reshape(n, m)
    return BatchResult(planes=planes, error=error.astype(np.int32), n=n, m=m)
