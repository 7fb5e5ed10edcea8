"""TLE catalogue ingest on the GPU (the data format on the
input side of the path).

``read_catalog_columns(path)`` returns the (7, n) fp64 element columns of
every record ``read_tle_file`` would find (a line starting ``"1 "`` followed
by a line starting ``"2 "``; name and blank lines skipped), decoded exactly
as :func:`~paper_2603_27830_b200.tle.parse_catalog_columns` decodes them
(reference: per-record ``parse_tle`` + ``_canonical_elements``,
tle.py:185-276), but on the device: the file's bytes cross PCIe once, line
starts come from one device-side newline scan, and ``sgp4b_tle_columns``
decodes one record per thread.  The columns stay in HBM, ready for
``init_batch``.

Bit-exactness: a decimal field's value m / 10^k is one correctly rounded
division on the device, which is what NumPy's correctly rounded text ->
float64 cast returns; B* and the canonical conversion repeat the host's
operation order.  Records whose fields fall outside the plain decimal syntax
(flagged by the kernel), and files whose layout the fast scan does not
cover (a blank line between line 1 and line 2, bare-CR line ends), are
decoded by the host path instead, so the result always equals the host's
(or raises the host's error).  Checksums are not verified, as in
``parse_catalog_columns``; use ``read_tle_file`` for diagnostics.
"""

from __future__ import annotations

import io
import os

import numpy as np
import torch

from . import _device, _native
from .tle import TleError, parse_catalog_columns

# 10.0**k for k = 0..22 (exact), then the host's 10.0**e for e = -9..9 (the
# B* exponent multiplier of tle._implied_exponent_columns)
_POW10 = np.array([10.0 ** k for k in range(23)] + [10.0 ** e for e in range(-9, 10)],
                  dtype=np.float64)
_pow10_dev: dict = {}


def _pow10(device) -> torch.Tensor:
    key = str(device)
    t = _pow10_dev.get(key)
    if t is None:
        t = torch.from_numpy(_POW10.copy()).to(device)
        _pow10_dev[key] = t
    return t


def _host_lines(data: np.ndarray) -> tuple[list[str], list[str]]:
    """The record lines ``read_tle_file`` pairs (universal newlines, blank
    lines dropped), for the host path."""
    text = data.tobytes().decode("utf-8", errors="surrogateescape")
    # as `for ln in open(path)` reads it: universal newlines only
    rows = [ln.rstrip("\n") for ln in io.StringIO(text, newline=None) if ln.strip()]
    l1, l2 = [], []
    i = 0
    while i < len(rows):
        if not rows[i].startswith("1 "):
            i += 1
            continue
        if i + 1 >= len(rows) or not rows[i + 1].startswith("2 "):
            raise TleError(f"record {len(l1)} at line {i + 1}: line 2 missing")
        l1.append(rows[i])
        l2.append(rows[i + 1])
        i += 2
    return l1, l2


def _as_bytes(source) -> np.ndarray:
    if isinstance(source, np.ndarray):
        arr = np.ascontiguousarray(source.reshape(-1).view(np.uint8))
        return arr if arr.flags.writeable else arr.copy()
    if isinstance(source, (bytes, bytearray, memoryview)):
        return np.frombuffer(bytearray(source), dtype=np.uint8)    # writable copy
    if isinstance(source, (str, os.PathLike)):
        return np.fromfile(source, dtype=np.uint8)
    raise TypeError("source must be a path, bytes or a uint8 array")


def read_catalog_columns(source, device=None) -> torch.Tensor:
    """(7, n) fp64 element columns (ELEMENT_COLUMNS order) of a TLE
    catalogue file, bytes or uint8 array, decoded on ``device``."""
    device = _device.require_cuda(device)
    data = _as_bytes(source)
    size = int(data.size)
    if size == 0:
        return torch.empty((7, 0), dtype=torch.float64, device=device)
    with torch.cuda.device(device):
        buf = torch.from_numpy(data).to(device)
        nl = torch.nonzero(buf == 10).squeeze(1)
        starts = torch.cat([torch.zeros(1, dtype=torch.int64, device=device), nl + 1])
        starts = starts[starts < size]
        nxt = torch.clamp(starts + 1, max=size - 1)
        first, second = buf[starts], buf[nxt]
        second = torch.where(starts + 1 < size, second, torch.zeros_like(second))
        is1 = (first == ord("1")) & (second == ord(" "))
        is2 = (first == ord("2")) & (second == ord(" "))
        follows = torch.zeros_like(is1)
        follows[:-1] = is2[1:]
        # the fast scan covers files where every line 1 is directly followed
        # by its line 2 and lines end in LF or CRLF
        bare_cr = bool(((buf[:-1] == 13) & (buf[1:] != 10)).any())
        if bare_cr or bool((is1 & ~follows).any()):
            l1, l2 = _host_lines(data)
            if not l1:
                return torch.empty((7, 0), dtype=torch.float64, device=device)
            return torch.from_numpy(parse_catalog_columns(l1, l2)).to(device)
        rec = torch.nonzero(is1).squeeze(1)
        n = int(rec.numel())
        if n == 0:
            return torch.empty((7, 0), dtype=torch.float64, device=device)
        line1 = starts[rec].contiguous()
        line2 = starts[rec + 1].contiguous()
        cols = torch.empty((7, n), dtype=torch.float64, device=device)
        status = torch.empty((n,), dtype=torch.int32, device=device)
        _native.check(_native.load().sgp4b_tle_columns(
            buf.data_ptr(), size, line1.data_ptr(), line2.data_ptr(), n,
            _pow10(device).data_ptr(), cols.data_ptr(), status.data_ptr(),
            torch.cuda.current_stream(device).cuda_stream))
        bad = torch.nonzero(status).squeeze(1)
        if bad.numel():
            idx = bad.cpu().numpy()
            o1, o2 = line1[bad].cpu().numpy(), line2[bad].cpu().numpy()

            def line_at(off):
                window = data[off:off + 128]
                nl_at = np.flatnonzero(window == 10)
                raw = window[:nl_at[0]] if nl_at.size else window
                return raw.tobytes().decode("utf-8", errors="surrogateescape")
            host = parse_catalog_columns([line_at(o) for o in o1], [line_at(o) for o in o2])
            cols[:, torch.from_numpy(idx).to(device)] = torch.from_numpy(host).to(device)
        return cols
