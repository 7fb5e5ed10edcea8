"""Scalar / broadcasting SGP4 API (mirror of sgp4kit.kernel, kernel.py:45-558).

``sgp4_init`` and ``sgp4_propagate`` keep the reference's signatures,
dataclasses and broadcasting rules, but both run on the GPU through
libsgp4b.so: init is the fp64 init kernel; propagate runs the same grid-
kernel instance as ``propagate_batch`` — as one dense grid when the
broadcast is a Cartesian product (satellite axes x time axes, e.g. init
(n, 1) against times (m,)), otherwise as one-step rows of (satellite, time)
pairs — so a batch cell equals the scalar call at the same precision bit for
bit (the reference's batch≡scalar contract, tests/test_batch.py:39-64).
"""

from __future__ import annotations

import enum
import dataclasses
from dataclasses import dataclass, fields as dataclass_fields
from typing import Any

import numpy as np
import torch

from . import _device, _hostmem
from .gravity import WGS72, GravityModel
from .tle import ELEMENT_COLUMNS, MeanElements

TWOPI = 2.0 * np.pi
KEPLER_MAX_ITER = 10
KEPLER_TOL = 1.0e-12
KEPLER_CLAMP = 0.95
DEEP_SPACE_PERIOD_MIN = 225.0


class ErrorCode(enum.IntEnum):
    """Per-cell status codes (kernel.py:45-52); 3 is declared, never produced."""

    OK = 0
    ECC_OUT_OF_RANGE = 1
    MEAN_MOTION_NONPOSITIVE = 2
    PERT_ECC_OUT_OF_RANGE = 3
    SEMILATUS_NEGATIVE = 4
    SUBORBITAL = 6
    DEEP_SPACE_UNSUPPORTED = 7


#: SatInit float fields in the order of the device SoA satrec (33 columns)
SATREC_FIELD_NAMES = (
    "no_kozai", "ecco", "inclo", "nodeo", "argpo", "mo", "bstar",
    "no_unkozai", "ao", "con41", "x1mth2", "x7thm1",
    "mdot", "argpdot", "nodedot", "nodecf",
    "cc1", "cc4", "cc5", "d2", "d3", "d4", "t2cof", "t3cof", "t4cof", "t5cof",
    "eta", "omgcof", "xmcof", "delmo", "sinmao", "aycof", "xlcof",
)
assert len(SATREC_FIELD_NAMES) == _device.SATREC_FIELDS


@dataclass(frozen=True)
class SatInit:
    """Initialisation constants (kernel.py:55-109), scalars or parallel arrays.

    An instance produced by :func:`sgp4_init` / ``init_batch`` also carries
    (as a non-field attribute) the GPU-resident packed records it was built
    from; an instance built or edited by hand is re-packed on the GPU on
    first use.
    """

    grav: GravityModel
    dtype: Any
    no_kozai: Any
    ecco: Any
    inclo: Any
    nodeo: Any
    argpo: Any
    mo: Any
    bstar: Any
    no_unkozai: Any
    ao: Any
    con41: Any
    x1mth2: Any
    x7thm1: Any
    mdot: Any
    argpdot: Any
    nodedot: Any
    nodecf: Any
    isimp: Any
    cc1: Any
    cc4: Any
    cc5: Any
    d2: Any
    d3: Any
    d4: Any
    t2cof: Any
    t3cof: Any
    t4cof: Any
    t5cof: Any
    eta: Any
    omgcof: Any
    xmcof: Any
    delmo: Any
    sinmao: Any
    aycof: Any
    xlcof: Any
    error_code_at_init: Any


@dataclass(frozen=True)
class StateVector:
    """TEME position (km) and velocity (km/s) plus the int32 status."""

    r: Any
    v: Any
    error_code: Any


def satinit_from_device(dev: "_device.DeviceSatrec", shape: tuple) -> SatInit:
    """Materialise the public SatInit (host numpy) from a device satrec."""
    dtype = _device.np_dtype(dev.precision)
    sr = dev.satrec.cpu().numpy()
    values = {name: sr[k].astype(dtype).reshape(shape)
              for k, name in enumerate(SATREC_FIELD_NAMES)}
    values["isimp"] = dev.isimp.cpu().numpy().astype(bool).reshape(shape)
    values["error_code_at_init"] = dev.codes.cpu().numpy().astype(np.int32).reshape(shape)
    init = SatInit(grav=dev.grav, dtype=dtype, **values)
    object.__setattr__(init, "_sgp4b_dev", dev)
    object.__setattr__(init, "_sgp4b_shape", tuple(shape))
    return init


def _element_columns(elems: MeanElements) -> tuple[np.ndarray, tuple]:
    arrays = [np.asarray(getattr(elems, name), dtype=np.float64) for name in ELEMENT_COLUMNS]
    shape = np.broadcast_shapes(*(a.shape for a in arrays))
    cols = np.stack([np.broadcast_to(a, shape).ravel() for a in arrays])
    return cols, shape


def sgp4_init(elems: MeanElements, grav: GravityModel = WGS72,
              dtype=np.float64) -> SatInit:
    """All propagation constants from canonical mean elements (kernel.py:139).

    Runs the fp64 init kernel (including the epoch evaluation that flags
    immediate decay) and rounds the constants to ``dtype``.  Never raises on
    anomalous elements: ``error_code_at_init`` is non-zero instead.
    """
    precision = _device.precision_of(dtype)
    cols, shape = _element_columns(elems)
    if cols.shape[1] == 0:
        raise ValueError("empty element arrays")
    dev = _device.init_device(cols, grav, precision)
    return satinit_from_device(dev, shape)


def _device_of(init: SatInit) -> tuple["_device.DeviceSatrec", tuple]:
    """The packed GPU records behind ``init`` (re-packed if hand-built)."""
    dev = getattr(init, "_sgp4b_dev", None)
    if dev is not None:
        return dev, init._sgp4b_shape
    precision = _device.precision_of(init.dtype)
    arrays = [np.asarray(getattr(init, name), dtype=np.float64) for name in SATREC_FIELD_NAMES]
    isimp = np.asarray(init.isimp)
    codes = np.asarray(init.error_code_at_init)
    shape = np.broadcast_shapes(*(a.shape for a in arrays), isimp.shape, codes.shape)
    sr = np.stack([np.broadcast_to(a, shape).ravel() for a in arrays])
    dev = _device.pack_device(sr, np.broadcast_to(codes, shape).ravel(),
                              np.broadcast_to(isimp, shape).ravel(), init.grav, precision)
    object.__setattr__(init, "_sgp4b_dev", dev)
    object.__setattr__(init, "_sgp4b_shape", tuple(shape))
    return dev, tuple(shape)


def sgp4_propagate(init: SatInit, tsince_min) -> StateVector:
    """Propagate to ``tsince_min`` minutes since epoch (kernel.py:513-534).

    Broadcasts the satellite shape of ``init`` against the time shape; scalar
    in, scalar out; r/v have a trailing axis of 3.  Times are cast to the
    init dtype first, as in the reference.
    """
    dtype = np.dtype(init.dtype)
    t = np.asarray(tsince_min, dtype=dtype)
    dev, sat_shape = _device_of(init)
    out_shape = np.broadcast_shapes(sat_shape, t.shape)
    p = int(np.prod(out_shape, dtype=np.int64))
    if p == 0:
        return StateVector(r=np.empty(out_shape + (3,), dtype=dtype),
                           v=np.empty(out_shape + (3,), dtype=dtype),
                           error_code=np.zeros(out_shape, dtype=np.int32))
    device = dev.device
    nd = len(out_shape)
    sat_p = (1,) * (nd - len(sat_shape)) + tuple(sat_shape)
    t_p = (1,) * (nd - t.ndim) + tuple(t.shape)
    sat_axes = [k for k in range(nd) if sat_p[k] > 1]
    t_axes = [k for k in range(nd) if t_p[k] > 1]
    dt = _device.torch_dtype(dev.precision)
    with torch.cuda.device(device):
        if not set(sat_axes) & set(t_axes):
            # Cartesian product (e.g. init (n, 1) x times (m,)): one dense grid
            perm = sat_axes + t_axes + [k for k in range(nd) if k not in sat_axes + t_axes]
            n_sel = int(np.prod([out_shape[k] for k in sat_axes], dtype=np.int64))
            m_sel = int(np.prod([out_shape[k] for k in t_axes], dtype=np.int64))
            sats = np.broadcast_to(np.arange(dev.n, dtype=np.int64).reshape(sat_shape), out_shape)
            rows = np.ascontiguousarray(sats.transpose(perm).reshape(n_sel, m_sel, -1)[:, 0, 0])
            tsel = np.ascontiguousarray(
                np.broadcast_to(t, out_shape).transpose(perm).reshape(n_sel, m_sel, -1)[0, :, 0])
            planes, codes = _grid_of_rows(dev, rows, tsel)
            # (3, n_sel, m_sel) -> out_shape + (3,) on the device, then one D2H each
            shape_p = tuple(out_shape[k] for k in perm)
            inv = [int(a) for a in np.argsort(perm)]
            order = [1 + a for a in inv] + [0]

            def arrange(blk):
                return blk.reshape((3,) + shape_p).permute(order).contiguous()
            r_d = arrange(planes[0:3])
            v_d = arrange(planes[3:6])
            c_d = codes.reshape(shape_p).permute(inv).contiguous()
        else:
            # general broadcast: one (satellite, time) pair per cell
            if tuple(sat_p) == tuple(out_shape):
                # every cell its own satellite, in order: no index array to upload
                idx_d = torch.arange(p, dtype=torch.int64, device=device)
            else:
                idx = np.broadcast_to(np.arange(dev.n, dtype=np.int64).reshape(sat_shape),
                                      out_shape).ravel()
                idx_d = torch.from_numpy(np.ascontiguousarray(idx)).to(device)
            tt = np.array(np.broadcast_to(t, out_shape).ravel())          # writable copy
            t_d = torch.from_numpy(tt).to(device)
            rv = torch.empty((6, p), dtype=dt, device=device)
            c_d = torch.empty((p,), dtype=torch.int32, device=device)
            _device.propagate_pairs(dev, idx_d, t_d, rv, c_d, t_absmax=_device.times_absmax(tt))
            r_d = rv[0:3].t().contiguous()
            v_d = rv[3:6].t().contiguous()
        # one page-locked block for r, v and the codes (pooled, see _hostmem);
        # pageable arrays when the result is larger than the pool keeps
        specs = [(out_shape + (3,), dtype), (out_shape + (3,), dtype), (out_shape, np.int32)]
        nbytes = 2 * r_d.numel() * r_d.element_size() + 4 * p
        if nbytes <= _hostmem.cache_limit():
            r, v, codes_h = _hostmem.empty(specs)
            for dst, src in ((r, r_d), (v, v_d), (codes_h, c_d)):
                torch.from_numpy(dst).view(-1).copy_(src.view(-1), non_blocking=True)
            torch.cuda.current_stream(device).synchronize()
        else:
            r = r_d.cpu().numpy().reshape(out_shape + (3,))
            v = v_d.cpu().numpy().reshape(out_shape + (3,))
            codes_h = c_d.cpu().numpy().reshape(out_shape)
    return StateVector(r=r, v=v, error_code=codes_h)


def _grid_of_rows(dev, rows: np.ndarray, times: np.ndarray):
    """Dense grid for the satellites ``rows`` (indices into ``dev``) at
    ``times``, through the same padded grid-kernel instance as
    ``propagate_batch`` (so results equal the batch bit for bit)."""
    from .batch import _alloc_grid
    device = dev.device
    rows_d = torch.from_numpy(np.array(rows, dtype=np.int64)).to(device)
    sub = dataclasses.replace(dev, record=dev.record.index_select(0, rows_d).contiguous(),
                              codes=dev.codes.index_select(0, rows_d))
    t_d = torch.from_numpy(np.array(times)).to(device)
    planes, codes = _alloc_grid(int(rows.size), int(times.size), dev.precision, device)
    _device.propagate_grid(sub, t_d, planes, codes, t_absmax=_device.times_absmax(times))
    return planes, codes


def solve_kepler(axnl, aynl, u_init):
    """Newton solve of SGP4's Kepler equation (kernel.py:325-349): at most 10
    steps, step clamped to ±0.95, per-element freeze once |step| < 1e-12."""
    a, b, u = np.broadcast_arrays(np.asarray(axnl), np.asarray(aynl), np.asarray(u_init))
    dtype = np.result_type(a, b, u)
    if dtype not in (np.float32, np.float64):
        dtype = np.float64
    precision = _device.precision_of(dtype)
    device = _device.require_cuda()
    tens = [torch.from_numpy(np.array(x, dtype=dtype).ravel()).to(device)
            for x in (a, b, u)]
    if tens[0].numel() == 0:
        return np.empty(a.shape, dtype=dtype)
    out = _device.solve_kepler_device(*tens, precision).cpu().numpy().reshape(a.shape)
    return out if out.ndim else out[()]


_DAYS_BEFORE = (0, 31, 59, 90, 120, 151, 181, 212, 243, 273, 304, 334)


def epoch_to_julian(epoch_year: int, epoch_day_int: int, epoch_day_frac: float) -> float:
    """Julian date of a split TLE epoch, fp64 host arithmetic (kernel.py:544-558)."""
    leap = epoch_year % 4 == 0 and (epoch_year % 100 != 0 or epoch_year % 400 == 0)
    if not 1 <= epoch_day_int <= (366 if leap else 365):
        raise ValueError(f"day {epoch_day_int} out of range for year {epoch_year}")
    y = epoch_year - 1
    jan0 = 1721424.5 + 365 * y + y // 4 - y // 100 + y // 400
    return jan0 + float(epoch_day_int) + float(epoch_day_frac)
