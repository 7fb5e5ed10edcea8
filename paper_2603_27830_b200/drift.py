"""fp32-vs-fp64 drift study on the GPU (mirror of sgp4kit.drift,
drift.py:46-112).

``drift_report`` has the reference's definition: the corpus is propagated
over one minutes-since-epoch grid at 32 and at 64 bit *by this library*,
the 64-bit result is truth, and per-time nearest-rank percentiles of the
|dr| / |dv| norms are reported.  What it measures therefore follows the
library: the reference reports the drift of its NumPy fp32 path (fp32 init,
fp32 secular angles), this drop-in reports the drift of its B200 fp32
kernel (fp64 init, double-float secular angle), which is 3-100x smaller on
the same corpus.  ``PrecisionReport.fp32_arithmetic`` names which ("b200").

The machinery is pinned separately: ``drift_from_grids`` takes ANY pair of
fp32/fp64 grids (e.g. the reference's own, via the oracle in the tests) and
reproduces the reference's ``drift_report`` table bit for bit
(tests/golden/ref_drift.npz).  Norms come from the ``sgp4b_drift_norms``
kernel (NumPy's rounding order), the percentiles from a per-column radix
select on the device (``sgp4b_drift_percentiles``, excluded cells are +inf);
only the (6, M) table crosses to the host.
"""

from __future__ import annotations

import io
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .batch import init_batch, propagate_batch_device
from .gravity import WGS72, GravityModel
from .tle import TwoLineElement, elements_to_columns, tle_to_elements

HEURISTIC_KM_PER_DAY = 1.0

CSV_COLUMNS = ("day", "p5_km", "p50_km", "p95_km",
               "p5_kms", "p50_kms", "p95_kms", "heuristic_km")


class EmptyReportError(ValueError):
    """Every cell of the corpus was excluded by error codes."""


@dataclass(frozen=True)
class PrecisionReport:
    days: np.ndarray
    p5_km: np.ndarray
    p50_km: np.ndarray
    p95_km: np.ndarray
    p5_kms: np.ndarray
    p50_kms: np.ndarray
    p95_kms: np.ndarray
    heuristic_km: np.ndarray
    corpus_size: int
    excluded_cells: int
    included_cells: int
    fp32_arithmetic: str = "b200"     # whose fp32 path the drift belongs to


def _nearest_rank(sorted_values: np.ndarray, pct: float) -> float:
    """Nearest-rank percentile of a sorted 1-D array (drift.py:46-49)."""
    n = sorted_values.size
    rank = max(1, int(np.ceil(pct / 100.0 * n)))
    return float(sorted_values[rank - 1])


def drift_report(tles, horizon_days: float, step_minutes: float,
                 grav: GravityModel = WGS72) -> PrecisionReport:
    """Propagate the corpus at 32 and 64 bit and report drift percentiles
    (drift.py:52-100)."""
    if len(tles) == 0:
        raise ValueError("empty corpus")
    if horizon_days <= 0 or step_minutes <= 0:
        raise ValueError("horizon and step must be positive")
    elements = [tle_to_elements(t) if isinstance(t, TwoLineElement) else t for t in tles]
    cols = elements_to_columns(elements)
    times = np.arange(0.0, horizon_days * 1440.0 + 0.5 * step_minutes, step_minutes)
    lo = propagate_batch_device(init_batch(cols, grav, precision=32), times)
    hi = propagate_batch_device(init_batch(cols, grav, precision=64), times)
    return drift_from_grids(lo, hi, times, corpus_size=len(elements))


def _on_device(x, dtype: torch.dtype, device) -> torch.Tensor:
    if not isinstance(x, torch.Tensor):
        x = torch.from_numpy(np.ascontiguousarray(x))
    return x.to(device=device, dtype=dtype).contiguous()


def drift_from_grids(lo, hi, times, corpus_size: int | None = None,
                     fp32_arithmetic: str = "b200", device=None) -> PrecisionReport:
    """The report of an fp32 grid ``lo`` against an fp64 grid ``hi`` (both
    BatchResult-like: planes (6, n, m), error (n, m); host arrays or device
    tensors) over ``times`` (drift.py:67-100)."""
    n, m = int(hi.n), int(hi.m)
    if (int(lo.n), int(lo.m)) != (n, m) or len(times) != m:
        raise ValueError("lo, hi and times must describe the same n x m grid")
    if device is None:
        device = hi.planes.device if isinstance(hi.planes, torch.Tensor) else torch.device("cuda", 0)
    with torch.cuda.device(device):
        p32 = _on_device(lo.planes, torch.float32, device)
        p64 = _on_device(hi.planes, torch.float64, device)
        c32 = _on_device(lo.error, torch.int32, device)
        c64 = _on_device(hi.error, torch.int32, device)
        dr = torch.empty((n, m), dtype=torch.float64, device=device)
        dv = torch.empty((n, m), dtype=torch.float64, device=device)
        _native.check(_native.load().sgp4b_drift_norms(
            p32.data_ptr(), p64.data_ptr(), c32.data_ptr(), c64.data_ptr(), n, m,
            dr.data_ptr(), dv.data_ptr(),
            torch.cuda.current_stream(device).cuda_stream))
        # per-column nearest-rank selection on the device (radix select,
        # exact: the element a full column sort would put at the rank)
        table_d = torch.empty((6, m), dtype=torch.float64, device=device)
        counts = torch.empty((m,), dtype=torch.int64, device=device)
        frac = np.array([p / 100.0 for p in (5, 50, 95)], dtype=np.float64)
        _native.check(_native.load().sgp4b_drift_percentiles(
            dr.data_ptr(), dv.data_ptr(), n, m, frac.ctypes.data, table_d.data_ptr(),
            counts.data_ptr(), torch.cuda.current_stream(device).cuda_stream))
        included = int(counts.sum())
        if included == 0:
            raise EmptyReportError("all corpus cells carry nonzero error codes")
        table = table_d.cpu().numpy()
    days = np.asarray(times, dtype=np.float64) / 1440.0
    return PrecisionReport(
        days=days, p5_km=table[0], p50_km=table[1], p95_km=table[2],
        p5_kms=table[3], p50_kms=table[4], p95_kms=table[5],
        heuristic_km=HEURISTIC_KM_PER_DAY * days,
        corpus_size=n if corpus_size is None else corpus_size,
        excluded_cells=n * m - included, included_cells=included,
        fp32_arithmetic=fp32_arithmetic)


def emit_report_csv(report: PrecisionReport) -> str:
    """Deterministic CSV at 9 significant digits, one row per grid time."""
    out = io.StringIO()
    out.write(",".join(CSV_COLUMNS) + "\n")
    cols = (report.days, report.p5_km, report.p50_km, report.p95_km,
            report.p5_kms, report.p50_kms, report.p95_kms, report.heuristic_km)
    for j in range(report.days.size):
        out.write(",".join(f"{c[j]:.9g}" for c in cols) + "\n")
    return out.getvalue()
