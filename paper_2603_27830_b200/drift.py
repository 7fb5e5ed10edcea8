"""fp32-vs-fp64 drift study on the GPU (mirror of sgp4kit.drift,
drift.py:46-112).

Both precisions are propagated on the device over the same minutes-since-
epoch grid; the per-cell deviation norms come from the ``sgp4b_drift_norms``
kernel, and the per-time nearest-rank percentiles are taken on the device
(excluded cells sort last as +inf).  Only the (6, M) percentile table
crosses to the host, so catalogue-scale reports stay cheap.

The fp32 path here is this repo's kernel (fp64 init, double-float Kepler
argument), so its drift is smaller than the reference's own fp32 path; the
64-bit truth is the reference-faithful fp64 kernel.
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


def _nearest_rank_columns(sorted_vals: torch.Tensor, counts: torch.Tensor, pct: float) -> torch.Tensor:
    """Nearest-rank percentile per column of a column-sorted (n, m) tensor
    whose first counts[j] entries of column j are valid (drift.py:46-49)."""
    rank = torch.clamp(torch.ceil(counts.double() * (pct / 100.0)).long(), min=1)
    idx = (rank - 1).clamp(max=sorted_vals.shape[0] - 1)
    vals = sorted_vals.gather(0, idx.unsqueeze(0)).squeeze(0)
    return torch.where(counts > 0, vals, torch.full_like(vals, float("nan")))


def drift_report(tles, horizon_days: float, step_minutes: float,
                 grav: GravityModel = WGS72) -> PrecisionReport:
    """Propagate the corpus at 32 and 64 bit and report drift percentiles."""
    if len(tles) == 0:
        raise ValueError("empty corpus")
    if horizon_days <= 0 or step_minutes <= 0:
        raise ValueError("horizon and step must be positive")
    elements = [tle_to_elements(t) if isinstance(t, TwoLineElement) else t for t in tles]
    cols = elements_to_columns(elements)
    times = np.arange(0.0, horizon_days * 1440.0 + 0.5 * step_minutes, step_minutes)

    lo = propagate_batch_device(init_batch(cols, grav, precision=32), times)
    hi = propagate_batch_device(init_batch(cols, grav, precision=64), times)
    n, m = lo.n, lo.m
    dev = lo.planes.device
    with torch.cuda.device(dev):
        p32, p64 = lo.planes.contiguous(), hi.planes.contiguous()
        c32, c64 = lo.error.contiguous(), hi.error.contiguous()
        dr = torch.empty((n, m), dtype=torch.float64, device=dev)
        dv = torch.empty((n, m), dtype=torch.float64, device=dev)
        _native.check(_native.load().sgp4b_drift_norms(
            p32.data_ptr(), p64.data_ptr(), c32.data_ptr(), c64.data_ptr(), n, m,
            dr.data_ptr(), dv.data_ptr(),
            torch.cuda.current_stream(dev).cuda_stream))
        counts = torch.isfinite(dr).sum(dim=0)
        included = int(counts.sum())
        if included == 0:
            raise EmptyReportError("all corpus cells carry nonzero error codes")
        dr_s = torch.sort(dr, dim=0).values
        dv_s = torch.sort(dv, dim=0).values
        table = torch.stack([_nearest_rank_columns(x, counts, p)
                             for x in (dr_s, dv_s) for p in (5, 50, 95)]).cpu().numpy()
    days = times / 1440.0
    return PrecisionReport(
        days=days, p5_km=table[0], p50_km=table[1], p95_km=table[2],
        p5_kms=table[3], p50_kms=table[4], p95_kms=table[5],
        heuristic_km=HEURISTIC_KM_PER_DAY * days, corpus_size=len(elements),
        excluded_cells=n * m - included, included_cells=included)


def emit_report_csv(report: PrecisionReport) -> str:
    """Deterministic CSV at 9 significant digits, one row per grid time."""
    out = io.StringIO()
    out.write(",".join(CSV_COLUMNS) + "\n")
    cols = (report.days, report.p5_km, report.p50_km, report.p95_km,
            report.p5_kms, report.p50_kms, report.p95_kms, report.heuristic_km)
    for j in range(report.days.size):
        out.write(",".join(f"{c[j]:.9g}" for c in cols) + "\n")
    return out.getvalue()
