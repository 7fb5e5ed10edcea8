"""CPU ORACLE — test infrastructure only, never shipped, never on the product path.

Full-grid parity of a device grid against the oracle (sgp4_oracle.py, which
is pinned bit-for-bit to the reference).  Used by the ``-m gpu`` parity tests
on every BASELINE.json config that fits one GPU and by ``bench.py``'s
accuracy/cpu-baseline leg (the checker, never the thing measured).

The comparison follows the reference's own equivalence bar
(pkg/tests/test_acceptance.py:42-69: per-cell codes equal, |dr| / |dv| on
cells whose code is 0) and its precision study (pkg/src/sgp4kit/drift.py:
64-72: fp32 measured against the reference's own fp64 path).  Work is done in
row bands so a 144 M-cell grid (C4) never needs a full fp64 host copy.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import sgp4_oracle as oracle


@dataclass
class GridParity:
    """Outcome of one full-grid comparison."""

    n: int
    m: int
    precision: int
    cells: int = 0
    ok_cells: int = 0                       # cells whose oracle fp64 code is 0
    code_mismatch_fp64: int = 0             # cells whose code differs from oracle fp64
    code_mismatch_same: int = 0             # ... from the oracle at the grid's precision
    dr_max: float = 0.0                     # km, vs oracle fp64, ok cells
    dv_max: float = 0.0                     # km/s
    ref32_dr_max: float | None = None       # the reference's own fp32 error (fp32 grids)
    _dr: list = field(default_factory=list, repr=False)
    _dv: list = field(default_factory=list, repr=False)
    _dr32: list = field(default_factory=list, repr=False)

    def percentiles(self) -> dict:
        dr = np.concatenate(self._dr) if self._dr else np.zeros(0)
        dv = np.concatenate(self._dv) if self._dv else np.zeros(0)
        out = {"dr_median_km": _pct(dr, 50), "dr_p99_km": _pct(dr, 99), "dr_max_km": self.dr_max,
               "dv_median_kms": _pct(dv, 50), "dv_p99_kms": _pct(dv, 99), "dv_max_kms": self.dv_max}
        if self._dr32:
            d32 = np.concatenate(self._dr32)
            out.update({"ref_fp32_dr_median_km": _pct(d32, 50), "ref_fp32_dr_p99_km": _pct(d32, 99),
                        "ref_fp32_dr_max_km": self.ref32_dr_max})
        return out

    def summary(self) -> dict:
        d = {"n_sats": self.n, "n_steps": self.m, "precision": self.precision,
             "cells_compared": self.cells, "ok_cells": self.ok_cells,
             "code_mismatch_vs_ref_fp64": self.code_mismatch_fp64,
             "code_mismatch_vs_ref_same_precision": self.code_mismatch_same}
        d.update(self.percentiles())
        return d


def _pct(x: np.ndarray, q: float) -> float | None:
    return float(np.percentile(x, q)) if x.size else None


def _norms(a: np.ndarray, b: np.ndarray, mask: np.ndarray):
    """|a - b| over the 3 components of (3, rows, m) planes at masked cells,
    in fp64 (squares summed left to right, as np.linalg.norm does)."""
    d = a.astype(np.float64) - b
    n = np.sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2])
    return n[mask]


def compare_grid(cols: np.ndarray, times: np.ndarray, get_rows, precision: int,
                 workers: int = 1, band_rows: int | None = None,
                 with_ref32_states: bool = True) -> GridParity:
    """Compare a device grid with the oracle, every cell.

    ``cols``      (7, n) element columns the grid was built from;
    ``get_rows``  callable (lo, hi) -> (planes (6, hi-lo, m), codes (hi-lo, m))
                  as host numpy arrays (the device grid's rows lo..hi);
    ``precision`` of the device grid.  Codes are compared with the oracle at
    fp64 and (for fp32 grids) at fp32; states are compared with the oracle
    fp64 on cells whose fp64 code is 0.  For fp32 grids the reference's own
    fp32 error on the same cells is collected too.
    """
    n, m = cols.shape[1], int(np.asarray(times).size)
    if band_rows is None:
        band_rows = max(1, min(n, (1 << 24) // max(m, 1)))
    res = GridParity(n=n, m=m, precision=precision)
    for lo in range(0, n, band_rows):
        hi = min(n, lo + band_rows)
        planes, codes = get_rows(lo, hi)
        sub = cols[:, lo:hi]
        ref64, c64 = oracle.grid(oracle.init_columns(sub, 64), times, workers=workers)
        res.cells += codes.size
        res.code_mismatch_fp64 += int(np.count_nonzero(codes != c64))
        if precision == 32:
            ref32, c32 = oracle.grid(oracle.init_columns(sub, 32), times, workers=workers)
            res.code_mismatch_same += int(np.count_nonzero(codes != c32))
        else:
            ref32 = None
            res.code_mismatch_same = res.code_mismatch_fp64
        ok = c64 == 0
        res.ok_cells += int(np.count_nonzero(ok))
        dr = _norms(planes[:3], ref64[:3], ok)
        dv = _norms(planes[3:], ref64[3:], ok)
        if dr.size:
            res.dr_max = max(res.dr_max, float(dr.max()))
            res.dv_max = max(res.dv_max, float(dv.max()))
            res._dr.append(dr.astype(np.float32))
            res._dv.append(dv.astype(np.float32))
        if ref32 is not None and with_ref32_states and dr.size:
            d32 = _norms(ref32[:3], ref64[:3], ok & (c32 == 0))
            if d32.size:
                res.ref32_dr_max = max(res.ref32_dr_max or 0.0, float(d32.max()))
                res._dr32.append(d32.astype(np.float32))
    return res
