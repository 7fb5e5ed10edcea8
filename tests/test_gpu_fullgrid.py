"""Full-grid parity on every BASELINE.json config that fits one GPU.

Every cell of the device grid is compared with the CPU oracle (bit-exact
with the reference, tests/test_oracle.py) — no sampling:

  C1  ISS x linspace(0, 1440, 1000), fp64           (BASELINE configs[0])
  C2  Starlink-like 9,341 x linspace(0, 1440, 1000), fp32   (the headline)
  C3  the same catalogue and grid, fp64
  C4  100,000 x arange(1440), fp32

Bars (BASELINE.json north_star; reference acceptance test_acceptance.py:42-69):
  * error codes bit-exact per cell vs the reference at the grid's precision
    AND vs the reference fp64 path;
  * fp64: |dr| <= 1 mm (1e-6 km) and |dv| <= 1e-6 km/s on every code-0 cell;
  * fp32: |dr| / |dv| against the reference's fp64 path are reported (median,
    p99, max) and must sit at or below the reference's OWN fp32 error on the
    same cells (drift.py:64-72 measures that error), with max |dr| < 100 m.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL64_R = 1.0e-6     # km
TOL64_V = 1.0e-6     # km/s


def _run(cols, times, precision):
    import paper_2603_27830_b200 as pkg
    return pkg.propagate_batch_device(pkg.init_batch(cols, precision=precision), times)


def _rows_of(res):
    def get(lo, hi):
        return res.planes[:, lo:hi].cpu().numpy(), res.error[lo:hi].cpu().numpy()
    return get


def _check(cols, times, precision, label, band_rows=None):
    from oracle import sgp4_oracle as oracle
    from oracle.parity import compare_grid
    res = _run(cols, times, precision)
    par = compare_grid(cols, times, _rows_of(res), precision,
                       workers=oracle.default_workers(), band_rows=band_rows)
    s = par.summary()
    print(f"\n{label}: {s}")
    assert par.cells == cols.shape[1] * times.size
    assert par.code_mismatch_fp64 == 0, s
    assert par.code_mismatch_same == 0, s
    return par, s


def test_c1_iss_fp64_all_cells():
    from paper_2603_27830_b200.catalog import iss_columns
    times = np.linspace(0.0, 1440.0, 1000)
    par, s = _check(iss_columns(), times, 64, "C1 ISS fp64")
    assert par.ok_cells == 1000
    assert par.dr_max <= TOL64_R and par.dv_max <= TOL64_V, s


def test_c2_starlink_fp32_all_cells():
    from paper_2603_27830_b200.catalog import starlink_like
    times = np.linspace(0.0, 1440.0, 1000)
    par, s = _check(starlink_like(9341), times, 32, "C2 Starlink fp32")
    assert par.ok_cells == 9341 * 1000
    # fp32 error vs the reference fp64 path, at or below the reference's own
    # fp32 error on the same cells
    assert s["dr_max_km"] < 0.1, s
    assert s["dr_median_km"] <= s["ref_fp32_dr_median_km"], s
    assert s["dr_p99_km"] <= s["ref_fp32_dr_p99_km"], s
    assert s["dr_max_km"] <= s["ref_fp32_dr_max_km"], s
    assert s["dv_max_kms"] < 1e-4, s


def test_c3_starlink_fp64_all_cells():
    from paper_2603_27830_b200.catalog import starlink_like
    times = np.linspace(0.0, 1440.0, 1000)
    par, s = _check(starlink_like(9341), times, 64, "C3 Starlink fp64")
    assert par.ok_cells == 9341 * 1000
    assert par.dr_max <= TOL64_R and par.dv_max <= TOL64_V, s


def test_c4_megaconstellation_fp32_all_cells():
    from paper_2603_27830_b200.catalog import starlink_like
    times = np.arange(1440.0)
    par, s = _check(starlink_like(100_000), times, 32, "C4 100k x 1440 fp32",
                    band_rows=10_000)
    assert par.ok_cells == 100_000 * 1440
    assert s["dr_max_km"] < 0.1, s
    assert s["dr_median_km"] <= s["ref_fp32_dr_median_km"], s
    assert s["dr_max_km"] <= s["ref_fp32_dr_max_km"], s
