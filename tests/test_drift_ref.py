"""drift_report pinned to the reference's own output (
reference drift.py:46-112, test_drift.py, test_acceptance.py:107-122).

tests/golden/ref_drift.npz / ref_drift.csv are the reference
``drift_report(first 120 LEO records, 14 d, 90 min)`` and its CSV.  The
oracle reproduces the reference's fp32 and fp64 grids bit for bit
(test_oracle.py), so feeding those grids through this library's device
machinery (``drift_from_grids``) must reproduce the reference table exactly;
``drift_report`` itself reports this library's fp32 path, which the
acceptance bands bound and which must not drift more than the reference."""

from __future__ import annotations

import numpy as np
import pytest

from paper_2603_27830_b200.drift import CSV_COLUMNS, _nearest_rank

from .conftest import GOLDEN

FIELDS = ("p5_km", "p50_km", "p95_km", "p5_kms", "p50_kms", "p95_kms")


@pytest.fixture(scope="module")
def ref_drift():
    return dict(np.load(GOLDEN / "ref_drift.npz"))


@pytest.fixture(scope="module")
def reference_grids(corpus_columns, oracle, ref_drift):
    """The reference's fp32 and fp64 grids for the acceptance corpus."""
    cols = corpus_columns[:, :120]
    times = ref_drift["days"] * 1440.0
    lo = oracle.grid(oracle.init_columns(cols, 32), times)
    hi = oracle.grid(oracle.init_columns(cols, 64), times)
    return cols, times, lo, hi


class _Grid:
    def __init__(self, planes, error):
        self.planes, self.error = planes, error
        self.n, self.m = error.shape


def test_nearest_rank_definition():
    v = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
    assert [_nearest_rank(v, p) for p in (50, 5, 95, 100)] == [3.0, 1.0, 5.0, 5.0]
    assert _nearest_rank(np.array([7.0]), 95) == 7.0


def test_fixture_is_reproduced_by_host_recomputation(reference_grids, ref_drift):
    """The checker side: NumPy nearest-rank over the oracle's grids gives
    the reference fixture exactly (pins oracle + fixture together)."""
    _, times, (p32, c32), (p64, c64) = reference_grids
    inc = (c32 == 0) & (c64 == 0)
    dr = np.linalg.norm(np.moveaxis(p32[:3], 0, -1).astype(np.float64) - np.moveaxis(p64[:3], 0, -1), axis=-1)
    for j in (0, 100, times.size - 1):
        col = np.sort(dr[inc[:, j], j])
        assert _nearest_rank(col, 50) == ref_drift["p50_km"][j]
        assert _nearest_rank(col, 95) == ref_drift["p95_km"][j]
    assert int(inc.sum()) == int(ref_drift["included_cells"])


@pytest.mark.gpu
def test_device_machinery_reproduces_reference_table(reference_grids, ref_drift):
    from paper_2603_27830_b200.drift import drift_from_grids, emit_report_csv

    _, times, (p32, c32), (p64, c64) = reference_grids
    rep = drift_from_grids(_Grid(p32, c32), _Grid(p64, c64), times, corpus_size=120,
                           fp32_arithmetic="reference")
    for f in FIELDS + ("days", "heuristic_km"):
        assert np.array_equal(getattr(rep, f), ref_drift[f], equal_nan=True), f
    assert rep.included_cells == int(ref_drift["included_cells"])
    assert rep.excluded_cells == int(ref_drift["excluded_cells"])
    assert emit_report_csv(rep) == (GOLDEN / "ref_drift.csv").read_text()


@pytest.mark.gpu
def test_drift_report_bands_and_no_worse_than_reference(ref_drift):
    """test_acceptance.py:107-122 bands on this library's fp32 path, and its
    median drift at every grid time at most the reference fp32 path's."""
    from paper_2603_27830_b200 import drift_report, emit_report_csv
    from paper_2603_27830_b200.tle import parse_tle, tle_to_elements

    from .conftest import read_tle_pairs

    pairs = read_tle_pairs(GOLDEN / "leo_corpus.tle")[1][:120]
    rep = drift_report([tle_to_elements(parse_tle(a, b)) for a, b in pairs], 14.0, 90.0)
    assert rep.fp32_arithmetic == "b200"
    assert np.array_equal(rep.days, ref_drift["days"])
    assert rep.included_cells + rep.excluded_cells == 120 * rep.days.size
    assert rep.included_cells == int(ref_drift["included_cells"])
    assert 0.1 <= rep.p50_km[0] * 1000.0 <= 10.0
    assert rep.p50_km[-1] < 1.0 and rep.p50_kms[-1] * 1000.0 < 10.0
    ok = ~np.isnan(ref_drift["p50_km"])
    assert (rep.p50_km[ok] <= ref_drift["p50_km"][ok]).all()
    assert (rep.p95_km[ok] <= ref_drift["p95_km"][ok]).all()
    head = emit_report_csv(rep).splitlines()[0]
    assert head == ",".join(CSV_COLUMNS)
    print(f"\ndrift day-14 median: b200 fp32 {rep.p50_km[-1] * 1e3:.2f} m, "
          f"reference fp32 {ref_drift['p50_km'][-1] * 1e3:.2f} m")
