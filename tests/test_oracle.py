"""Pin the CPU oracle to the real reference: bit-for-bit equality with the
golden vectors sgp4kit itself produced (tests/golden/make_golden.py)."""

import math

import numpy as np
import pytest

FIELDS_CHECKED = 33


@pytest.mark.parametrize("precision", [64, 32])
def test_init_bitwise_vs_reference(oracle, golden_columns, golden_states, precision):
    g = golden_states[precision]
    sat = oracle.init_columns(golden_columns, precision)
    for name in oracle.SATREC_FIELDS:
        assert np.array_equal(np.asarray(sat[name]), g["init_" + name]), name
    assert np.array_equal(sat["isimp"], g["init_isimp"])
    assert np.array_equal(sat["error_code_at_init"], g["init_error_code_at_init"])
    assert len(oracle.SATREC_FIELDS) == FIELDS_CHECKED


@pytest.mark.parametrize("precision", [64, 32])
@pytest.mark.parametrize("workers", [1, 3])
def test_grid_bitwise_vs_reference(oracle, golden_columns, golden_states, precision, workers):
    g = golden_states[precision]
    sat = oracle.init_columns(golden_columns, precision)
    planes, codes = oracle.grid(sat, g["times"], workers=workers, tile_cells=1000)
    assert planes.dtype == (np.float32 if precision == 32 else np.float64)
    assert np.array_equal(planes, g["planes"])
    assert np.array_equal(codes, g["error"])


def test_known_answer_states(oracle, golden_columns):
    """SURVEY.md §8(c) anchors (reference fp64, t = 720 min)."""
    sat = oracle.init_columns(golden_columns[:, :4], 64)
    r, v, code = oracle.propagate_merged(oracle._rows(sat, 0, 4), np.array([720.0]))
    want_r = np.array([[1406.824966466, -3981.383365658, -5331.554241199],
                       [3210.481648468, 6006.615087005, -1267.317604605],
                       [3434.731618601, -4940.31924392, 3958.515935818],
                       [-489.92471512, 5170.826556783, 4040.840299224]])
    want_v = np.array([[7.237716791215, 2.476868653163, 0.061990211066],
                       [-4.604275511693, 1.222321635828, -5.905282841396],
                       [-3.409214852293, 2.538309873412, 6.107546283396],
                       [1.559087790238, -4.620267045956, 6.068207469481]])
    assert np.abs(r[:, 0] - want_r).max() < 1e-8
    assert np.abs(v[:, 0] - want_v).max() < 1e-11
    assert (code == 0).all()
    assert float(sat["no_unkozai"][0]) == pytest.approx(6.759386610326881e-02, rel=1e-15)
    assert float(sat["cc1"][0]) == pytest.approx(1.712672703602596e-09, rel=1e-14)


def test_failure_codes_vs_reference(oracle, failure_table):
    times = np.array(failure_table["times"])
    for key, row in failure_table["cases"].items():
        cols = np.array(row["elements"], dtype=np.float64)[:, None]
        for precision in (64, 32):
            sat = oracle.init_columns(cols, precision)
            assert int(sat["error_code_at_init"][0]) == row[f"init_code_{precision}"], key
            _, codes = oracle.grid(sat, times)
            assert codes[0].tolist() == row[f"codes_{precision}"], (key, precision)


def test_kepler_against_bisection(oracle):
    """kernel tests :182-229: Newton agrees with bisection; e=0 gives E=u."""
    def bisect(ax, ay, u):
        f = lambda e: u - (e - ax * math.sin(e) + ay * math.cos(e))  # noqa: E731
        lo, hi = u - 1.0, u + 1.0
        while f(lo) * f(hi) > 0:
            lo, hi = lo - 1.0, hi + 1.0
        for _ in range(200):
            mid = 0.5 * (lo + hi)
            lo, hi = (lo, mid) if f(lo) * f(mid) <= 0 else (mid, hi)
        return 0.5 * (lo + hi)

    for ax, ay, u in [(0.1, 0.0, 1.0), (0.0, 0.05, 2.5), (0.02, 0.03, 5.9), (0.3, -0.2, 0.4)]:
        e = float(oracle.kepler(np.float64(ax), np.float64(ay), np.float64(u)))
        assert e == pytest.approx(bisect(ax, ay, u), abs=1e-10)
    assert float(oracle.kepler(np.float64(0), np.float64(0), np.float64(1.2345))) == 1.2345


def test_parity_helper_detects_differences(oracle, corpus_columns):
    """oracle/parity.compare_grid (the full-grid checker of the GPU tests):
    the oracle against itself is exact; a perturbed cell and a flipped code
    are both caught; fp32 grids carry the reference's own fp32 error."""
    from oracle.parity import compare_grid
    cols = corpus_columns[:, :23]
    times = np.linspace(0.0, 1440.0, 17)
    p64, c64 = oracle.grid(oracle.init_columns(cols, 64), times)
    same = compare_grid(cols, times, lambda lo, hi: (p64[:, lo:hi], c64[lo:hi]), 64, band_rows=5)
    assert same.cells == 23 * 17 and same.code_mismatch_fp64 == 0 and same.dr_max == 0.0
    bad_p, bad_c = p64.copy(), c64.copy()
    ok = np.argwhere(c64 == 0)
    i, j = ok[len(ok) // 2]
    bad_p[1, i, j] += 2e-6
    bad_c[ok[0][0], ok[0][1]] = 6
    bad = compare_grid(cols, times, lambda lo, hi: (bad_p[:, lo:hi], bad_c[lo:hi]), 64, band_rows=7)
    assert bad.code_mismatch_fp64 == 1 and abs(bad.dr_max - 2e-6) < 1e-9
    p32, c32 = oracle.grid(oracle.init_columns(cols, 32), times)
    s32 = compare_grid(cols, times, lambda lo, hi: (p32[:, lo:hi], c32[lo:hi]), 32).summary()
    assert s32["code_mismatch_vs_ref_same_precision"] == 0
    assert s32["dr_max_km"] == s32["ref_fp32_dr_max_km"] > 0
