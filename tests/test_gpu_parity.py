"""GPU parity: the CUDA kernels (through the C ABI) against the CPU oracle,
which is itself pinned bit-for-bit to the reference (test_oracle.py).

Tolerances (BASELINE.json north_star):
  fp64: |dr| <= 1 mm (1e-6 km), |dv| <= 1e-6 km/s, error codes bit-exact;
  fp32: error codes bit-exact vs the reference at fp32 AND fp64; position /
        velocity error vs the reference fp64 path is reported (and bounded
        loosely so a regression cannot hide).
"""

import dataclasses
import io

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL64_R = 1.0e-6     # km
TOL64_V = 1.0e-6     # km/s


def _gpu():
    import paper_2603_27830_b200 as pkg
    return pkg


def _diff(planes, ref_planes, mask):
    dr = np.linalg.norm((planes[:3].astype(np.float64) - ref_planes[:3])[:, mask], axis=0)
    dv = np.linalg.norm((planes[3:].astype(np.float64) - ref_planes[3:])[:, mask], axis=0)
    return dr, dv


@pytest.fixture(scope="module")
def corpus_ref64(oracle, corpus_columns):
    times = np.linspace(0.0, 1440.0, 200)
    sat = oracle.init_columns(corpus_columns, 64)
    return times, oracle.grid(sat, times, workers=4)


@pytest.mark.parametrize("times_kind", ["day", "fortnight"])
def test_fp64_corpus_parity(oracle, corpus_columns, corpus_ref64, times_kind):
    pkg = _gpu()
    if times_kind == "day":
        times, (ref_planes, ref_codes) = corpus_ref64
    else:
        times = np.arange(0.0, 20160.0, 101.0)
        ref_planes, ref_codes = oracle.grid(oracle.init_columns(corpus_columns, 64), times,
                                            workers=4)
    res = pkg.propagate_batch(pkg.init_batch(corpus_columns, precision=64), times)
    assert res.planes.dtype == np.float64 and res.error.dtype == np.int32
    assert np.array_equal(res.error, ref_codes)
    ok = ref_codes == 0
    dr, dv = _diff(res.planes, ref_planes, ok)
    print(f"\nfp64 {times_kind}: {ok.sum()} ok cells, max|dr|={dr.max():.3e} km, "
          f"max|dv|={dv.max():.3e} km/s, nonzero codes={int((~ok).sum())}")
    assert dr.max() <= TOL64_R and dv.max() <= TOL64_V
    assert np.isfinite(res.planes).all()


def test_fp64_matches_reference_goldens(golden_columns, golden_states):
    pkg = _gpu()
    g = golden_states[64]
    res = pkg.propagate_batch(pkg.init_batch(golden_columns, precision=64), g["times"])
    assert np.array_equal(res.error, g["error"])
    dr, dv = _diff(res.planes, g["planes"], g["error"] == 0)
    assert dr.max() <= TOL64_R and dv.max() <= TOL64_V


def test_fp32_codes_and_accuracy(oracle, corpus_columns, corpus_ref64):
    pkg = _gpu()
    times, (ref64, codes64) = corpus_ref64
    ref32, codes32 = oracle.grid(oracle.init_columns(corpus_columns, 32), times, workers=4)
    res = pkg.propagate_batch(pkg.init_batch(corpus_columns, precision=32), times)
    assert res.planes.dtype == np.float32
    assert np.array_equal(res.error, codes64)
    assert np.array_equal(res.error, codes32)
    ok = codes64 == 0
    dr, dv = _diff(res.planes, ref64, ok)
    print(f"\nfp32 vs reference fp64 (1,200 x 200, 1 day): |dr| median "
          f"{np.median(dr) * 1e3:.2f} m p99 {np.percentile(dr, 99) * 1e3:.2f} m max "
          f"{dr.max() * 1e3:.2f} m; |dv| max {dv.max() * 1e3:.4f} m/s")
    assert np.median(dr) < 0.05 and dr.max() < 1.0 and dv.max() < 1e-3
    # and well inside the reference's own fp32 error on the same cells
    dr_ref, _ = _diff(ref32, ref64, ok)
    assert np.median(dr) < 0.5 * np.median(dr_ref)
    assert np.percentile(dr, 99) < 0.5 * np.percentile(dr_ref, 99) and dr.max() < dr_ref.max()


def test_fp32_goldens_codes(golden_columns, golden_states):
    pkg = _gpu()
    g = golden_states[32]
    res = pkg.propagate_batch(pkg.init_batch(golden_columns, precision=32), g["times"])
    assert np.array_equal(res.error, g["error"])
    assert np.array_equal(res.error, golden_states[64]["error"])


@pytest.mark.parametrize("precision", [64, 32])
def test_failure_modes(failure_table, precision):
    pkg = _gpu()
    times = np.array(failure_table["times"])
    cols = np.array([row["elements"] for row in failure_table["cases"].values()]).T
    sats = pkg.init_batch(cols, precision=precision)
    res = pkg.propagate_batch(sats, times)
    for k, (key, row) in enumerate(failure_table["cases"].items()):
        assert int(sats.error_codes[k]) == row[f"init_code_{precision}"], key
        assert res.error[k].tolist() == row[f"codes_{precision}"], key
        if row[f"finite_{precision}"]:       # the reference itself overflows on 2 cases
            assert np.isfinite(res.planes[:, k]).all(), key


def test_init_constants_vs_oracle(oracle, golden_columns, golden_states):
    pkg = _gpu()
    sats = pkg.init_batch(golden_columns, precision=64)
    init = sats.init
    ref = golden_states[64]
    for name in oracle.SATREC_FIELDS:
        np.testing.assert_allclose(np.asarray(getattr(init, name)), ref["init_" + name],
                                   rtol=1e-12, atol=1e-300, err_msg=name)
    assert np.array_equal(init.isimp, ref["init_isimp"])
    assert np.array_equal(init.error_code_at_init, ref["init_error_code_at_init"])
    init32 = pkg.init_batch(golden_columns, precision=32).init
    assert init32.cc1.dtype == np.float32 and init32.dtype == np.float32


@pytest.mark.parametrize("precision,dtype", [(64, np.float64), (32, np.float32)])
def test_batch_equals_scalar_bitwise(real_elements, precision, dtype):
    """tests/test_batch.py:39-64 of the reference: batch cell == scalar call."""
    pkg = _gpu()
    els = list(real_elements.values())
    times = np.array([0.0, 30.0, 720.0, 1440.0, -60.0, 4321.5, 20160.0])
    res = pkg.propagate_batch(pkg.init_batch(els, precision=precision), times)
    for i, el in enumerate(els):
        init = pkg.sgp4_init(el, dtype=dtype)
        for j, t in enumerate(times):
            s = pkg.sgp4_propagate(init, dtype(t))
            assert np.asarray(s.r).dtype == dtype
            assert np.array_equal(res.planes[:3, i, j], np.asarray(s.r))
            assert np.array_equal(res.planes[3:, i, j], np.asarray(s.v))
            assert res.error[i, j] == int(np.asarray(s.error_code))


def test_scalar_broadcast_shapes(real_elements):
    pkg = _gpu()
    el = real_elements["ISS"]
    init = pkg.sgp4_init(el)
    s = pkg.sgp4_propagate(init, 60.0)
    assert np.asarray(s.r).shape == (3,) and np.asarray(s.error_code).shape == ()
    s = pkg.sgp4_propagate(init, np.array([0.0, 60.0, 120.0]))
    assert s.r.shape == (3, 3) and s.error_code.shape == (3,)
    # edited SatInit (dataclasses.replace) is re-packed on the GPU
    edited = dataclasses.replace(init, bstar=np.asarray(init.bstar) * 2)
    s2 = pkg.sgp4_propagate(edited, 60.0)
    assert np.isfinite(s2.r).all()


@pytest.mark.parametrize("n,m", [(1, 1), (2, 3), (33, 5), (7, 127), (5, 129), (3, 1001)])
def test_odd_shapes_match_oracle(oracle, corpus_columns, n, m):
    pkg = _gpu()
    cols = corpus_columns[:, :n]
    times = np.linspace(-100.0, 3000.0, m)
    res = pkg.propagate_batch(pkg.init_batch(cols, precision=64), times)
    ref_planes, ref_codes = oracle.grid(oracle.init_columns(cols, 64), times)
    assert np.array_equal(res.error, ref_codes)
    dr, dv = _diff(res.planes, ref_planes, ref_codes == 0)
    assert dr.max(initial=0) <= TOL64_R and dv.max(initial=0) <= TOL64_V


@pytest.mark.parametrize("precision", [64, 32])
def test_row_shards_bitwise_equal_full_grid(corpus_columns, precision):
    """Satellite sharding (one GPU per range, no collective) is bitwise
    invariant — the analogue of reference worker invariance."""
    import torch
    from paper_2603_27830_b200 import _device
    pkg = _gpu()
    sats = pkg.init_batch(corpus_columns[:, :301], precision=precision)
    times = np.linspace(0.0, 1440.0, 77)
    full = pkg.propagate_batch_device(sats, times)
    from paper_2603_27830_b200.batch import _alloc_grid
    t_d = torch.from_numpy(times.astype(sats.dtype)).cuda()
    for lo, hi in pkg.partition_work(301, 1, 4):
        planes, err = _alloc_grid(hi - lo, 77, precision, torch.device("cuda"))
        _device.propagate_grid(sats.device_satrec, t_d, planes, err, rows=(lo, hi))
        assert torch.equal(planes, full.planes[:, lo:hi])
        assert torch.equal(err, full.error[lo:hi])


def test_streamed_tiles_match_dense(corpus_columns):
    pkg = _gpu()
    sats = pkg.init_batch(corpus_columns[:, :7])
    times = np.linspace(0.0, 720.0, 9)
    dense = pkg.propagate_batch(sats, times)
    got = np.full_like(dense.planes, np.nan)
    got_err = np.full_like(dense.error, -1)
    seen = []

    def sink(rows, cols, planes, error):
        seen.append((rows.start, cols.start))
        got[:, rows, cols] = planes
        got_err[rows, cols] = error

    summary = pkg.propagate_batch_streamed(sats, times, tile_rows=3, tile_cols=4, sink=sink)
    assert seen == sorted(seen)
    assert np.array_equal(got, dense.planes) and np.array_equal(got_err, dense.error)
    assert summary.cells_emitted == 7 * 9
    assert summary.nonzero_error_count == int(np.count_nonzero(dense.error))

    calls = []

    def failing(rows, cols, planes, error):
        calls.append(1)
        if len(calls) == 3:
            raise IOError("disk full")

    with pytest.raises(pkg.StreamAborted) as exc:
        pkg.propagate_batch_streamed(pkg.init_batch(corpus_columns[:, :4]),
                                     np.linspace(0.0, 720.0, 4), 1, 2, failing)
    assert exc.value.tiles_completed == 2


def test_sgb1_from_device_equals_host(corpus_columns):
    pkg = _gpu()
    sats = pkg.init_batch(corpus_columns[:, :3], precision=32)
    times = np.array([0.0, 60.0, 120.0, 240.0, 480.0])
    host = pkg.propagate_batch(sats, times)
    dev = pkg.propagate_batch_device(sats, times)
    a, b = io.BytesIO(), io.BytesIO()
    pkg.write_grid_binary(host, a)
    pkg.write_grid_binary(dev, b)
    assert a.getvalue() == b.getvalue()
    raw = a.getvalue()
    assert raw[:4] == b"SGB1" and raw[24:32] == b"rrrvvve\x00"
    back = pkg.read_grid_binary(io.BytesIO(raw))
    assert np.array_equal(back.planes, host.planes) and np.array_equal(back.error, host.error)


def test_validation_errors(corpus_columns):
    pkg = _gpu()
    sats = pkg.init_batch(corpus_columns[:, :1])
    with pytest.raises(ValueError):
        pkg.propagate_batch(sats, np.empty(0))
    with pytest.raises(ValueError):
        pkg.propagate_batch(sats, np.zeros((2, 2)))
    with pytest.raises(ValueError):
        pkg.init_batch([])
    with pytest.raises(ValueError):
        pkg.init_batch(corpus_columns[:, :1], precision=16)
    with pytest.raises(pkg.GridAllocationError):
        pkg.propagate_batch_device(pkg.init_batch(corpus_columns), np.zeros(10 ** 9))


def test_solve_kepler_gpu():
    import math
    from paper_2603_27830_b200.kernel import solve_kepler
    ax = np.array([0.1, 0.0, 0.02, 0.3])
    ay = np.array([0.0, 0.05, 0.03, -0.2])
    u = np.array([1.0, 2.5, 5.9, 0.4])
    e = solve_kepler(ax, ay, u)
    res = u - (e - ax * np.sin(e) + ay * np.cos(e))
    assert np.abs(res).max() < 1e-12
    assert float(solve_kepler(np.float64(0), np.float64(0), np.float64(1.2345))) == 1.2345
    singles = np.array([float(solve_kepler(a, b, c)) for a, b, c in zip(ax, ay, u)])
    assert np.array_equal(singles, e)
    assert math.isfinite(float(solve_kepler(np.float32(0.3), np.float32(0.2), np.float32(1.0))))


def test_starlink_full_size_properties():
    """C2 at full size (9,341 x 1,000): properties that need no oracle —
    no error codes, finite, plausible LEO radii/speeds, fp32 close to fp64
    on every cell — plus a 2,000-cell random sample checked against the
    oracle."""
    import torch
    from oracle import sgp4_oracle as oracle
    from paper_2603_27830_b200.catalog import starlink_like
    pkg = _gpu()
    cols = starlink_like(9341)
    times = np.linspace(0.0, 1440.0, 1000)
    r32 = pkg.propagate_batch_device(pkg.init_batch(cols, precision=32), times)
    r64 = pkg.propagate_batch_device(pkg.init_batch(cols, precision=64), times)
    assert int(torch.count_nonzero(r32.error)) == 0 and int(torch.count_nonzero(r64.error)) == 0
    rad = torch.linalg.vector_norm(r64.planes[:3], dim=0)
    spd = torch.linalg.vector_norm(r64.planes[3:], dim=0)
    assert 6700 < float(rad.min()) and float(rad.max()) < 7000
    assert 7.2 < float(spd.min()) and float(spd.max()) < 7.9
    d = torch.linalg.vector_norm(r32.planes[:3].double() - r64.planes[:3], dim=0)
    print(f"\nC2 fp32 vs GPU fp64: median {float(d.median()) * 1e3:.2f} m, "
          f"max {float(d.max()) * 1e3:.2f} m")
    assert float(d.max()) < 1.0
    rng = np.random.default_rng(7)
    ii = rng.integers(0, 9341, 2000)
    jj = rng.integers(0, 1000, 2000)
    sat = oracle.init_columns(cols[:, ii], 64)
    ref_r, ref_v, ref_c = oracle.propagate_merged(sat, times[jj])
    got = r64.planes[:, ii, jj].cpu().numpy()
    assert (ref_c == 0).all()
    assert np.abs(got[:3].T - ref_r).max() <= TOL64_R
    assert np.abs(got[3:].T - ref_v).max() <= TOL64_V


def test_drift_report_gpu(corpus_columns):
    """drift_report on the GPU: the reference's acceptance bands
    (test_acceptance.py:107-122) and nearest-rank percentiles identical to a
    host recomputation from the same two device grids."""
    import dataclasses as dc
    import math as _m
    pkg = _gpu()
    from paper_2603_27830_b200.tle import MeanElements
    els = [MeanElements(*corpus_columns[:, i], 2023, 1, 0.0) for i in range(120)]
    rep = pkg.drift_report(els, horizon_days=14.0, step_minutes=90.0)
    epoch_m = rep.p50_km[0] * 1000.0
    print(f"\ndrift: epoch median {epoch_m:.3f} m, day-14 median {rep.p50_km[-1]:.4f} km, "
          f"{rep.p50_kms[-1] * 1000:.4f} m/s")
    assert 0.1 <= epoch_m <= 10.0
    assert rep.p50_km[-1] < 1.0 and rep.p50_kms[-1] * 1000.0 < 10.0
    # host recomputation with the reference's nearest-rank rule
    times = np.arange(0.0, 14.0 * 1440.0 + 45.0, 90.0)
    lo = pkg.propagate_batch(pkg.init_batch(els, precision=32), times)
    hi = pkg.propagate_batch(pkg.init_batch(els, precision=64), times)
    inc = (lo.error == 0) & (hi.error == 0)
    dr = np.linalg.norm(lo.r.astype(np.float64) - hi.r, axis=-1)
    for j in (0, 37, len(times) - 1):
        v = np.sort(dr[inc[:, j], j])
        want = v[max(1, int(np.ceil(0.5 * v.size))) - 1]
        assert rep.p50_km[j] == want
    assert rep.included_cells == int(inc.sum())
    csv_text = pkg.emit_report_csv(rep)
    assert csv_text.splitlines()[0].startswith("day,p5_km")
    bad = [dc.replace(els[0], no_kozai=0.0)]
    with pytest.raises(pkg.EmptyReportError):
        pkg.drift_report(bad, 1.0, 60.0)
    assert not _m.isnan(rep.p95_kms[-1])


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_randomized_grids(oracle, corpus_columns, seed):
    """Random sub-catalogues and time grids (incl. negative and 14-day
    times): fp64 within tolerance, codes equal at both precisions, and the
    broadcasting scalar API equal to the batch bit for bit."""
    pkg = _gpu()
    rng = np.random.default_rng(seed)
    n, m = int(rng.integers(1, 40)), int(rng.integers(1, 300))
    cols = corpus_columns[:, rng.integers(0, corpus_columns.shape[1], n)]
    times = np.sort(rng.uniform(-1440.0, 20160.0, m))
    ref64, codes64 = oracle.grid(oracle.init_columns(cols, 64), times)
    _, codes32 = oracle.grid(oracle.init_columns(cols, 32), times)
    for precision, dtype, ref_codes in ((64, np.float64, codes64), (32, np.float32, codes32)):
        sats = pkg.init_batch(cols, precision=precision)
        res = pkg.propagate_batch(sats, times)
        assert np.array_equal(res.error, ref_codes)
        assert np.array_equal(res.error, codes64)
        if precision == 64:
            dr, dv = _diff(res.planes, ref64, ref_codes == 0)
            assert dr.max(initial=0) <= TOL64_R and dv.max(initial=0) <= TOL64_V
        # broadcasting scalar API: the batch's own SatInit (n,) against
        # times (m, 1) -> (m, n).  (A hand-edited fp32 SatInit would be
        # re-packed from its fp32-rounded fields, like the reference's fp32
        # path, so it is not expected to match the fp64-initialised batch.)
        st = pkg.sgp4_propagate(sats.init, times.astype(dtype)[:, None])
        assert st.r.shape == (m, n, 3)
        # error cells may carry NaN (as in the reference), hence equal_nan
        assert np.array_equal(np.transpose(st.r, (2, 1, 0)), res.planes[:3], equal_nan=True)
        assert np.array_equal(np.transpose(st.v, (2, 1, 0)), res.planes[3:], equal_nan=True)
        st = type(st)(r=st.r, v=st.v, error_code=st.error_code.T)
        assert np.array_equal(st.error_code, res.error)
        # general (non-Cartesian) broadcast: satellite i at its own time
        jj = rng.integers(0, m, n)
        sd = pkg.sgp4_propagate(sats.init, times.astype(dtype)[jj])
        assert sd.r.shape == (n, 3)
        ii = np.arange(n)
        assert np.array_equal(sd.r.T, res.planes[:3, ii, jj], equal_nan=True)
        assert np.array_equal(sd.v.T, res.planes[3:, ii, jj], equal_nan=True)
        assert np.array_equal(sd.error_code, res.error[ii, jj])


@pytest.mark.parametrize("n,m", [(1, 1), (3, 5), (33, 127), (5, 1001)])
def test_fp32_odd_shapes_codes_and_bounds(oracle, corpus_columns, n, m):
    """fp32 grids of unaligned width (padded device rows): codes equal the
    reference at both precisions, errors bounded against the fp64 oracle."""
    pkg = _gpu()
    cols = corpus_columns[:, 7:7 + n]
    times = np.linspace(-100.0, 3000.0, m)
    res = pkg.propagate_batch(pkg.init_batch(cols, precision=32), times)
    assert res.planes.shape == (6, n, m) and res.planes.flags["C_CONTIGUOUS"]
    ref64, codes64 = oracle.grid(oracle.init_columns(cols, 64), times)
    _, codes32 = oracle.grid(oracle.init_columns(cols, 32), times)
    assert np.array_equal(res.error, codes64) and np.array_equal(res.error, codes32)
    dr, _ = _diff(res.planes, ref64, codes64 == 0)
    assert dr.max(initial=0) < 0.5


def test_streamed_fp32_matches_dense(corpus_columns):
    pkg = _gpu()
    sats = pkg.init_batch(corpus_columns[:, :50], precision=32)
    times = np.linspace(0.0, 2880.0, 301)
    dense = pkg.propagate_batch(sats, times)
    got = np.empty_like(dense.planes)
    got_err = np.empty_like(dense.error)

    def sink(rows, cols, planes, error):
        assert planes.dtype == np.float32
        got[:, rows, cols] = planes
        got_err[rows, cols] = error

    summary = pkg.propagate_batch_streamed(sats, times, tile_rows=17, tile_cols=64, sink=sink)
    assert summary.cells_emitted == 50 * 301
    assert np.array_equal(got, dense.planes) and np.array_equal(got_err, dense.error)


def test_device_result_views_and_gather(corpus_columns):
    """propagate_batch_device returns (6, N, M)/(N, M) views (rows padded to
    4 steps); BatchResult.r/.v work on device tensors; shard gather on one
    rank is the identity."""
    import torch
    from paper_2603_27830_b200.shard import gather_grid, propagate_sharded, shard_bounds
    pkg = _gpu()
    res = pkg.propagate_batch_device(pkg.init_batch(corpus_columns[:, :9], precision=32),
                                     np.linspace(0.0, 100.0, 7))
    assert tuple(res.planes.shape) == (6, 9, 7) and tuple(res.r.shape) == (9, 7, 3)
    assert res.planes.stride(1) == 8          # padded row
    host = pkg.propagate_batch(pkg.init_batch(corpus_columns[:, :9], precision=32),
                               np.linspace(0.0, 100.0, 7))
    assert np.array_equal(res.planes.cpu().numpy(), host.planes)
    local, (axis, lo, hi) = propagate_sharded(corpus_columns[:, :9], np.linspace(0.0, 100.0, 7))
    assert axis == "rows" and (lo, hi) == shard_bounds(9, 1, 0) == (0, 9)
    p, e = gather_grid(local.planes, local.error, 9)
    assert torch.equal(p, local.planes) and torch.equal(e, local.error)


def test_fp32_kepler_classes_and_drag(oracle, corpus_columns):
    """The fp32 cell specialises on the satellite's Kepler class (e < 0.003:
    series for 1/den, betal, 1/(1+betal), 1/pl; e < 0.1; e < 0.4; other) and
    on isimp.  Sweep eccentricity across every class boundary and B* (either sign) over
    three decades for two weeks: codes must equal the reference fp64 codes,
    and the fp32 error against reference fp64 must stay within the
    reference's own fp32 error on the same cells (+50 m)."""
    pkg = _gpu()
    eccs = [1e-5, 1e-4, 0.0029, 0.0031, 0.02, 0.099, 0.101, 0.3, 0.41, 0.6]
    bstars = [1e-5, 3e-4, 5e-3, -3e-4, -5e-3]
    base = corpus_columns[:, :2]          # one regular, one low-perigee-ish LEO
    cols = []
    for e in eccs:
        for b in bstars:
            for k in range(base.shape[1]):
                c = base[:, k].copy()
                c[1] = e
                c[6] = b
                cols.append(c)
    cols = np.array(cols).T
    times = np.arange(0.0, 20160.0, 97.0)
    ref64, codes64 = oracle.grid(oracle.init_columns(cols, 64), times, workers=4)
    ref32, _ = oracle.grid(oracle.init_columns(cols, 32), times, workers=4)
    res = pkg.propagate_batch(pkg.init_batch(cols, precision=32), times)
    assert np.array_equal(res.error, codes64)
    ok = codes64 == 0
    dr, _ = _diff(res.planes, ref64, ok)
    dr_ref, _ = _diff(ref32, ref64, ok)
    print(f"\nfp32 class sweep ({cols.shape[1]} sats x {times.size}): max|dr| {dr.max() * 1e3:.1f} m "
          f"(reference fp32 {dr_ref.max() * 1e3:.1f} m), ok cells {int(ok.sum())}")
    assert dr.max() <= dr_ref.max() + 0.05 and dr.max() < 0.5
    res64 = pkg.propagate_batch(pkg.init_batch(cols, precision=64), times)
    assert np.array_equal(res64.error, codes64)
    dr64, dv64 = _diff(res64.planes, ref64, ok)
    assert dr64.max() <= TOL64_R and dv64.max() <= TOL64_V


def test_c5_full_size_properties():
    """C5 at full size on one GPU (1,000,000 x 1,000 fp32: 28 GB of output):
    no error codes, finite, plausible LEO radii and speeds on every cell,
    rows sharded 8 ways into the same buffer reproduce it bitwise, and a
    random sample of cells agrees with the oracle's fp64 path."""
    import torch
    from oracle import sgp4_oracle as oracle
    from paper_2603_27830_b200 import _device
    from paper_2603_27830_b200.catalog import starlink_like
    from paper_2603_27830_b200.shard import shard_bounds
    pkg = _gpu()
    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~30 GB of free HBM")
    n, m = 1_000_000, 1000
    cols = starlink_like(n)
    times = np.linspace(0.0, 1440.0, m)
    sats = pkg.init_batch(cols, precision=32)
    res = pkg.propagate_batch_device(sats, times)
    assert int(torch.count_nonzero(res.error)) == 0
    for p0 in (0, 3):
        norm = torch.linalg.vector_norm(res.planes[p0:p0 + 3].float(), dim=0)
        lo, hi = float(norm.min()), float(norm.max())
        assert np.isfinite(lo) and np.isfinite(hi)
        if p0 == 0:
            assert 6650 < lo and hi < 7050
        else:
            assert 7.2 < lo and hi < 7.95
        del norm
    # 8 row shards launched into a second buffer equal the single launch
    t_d = torch.from_numpy(times.astype(np.float32)).cuda()
    planes2 = torch.empty_like(res.planes)
    codes2 = torch.empty_like(res.error)
    for r in range(8):
        a, b = shard_bounds(n, 8, r)
        _device.propagate_grid(sats.device_satrec, t_d, planes2[:, a:b], codes2[a:b],
                               rows=(a, b))
    assert torch.equal(planes2, res.planes) and torch.equal(codes2, res.error)
    del planes2, codes2
    rng = np.random.default_rng(11)
    ii = rng.integers(0, n, 3000)
    jj = rng.integers(0, m, 3000)
    sat = oracle.init_columns(cols[:, ii], 64)
    ref_r, ref_v, ref_c = oracle.propagate_merged(sat, times[jj])
    got = res.planes[:, torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda()].cpu().numpy()
    assert (ref_c == 0).all()
    dr = np.linalg.norm(got[:3].T.astype(np.float64) - ref_r, axis=1)
    print(f"\nC5 fp32 sample vs oracle fp64: median {np.median(dr) * 1e3:.2f} m, "
          f"max {dr.max() * 1e3:.2f} m")
    assert dr.max() < 0.2


def test_scaling_sweep_gpu(real_elements):
    """The reference's sweep harness over the GPU path (bench.py:91-124)."""
    pkg = _gpu()
    els = list(real_elements.values())
    recs = pkg.scaling_sweep("satellites", [3, 17], 50, els, precision=32, full_pipeline=False)
    assert [r.n for r in recs] == [3, 17] and all(r.m == 50 for r in recs)
    assert all(r.throughput_cells_per_s > 0 and r.trials == 5 for r in recs)
    from paper_2603_27830_b200.timing import emit_bench_csv
    assert emit_bench_csv(recs).splitlines()[1].startswith("satellites-3,satellites,3,50,32")


def test_streamed_memory_contract(corpus_columns):
    """propagate_batch_streamed keeps O(tile) host memory (the reference's
    tracemalloc contract, test_batch.py:152-173): the pinned host bytes
    while streaming a 2,000 x 2,000 grid (112 MB dense) in 100 x 500 tiles
    stay within a few tiles, and no dense device grid is allocated either."""
    import torch
    from paper_2603_27830_b200 import _hostmem
    pkg = _gpu()
    sats = pkg.init_batch(np.tile(corpus_columns, (1, 2))[:, :2000], precision=32)
    times = np.linspace(0.0, 1440.0, 2000)
    tile_bytes = 100 * 500 * 28
    torch.cuda.synchronize()
    _hostmem.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    host0 = _hostmem.stats()["pinned_bytes"]
    dev0 = torch.cuda.memory_allocated()
    count = [0]
    peak = [0]

    def sink(rows, cols, planes, error):
        count[0] += 1
        peak[0] = max(peak[0], _hostmem.stats()["pinned_bytes"] - host0)
    summary = pkg.propagate_batch_streamed(sats, times, 100, 500, sink)
    assert count[0] == 20 * 4 and summary.cells_emitted == 2000 * 2000
    dev_peak = torch.cuda.max_memory_allocated() - dev0
    assert peak[0] <= 4 * tile_bytes, peak[0]
    assert dev_peak <= 8 * tile_bytes + (1 << 20), dev_peak


def test_pinned_results_released(corpus_columns):
    """propagate_batch's arrays live in one pooled page-locked block of the
    grid's exact size (2 MiB rounding, not a power of two); the block returns
    to the pool when the arrays die and empty_cache() unpins it."""
    import gc
    from paper_2603_27830_b200 import _hostmem
    pkg = _gpu()
    gc.collect()                  # earlier tests' blocks still waiting in cycles
    _hostmem.empty_cache()
    base = _hostmem.stats()["pinned_bytes"]
    sats = pkg.init_batch(np.tile(corpus_columns, (1, 3))[:, :3000], precision=32)
    res = pkg.propagate_batch(sats, np.linspace(0.0, 1440.0, 1000))
    want = 3000 * 1000 * 28
    live = _hostmem.stats()["pinned_bytes"] - base
    assert want <= live <= want + (2 << 20) + 256, live
    again = pkg.propagate_batch(sats, np.linspace(0.0, 1440.0, 1000))
    assert np.array_equal(again.planes, res.planes) and np.array_equal(again.error, res.error)
    del res, again
    gc.collect()
    st = _hostmem.stats()
    assert st["cached_bytes"] >= want and st["reuses"] >= 0
    _hostmem.empty_cache()
    assert _hostmem.stats()["pinned_bytes"] == base


def test_times_lo_path_matches_oracle(oracle, corpus_columns):
    """fp32 batch fed fp64 times as (hi, lo) float32 words (times_lo): codes
    equal the reference fp64 codes and states stay within the fp32 bound of
    the oracle's fp64 path evaluated at the exact fp64 times."""
    import torch
    from paper_2603_27830_b200.batch import split_times
    pkg = _gpu()
    cols = corpus_columns[:, :40]
    times = np.linspace(-300.0, 20160.0, 203) + 1.0 / 3.0
    hi, lo = split_times(times)
    sats = pkg.init_batch(cols, precision=32)
    res = pkg.propagate_batch_device(sats, torch.from_numpy(hi).cuda(),
                                     times_lo=torch.from_numpy(lo).cuda())
    ref64, codes64 = oracle.grid(oracle.init_columns(cols, 64), times)
    assert np.array_equal(res.error.cpu().numpy(), codes64)
    planes = res.planes.cpu().numpy()
    dr, _ = _diff(planes, ref64, codes64 == 0)
    plain = pkg.propagate_batch(sats, hi)
    dr_plain, _ = _diff(plain.planes, ref64, codes64 == 0)
    print(f"\ntimes_lo: max|dr| {dr.max() * 1e3:.2f} m (hi word only: {dr_plain.max() * 1e3:.2f} m)")
    assert dr.max() < 0.5 and dr.max() <= dr_plain.max()
    with pytest.raises(ValueError):
        pkg.propagate_batch_device(sats, torch.from_numpy(hi).cuda(),
                                   times_lo=torch.from_numpy(lo[:-1]).cuda())
    with pytest.raises(TypeError):
        pkg.propagate_batch_device(sats, torch.from_numpy(hi).cuda(),
                                   times_lo=torch.from_numpy(lo.astype(np.float64)).cuda())


def test_out_validation(corpus_columns):
    """propagate_batch_device(out=...) rejects buffers the kernel would
    overrun or misinterpret, and accepts a correct pair."""
    import torch
    pkg = _gpu()
    sats = pkg.init_batch(corpus_columns[:, :5], precision=32)
    t = np.linspace(0.0, 60.0, 8)
    dev = torch.device("cuda", torch.cuda.current_device())
    good = (torch.empty((6, 5, 8), device=dev), torch.empty((5, 8), dtype=torch.int32, device=dev))
    res = pkg.propagate_batch_device(sats, t, out=good)
    assert res.planes.data_ptr() == good[0].data_ptr()
    bad = [
        (torch.empty((6, 4, 8), device=dev), good[1]),                      # too few rows
        (torch.empty((5, 5, 8), device=dev), good[1]),                      # too few planes
        (good[0], torch.empty((5, 7), dtype=torch.int32, device=dev)),      # short code rows
        (torch.empty((6, 5, 16), device=dev)[:, :, ::2], good[1]),          # column stride 2
    ]
    for out in bad:
        with pytest.raises(ValueError):
            pkg.propagate_batch_device(sats, t, out=out)
    for out in [(good[0].double(), good[1]), (good[0], good[1].long())]:
        with pytest.raises(TypeError):
            pkg.propagate_batch_device(sats, t, out=out)
    with pytest.raises(ValueError):
        pkg.propagate_batch_device(sats, t, out=(good[0].cpu(), good[1].cpu()))


def test_bench_json_contract():
    """bench.py prints one JSON line with the driver's keys (N=1)."""
    import json
    import subprocess
    import sys
    from tests.conftest import ROOT
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "5", "--warmup", "3",
                          "--e2e-steps", "1", "--no-cpu"], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] >= 3 and d["gpu_launches"] == 5
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0
    # planes + code-row flags (the synthetic catalogue has no failing cell,
    # so no code row crosses PCIe; the host zero-fills the whole code plane)
    assert e["d2h_bytes_per_step"] == 9341 * 1000 * 24 + 9341
    assert e["code_plane_bytes_zero_filled_on_host"] == 9341 * 1000 * 4
    assert 0 < e["pcie_frac"] <= 1.1
    assert "workload" in d["config"] and d["value"] > 1e10
    acc = d["accuracy"]
    assert acc["cells_compared"] == 9341 * 1000 and acc["code_mismatch_vs_ref_fp64"] == 0
    assert acc["dr_max_km"] < 0.1


def test_bench_two_ranks_on_one_gpu():
    """The N>1 plumbing of bench.py (self-relaunch under torch.distributed.run,
    barrier, MAX over ranks, weak-scaling value) with 2 ranks sharing the one
    GPU through the gloo test backend."""
    import json
    import os
    import subprocess
    import sys
    from tests.conftest import ROOT
    env = dict(os.environ, SGP4B_BENCH_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "4",
                          "--warmup", "3", "--e2e-steps", "1", "--no-cpu", "--no-accuracy"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak"
    assert d["config"]["cells_per_gpu"] == 9341 * 1000
    assert abs(d["value"] - 2 * 9341 * 1000 / (d["ms_per_step"] * 1e-3)) < 1e-6 * d["value"]
    ref = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl",
                          "reference", "--steps", "1", "--warmup", "0", "--ref-rows", "50"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert ref.returncode == 0, ref.stderr[-3000:]
    rl = [ln for ln in ref.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(rl) == 1
    r = json.loads(rl[0])
    assert r["impl"] == "reference" and r["config"] == d["config"]


@pytest.mark.parametrize("precision", [32, 64])
def test_sparse_code_rows_with_errors(failure_table, corpus_columns, precision):
    """propagate_batch / propagate_batch_streamed move only the code rows that
    hold a nonzero code; with failure-mode satellites mixed into a corpus
    the host code planes still equal the device grid exactly."""
    import torch
    pkg = _gpu()
    bad = np.array([row["elements"] for row in failure_table["cases"].values()]).T
    cols = np.concatenate([corpus_columns[:, :5], bad, corpus_columns[:, 5:9]], axis=1)
    times = np.array(failure_table["times"] + [4000.0, 9000.0])
    sats = pkg.init_batch(cols, precision=precision)
    host = pkg.propagate_batch(sats, times)
    dev = pkg.propagate_batch_device(sats, times)
    assert np.count_nonzero(host.error) > 0
    assert np.array_equal(host.error, dev.error.cpu().numpy())
    assert np.array_equal(host.planes, dev.planes.cpu().numpy(), equal_nan=True)
    got = np.full_like(host.error, -1)

    def sink(rows, cols_, planes, error):
        got[rows, cols_] = error
    summary = pkg.propagate_batch_streamed(sats, times, 3, 4, sink)
    assert np.array_equal(got, host.error)
    assert summary.nonzero_error_count == int(np.count_nonzero(host.error))


@pytest.mark.parametrize("precision", [64, 32])
def test_epoch_code_near_decay_threshold(oracle, precision):
    """Init codes across the epoch decay threshold (mrt = 1 earth radius at
    t = 0) and at larger eccentricities: the init kernel's bound that lets
    ordinary orbits skip the exact epoch evaluation (epoch_clear) never
    changes a code.  Perigees sweep 0.97..1.03 earth radii."""
    pkg = _gpu()
    rng = np.random.default_rng(11)
    n = 4000
    ecc = np.concatenate([rng.uniform(1e-6, 2e-3, n // 2), rng.uniform(2e-3, 0.45, n // 2)])
    rp = rng.uniform(0.97, 1.03, n)                       # perigee radius, earth radii
    a = rp / (1.0 - ecc)
    xke = 0.07436691613317342                             # WGS72 (gravity.py)
    no = xke / a ** 1.5
    cols = np.stack([no, ecc, rng.uniform(0, np.pi, n), rng.uniform(0, 2 * np.pi, n),
                     rng.uniform(0, 2 * np.pi, n), rng.uniform(0, 2 * np.pi, n),
                     rng.uniform(-1e-3, 1e-3, n)])
    sats = pkg.init_batch(cols, precision=precision)
    want = np.asarray(oracle.init_columns(cols, 64)["error_code_at_init"])
    got = np.asarray(sats.error_codes)
    assert np.array_equal(got, want), np.flatnonzero(got != want)[:10]
    assert (want == 6).sum() > 100 and (want == 0).sum() > 100


@pytest.mark.parametrize("precision", [32, 64])
def test_staged_pageable_result_equals_device(failure_table, corpus_columns, precision,
                                              monkeypatch):
    """Grids above the pinned pool's cache limit come back in pageable
    arrays through the pinned staging ring (pieces smaller than the grid, so
    the ring wraps); planes and codes equal the device grid bit for bit,
    with failing rows mixed in."""
    import torch
    pkg = _gpu()
    from paper_2603_27830_b200 import batch as batch_mod
    monkeypatch.setenv("SGP4B_HOST_CACHE_BYTES", "1")
    monkeypatch.setattr(batch_mod._StagedD2H, "PIECE", 1 << 16)
    monkeypatch.setattr(batch_mod._StagedD2H, "RING", 3)
    bad = np.array([row["elements"] for row in failure_table["cases"].values()]).T
    cols = np.concatenate([corpus_columns[:, :300], bad, corpus_columns[:, 300:400]], axis=1)
    times = np.linspace(-100.0, 3000.0, 257)
    sats = pkg.init_batch(cols, precision=precision)
    host = pkg.propagate_batch(sats, times)
    dev = pkg.propagate_batch_device(sats, times)
    assert np.count_nonzero(host.error) > 0
    assert np.array_equal(host.error, dev.error.cpu().numpy())
    assert np.array_equal(host.planes.view(np.uint8), dev.planes.cpu().numpy().view(np.uint8))


@pytest.mark.parametrize("precision", [32, 64])
def test_long_rows_split_into_column_blocks(corpus_columns, precision, monkeypatch):
    """Rows longer than one launch takes (2^30 steps) run as column blocks
    of the same grid; with the block length forced down to 100 the grid is
    bitwise equal to a single launch."""
    import torch
    pkg = _gpu()
    from paper_2603_27830_b200 import _device
    sats = pkg.init_batch(corpus_columns[:, :37], precision=precision)
    times = np.linspace(-30.0, 2000.0, 1003)
    whole = pkg.propagate_batch_device(sats, times)
    monkeypatch.setattr(_device, "MAX_STEPS_PER_LAUNCH", 100)
    split = pkg.propagate_batch_device(sats, times)
    assert torch.equal(whole.error, split.error)
    assert torch.equal(whole.planes.contiguous().view(torch.int8),
                       split.planes.contiguous().view(torch.int8))


@pytest.mark.parametrize("n,m", [(1, 3), (7, 5), (1000, 17), (50_000, 4)])
def test_drift_percentile_select_matches_sort(n, m):
    """sgp4b_drift_percentiles (per-column radix select) returns exactly the
    nearest-rank elements of a full column sort, with +inf cells excluded,
    ties, subnormals and an all-excluded column (NaN)."""
    import torch
    from paper_2603_27830_b200 import _native
    rng = np.random.default_rng(n + m)
    dr = rng.lognormal(-6, 2, size=(n, m))
    dv = rng.lognormal(-12, 3, size=(n, m))
    dr[rng.random((n, m)) < 0.1] = np.inf
    dv[rng.random((n, m)) < 0.1] = np.inf
    dr[:, 0] = np.inf                                   # a column with no finite cell
    if n > 3:
        dr[: n // 2, 1] = 1e-310                        # ties, subnormal
        dv[:, 2] = 0.0
    frac = np.array([0.05, 0.5, 0.95])
    table = torch.empty((6, m), dtype=torch.float64, device="cuda")
    counts = torch.empty((m,), dtype=torch.int64, device="cuda")
    d_r, d_v = torch.from_numpy(dr).cuda(), torch.from_numpy(dv).cuda()
    _native.check(_native.load().sgp4b_drift_percentiles(
        d_r.data_ptr(), d_v.data_ptr(), n, m, frac.ctypes.data, table.data_ptr(),
        counts.data_ptr(), None))
    got = table.cpu().numpy()
    for j in range(m):
        assert counts[j].item() == int(np.isfinite(dr[:, j]).sum())
        for q, x in enumerate((dr, dv)):
            col = np.sort(x[:, j])
            c = int(np.isfinite(x[:, j]).sum())
            for k, f in enumerate(frac):
                want = col[max(1, int(np.ceil(c * f))) - 1] if c else np.nan
                g = got[3 * q + k, j]
                assert (np.isnan(want) and np.isnan(g)) or g == want, (j, q, k, g, want)


@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("ndev", [1, 2, 3])
def test_device_grid_multi_device_bitwise(corpus_columns, failure_table, precision, ndev):
    """propagate_batch_device(devices=...): each device stores its rows
    straight into the home device's grid (peer memory on a multi-GPU box;
    the same GPU named several times here) — bitwise equal to one launch,
    also into a caller-provided `out`."""
    import torch
    pkg = _gpu()
    bad = np.array([row["elements"] for row in failure_table["cases"].values()]).T
    cols = np.concatenate([corpus_columns[:, :100], bad, corpus_columns[:, 100:157]], axis=1)
    sats = pkg.init_batch(cols, precision=precision)
    times = np.linspace(-60.0, 2880.0, 130)
    one = pkg.propagate_batch_device(sats, times)
    devs = [0] * ndev
    multi = pkg.propagate_batch_device(sats, times, devices=devs)
    torch.cuda.synchronize()
    assert torch.equal(one.error, multi.error)
    assert torch.equal(one.planes.contiguous().view(torch.int8),
                       multi.planes.contiguous().view(torch.int8))
    dt = torch.float32 if precision == 32 else torch.float64
    out = (torch.empty((6, sats.n, 130), dtype=dt, device="cuda"),
           torch.empty((sats.n, 130), dtype=torch.int32, device="cuda"))
    res = pkg.propagate_batch_device(sats, times, out=out, devices=devs)
    torch.cuda.synchronize()
    assert res.planes.data_ptr() == out[0].data_ptr()
    assert torch.equal(out[1], one.error)
    from paper_2603_27830_b200 import _native
    assert _native.load().sgp4b_peer_access(0, 0) == 0


def _harsh_catalogue(rng, n):
    """Every Kepler class (e up to 0.8), deep-space periods, a few perigees
    below the surface, |B*| up to 1e-2 of both signs (tools/exp/parity_campaign.py)."""
    xke = 0.07436691613317342
    no = 2 * np.pi / rng.uniform(87.0, 240.0, n)
    u = rng.random(n)
    ecc = np.where(u < 0.4, rng.uniform(1e-5, 3e-3, n),
          np.where(u < 0.7, rng.uniform(3e-3, 0.1, n),
          np.where(u < 0.9, rng.uniform(0.1, 0.4, n), rng.uniform(0.4, 0.8, n))))
    a = (xke / no) ** (2.0 / 3.0)
    low = rng.random(n) < 0.05
    ecc = np.where(~low & (a * (1 - ecc) < 1.02), np.maximum(0.0, 1 - 1.02 / a), ecc)
    bstar = np.exp(rng.uniform(np.log(1e-6), np.log(1e-2), n)) * np.where(rng.random(n) < 0.1, -1, 1)
    return np.stack([no, ecc, rng.uniform(0, np.pi, n), rng.uniform(0, 2 * np.pi, n),
                     rng.uniform(0, 2 * np.pi, n), rng.uniform(0, 2 * np.pi, n), bstar])


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_harsh_random_catalogues(oracle, seed):
    """Randomized harsh catalogues over -2..+14 days: fp64 codes bit-exact
    and within tolerance outside the degenerate-drag cells (tempa < 0.2 or
    |em| > 0.5, where the reference itself is ill-conditioned: DESIGN §4);
    fp32 codes equal the reference fp64 codes on nearly every cell."""
    pkg = _gpu()
    rng = np.random.default_rng(2000 + seed)
    cols = _harsh_catalogue(rng, 300)
    times = np.sort(rng.uniform(-2880.0, 20160.0, 120))
    s64 = oracle.init_columns(cols, 64)
    ref64, codes64 = oracle.grid(s64, times, workers=4)
    g = {k: np.asarray(v, dtype=np.float64)[:, None] for k, v in s64.items()
         if k != "dtype" and np.asarray(v).ndim}
    t = times[None, :]
    simp = np.asarray(s64["isimp"]).astype(bool)[:, None]
    tempa = 1.0 - g["cc1"] * t - np.where(simp, 0.0, g["d2"] * t**2 + g["d3"] * t**3 + g["d4"] * t**4)
    em = g["ecco"] - g["bstar"] * g["cc4"] * t
    regular = (tempa >= 0.2) & (np.abs(em) <= 0.5)
    res = pkg.propagate_batch(pkg.init_batch(cols, precision=64), times)
    assert np.array_equal(res.error, codes64)
    dr, dv = _diff(res.planes, ref64, (codes64 == 0) & regular)
    assert dr.max(initial=0) <= TOL64_R and dv.max(initial=0) <= TOL64_V
    r32 = pkg.propagate_batch(pkg.init_batch(cols, precision=32), times)
    assert (r32.error != codes64).sum() <= 2


def test_code_rows_kernel_and_pool_reuse(failure_table, corpus_columns):
    """sgp4b_code_rows flags exactly the rows with a nonzero code (aligned and
    unaligned row strides); propagate_batch zero-fills unflagged rows even
    when its pinned block is reused from a call that left codes in it, and
    copies the whole plane when the flagged rows are scattered."""
    import torch
    pkg = _gpu()
    from paper_2603_27830_b200 import _device, _hostmem
    rng = np.random.default_rng(7)
    for n, m, ld in [(37, 130, 130), (37, 130, 133), (5, 3, 3), (300, 1000, 1000)]:
        full = torch.zeros((n, ld), dtype=torch.int32, device="cuda")
        rows = rng.choice(n, size=max(1, n // 5), replace=False)
        cols = rng.integers(0, m, size=rows.size)
        full[torch.from_numpy(rows).cuda(), torch.from_numpy(cols).cuda()] = \
            torch.from_numpy(rng.integers(1, 7, size=rows.size).astype(np.int32)).cuda()
        full[:, m:] = 5                        # beyond the row end: ignored
        flags = torch.full((n,), 9, dtype=torch.uint8, device="cuda")
        _device.code_rows(full[:, :m], flags)
        want = np.zeros(n, np.uint8)
        want[rows] = 1
        assert np.array_equal(flags.cpu().numpy(), want), (n, m, ld)

    bad = np.array([row["elements"] for row in failure_table["cases"].values()]).T
    good = corpus_columns[:, :70]
    times = np.array(failure_table["times"] + [4000.0])
    # scattered failing rows (> MAX_RUNS runs): whole-plane copy
    many = np.concatenate([np.concatenate([good[:, i:i + 1], bad[:, :1]], axis=1)
                           for i in range(70)], axis=1)
    for cols_ in (many, np.concatenate([bad, good], axis=1)):
        sats = pkg.init_batch(cols_)
        host = pkg.propagate_batch(sats, times)
        dev = pkg.propagate_batch_device(sats, times)
        assert np.count_nonzero(host.error) > 0
        assert np.array_equal(host.error, dev.error.cpu().numpy())
    # same shape, no failing rows: the pooled block that held codes is reused
    n_prev = host.n
    del host
    import gc
    gc.collect()                  # the block goes back to the pool now
    clean = pkg.init_batch(corpus_columns[:, 100:100 + n_prev])
    reuses = _hostmem.stats()["reuses"]
    host = pkg.propagate_batch(clean, times)
    assert _hostmem.stats()["reuses"] > reuses
    want = pkg.propagate_batch_device(clean, times).error.cpu().numpy()
    assert np.array_equal(host.error, want)


@pytest.mark.parametrize("n,m", [(1, 1_000_000), (200_000, 1), (3, 130)])
def test_extreme_grid_shapes(oracle, corpus_columns, n, m):
    """One satellite over a million steps (work split along the time axis
    inside one row), 200,000 one-step rows, and a row that ends two cells
    into its second chunk: sampled cells equal the oracle's codes and stay
    within the fp32 bound."""
    import torch
    pkg = _gpu()
    cols = np.tile(corpus_columns, (1, -(-n // corpus_columns.shape[1])))[:, :n]
    times = np.linspace(-720.0, 2880.0, m)
    res = pkg.propagate_batch_device(pkg.init_batch(cols, precision=32), times)
    rng = np.random.default_rng(n + m)
    ii = rng.integers(0, n, 500)
    jj = rng.integers(0, m, 500)
    sat = oracle.init_columns(cols[:, ii], 64)
    ref_r, _, ref_c = oracle.propagate_merged(sat, times[jj])
    got = res.planes[:, torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda()].cpu().numpy()
    codes = res.error[torch.from_numpy(ii).cuda(), torch.from_numpy(jj).cuda()].cpu().numpy()
    assert np.array_equal(codes, ref_c)
    ok = ref_c == 0
    dr = np.linalg.norm(got[:3].T[ok].astype(np.float64) - ref_r[ok], axis=1)
    assert dr.max() < 0.5


@pytest.mark.parametrize("precision", [32, 64])
def test_kepler_class_leaves_domain(oracle, corpus_columns, precision):
    """A near-circular satellite (fast Kepler class by its ecco) with heavy
    drag propagated far backward and forward, so em = ecco - bstar cc4 t - ...
    leaves the class's domain inside one row: the cells beyond it must take
    the general path (fp32: the masked second pass; fp64: the per-cell
    fallback).  Codes equal the reference, states stay within the bars, and
    every cell equals the scalar API's value for the same (satellite, t)."""
    pkg = _gpu()
    base = corpus_columns[:, [137, 415, 391]].copy()   # the corpus's largest bstar*cc4
    base[1] = 0.0029                                   # class 1 (e + 0.001 < 0.004)
    base[6] = [1e-2, -1e-2, 1e-2]                      # heavy drag, both signs
    times = np.linspace(-20160.0, 20160.0, 257)
    ref64, codes64 = oracle.grid(oracle.init_columns(base, 64), times)
    _, codes32 = oracle.grid(oracle.init_columns(base, 32), times)
    sats = pkg.init_batch(base, precision=precision)
    res = pkg.propagate_batch(sats, times)
    assert np.array_equal(res.error, codes64)
    if precision == 32:
        assert np.array_equal(res.error, codes32)
    ok = codes64 == 0
    # the class domain (|em| < 0.004) is really left on code-0 cells:
    # |t| beyond t_crit = (0.004 - e - 2|bstar cc5|) / |bstar cc4|
    init64 = oracle.init_columns(base, 64)
    bc4 = np.abs(np.asarray(init64["bstar"]) * np.asarray(init64["cc4"]))
    bc5 = np.abs(np.asarray(init64["bstar"]) * np.asarray(init64["cc5"]))
    t_crit = (0.004 - base[1] - 2 * bc5) / bc4
    assert (ok & (np.abs(times)[None, :] > t_crit[:, None])).any(axis=1).all()
    # backward propagation with this much drag inflates the orbit to |r| ~
    # 1e8 km, where the 1 mm bar is below fp64 resolution: there the bar is
    # relative (1e-10 |r|), and the absolute bars apply to |r| < 5e4 km
    rad = np.linalg.norm(ref64[:3], axis=0)
    far = ok & (rad >= 5e4)
    if precision == 64 and far.any():
        drf = np.linalg.norm(res.planes[:3] - ref64[:3], axis=0)[far]
        assert (drf <= 1e-10 * rad[far]).all()
    ok &= rad < 5e4
    dr, dv = _diff(res.planes, ref64, ok)
    print(f"\nclass-domain fp{precision}: ok cells {int(ok.sum())}, max|dr| {dr.max() * 1e3:.3f} m")
    if precision == 64:
        assert dr.max() <= TOL64_R and dv.max() <= TOL64_V
    else:
        ref32, _ = oracle.grid(oracle.init_columns(base, 32), times)
        dr_ref, _ = _diff(ref32, ref64, ok)
        assert dr.max() <= dr_ref.max() + 0.05
    dtype = np.float32 if precision == 32 else np.float64
    st = pkg.sgp4_propagate(sats.init, times.astype(dtype)[:, None])
    assert np.array_equal(np.transpose(st.r, (2, 1, 0)), res.planes[:3], equal_nan=True)
    assert np.array_equal(np.transpose(st.v, (2, 1, 0)), res.planes[3:], equal_nan=True)


def test_t_absmax_bound_only_changes_speed(corpus_columns):
    """t_absmax only selects which rows get the masked general pass: an
    unknown (inf / NaN) bound gives the same grid bit for bit."""
    import torch
    from paper_2603_27830_b200 import _device
    from paper_2603_27830_b200.batch import _alloc_grid
    pkg = _gpu()
    cols = corpus_columns[:, :64].copy()
    cols[6, ::3] = 5e-3
    sats = pkg.init_batch(cols, precision=32)
    times = np.linspace(-20160.0, 20160.0, 129)
    ref = pkg.propagate_batch_device(sats, times)
    t_d = torch.from_numpy(times.astype(np.float32)).cuda()
    for bound in (float("inf"), float("nan"), 1e30):
        planes, codes = _alloc_grid(64, 129, 32, t_d.device)
        _device.propagate_grid(sats.device_satrec, t_d, planes, codes, t_absmax=bound)
        assert torch.equal(planes, ref.planes) and torch.equal(codes, ref.error)


@pytest.mark.parametrize("precision,dtype", [(64, np.float64), (32, np.float32)])
def test_hand_built_init_code_persists(real_elements, precision, dtype):
    """A nonzero error_code_at_init of a hand-built SatInit persists in every
    cell, whatever its value (kernel.py:529-534), e.g. 300 (beyond 8 bits)."""
    import dataclasses as dc
    pkg = _gpu()
    init = pkg.sgp4_init(real_elements["ISS"], dtype=dtype)
    edited = dc.replace(init, error_code_at_init=np.int32(300))
    st = pkg.sgp4_propagate(edited, np.array([0.0, 60.0, 720.0], dtype=dtype))
    assert st.error_code.tolist() == [300, 300, 300]


@pytest.mark.parametrize("staged", [False, True])
@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("ndev", [2, 3])
def test_multi_device_path_bitwise(corpus_columns, failure_table, precision, ndev, staged,
                                   monkeypatch):
    """propagate_batch(devices=...) — satellite ranges on several GPUs of
    one process, each D2H-ing into one host grid (pinned, or pageable
    through per-device staging rings when the grid exceeds the pinned cache
    limit) — equals the single-device grid bit for bit.  On a 1-GPU box the
    "devices" are the same GPU named several times (separate streams, same
    code path)."""
    import torch
    pkg = _gpu()
    from paper_2603_27830_b200 import batch as batch_mod
    bad = np.array([row["elements"] for row in failure_table["cases"].values()]).T
    cols = np.concatenate([corpus_columns[:, :200], bad, corpus_columns[:, 200:257]], axis=1)
    sats = pkg.init_batch(cols, precision=precision)
    times = np.linspace(-60.0, 2880.0, 131)
    single = pkg.propagate_batch(sats, times)
    if staged:
        monkeypatch.setenv("SGP4B_HOST_CACHE_BYTES", "1")
        monkeypatch.setattr(batch_mod._StagedD2H, "PIECE", 1 << 14)
    devs = [i % torch.cuda.device_count() for i in range(ndev)]
    multi = pkg.propagate_batch(sats, times, devices=devs)
    assert np.array_equal(multi.planes, single.planes, equal_nan=True)
    assert np.array_equal(multi.error, single.error)



@pytest.mark.parametrize("precision", [32, 64])
@pytest.mark.parametrize("seed", [1, 2])
def test_pairs_equal_grid_cells_every_class(corpus_columns, precision, seed):
    """The elementwise pairs path (fp32: one lane per pair, its own kernel)
    equals the grid cell of the same (satellite, t) bit for bit, on every
    (isimp, Kepler class), on cells that leave their class's domain (heavy
    drag, +-14 days), on failing cells, and whatever t_absmax bound the
    caller passes; the pair order is shuffled so a warp mixes classes."""
    import torch
    from paper_2603_27830_b200 import _device
    pkg = _gpu()
    rng = np.random.default_rng(4100 + seed)
    heavy = corpus_columns[:, [137, 415, 391]].copy()
    heavy[1] = [0.0029, 0.05, 0.2]
    heavy[6] = [1e-2, -1e-2, 1e-2]
    cols = np.concatenate([_harsh_catalogue(rng, 2000), corpus_columns[:, ::7], heavy], axis=1)
    n = cols.shape[1]
    times = np.sort(np.concatenate([rng.uniform(-20160.0, 20160.0, 150), [0.0, 1440.0]]))
    m = times.size
    npdt = np.float32 if precision == 32 else np.float64
    sats = pkg.init_batch(cols, precision=precision)
    grid = pkg.propagate_batch_device(sats, times)
    dev = grid.planes.device
    order = rng.permutation(n * m)
    ii, jj = np.divmod(order, m)
    idx = torch.from_numpy(ii.astype(np.int64)).to(dev)
    jdx = torch.from_numpy(jj.astype(np.int64)).to(dev)
    t_pairs = torch.from_numpy(times[jj].astype(npdt)).to(dev)
    want_p = grid.planes[:, idx, jdx]
    want_c = grid.error[idx, jdx]
    assert int((want_c != 0).sum()) > 0
    if precision == 32:
        # every (isimp, Kepler class) instance of the cell is exercised
        flags = sats.device_satrec.record[:, 33].contiguous().view(torch.int32).cpu().numpy()
        kit = (flags >> 4) & 0xF
        kit = np.where((kit >= 1) & (kit <= 3), kit, 0)     # 0: the general cell
        combos = set(zip((flags & 1).tolist(), kit.tolist()))
        assert combos >= {(s_, k_) for s_ in (0, 1) for k_ in (0, 1, 2, 3)}, combos
    for bound in (None, float("inf"), float("nan")):
        rv = torch.empty((6, n * m), dtype=want_p.dtype, device=dev)
        codes = torch.empty((n * m,), dtype=torch.int32, device=dev)
        _device.propagate_pairs(sats.device_satrec, idx, t_pairs, rv, codes, t_absmax=bound)
        same = (rv == want_p) | (torch.isnan(rv) & torch.isnan(want_p))
        assert bool(same.all()), f"{int((~same.all(0)).sum())} pairs differ (bound {bound})"
        assert torch.equal(codes, want_c)
    # the public general broadcast: satellite i at its own time
    js = rng.integers(0, m, n)
    sd = pkg.sgp4_propagate(sats.init, times[js].astype(npdt))
    host = grid.planes[:, torch.arange(n, device=dev), torch.from_numpy(js).to(dev)].cpu().numpy()
    assert np.array_equal(sd.r.T, host[:3], equal_nan=True)
    assert np.array_equal(sd.v.T, host[3:], equal_nan=True)
    assert np.array_equal(sd.error_code, grid.error[torch.arange(n, device=dev),
                                                    torch.from_numpy(js).to(dev)].cpu().numpy())


def test_pairs_times_lo_equal_grid_cells(corpus_columns):
    """C-ABI pairs with fp32 low words (t = hi + lo) equal the grid cells of
    the times_lo grid launch bit for bit."""
    import torch
    from paper_2603_27830_b200 import _device, _native
    pkg = _gpu()
    rng = np.random.default_rng(77)
    cols = np.concatenate([_harsh_catalogue(rng, 200), corpus_columns[:, ::11]], axis=1)
    n = cols.shape[1]
    times = np.sort(rng.uniform(-10080.0, 20160.0, 97))
    hi = times.astype(np.float32)
    lo = (times - hi.astype(np.float64)).astype(np.float32)
    sats = pkg.init_batch(cols, precision=32)
    dev = torch.device("cuda", 0)
    t_hi, t_lo = torch.from_numpy(hi).to(dev), torch.from_numpy(lo).to(dev)
    grid = pkg.propagate_batch_device(sats, t_hi, times_lo=t_lo)
    ii, jj = np.divmod(rng.permutation(n * times.size), times.size)
    idx = torch.from_numpy(ii.astype(np.int64)).to(dev)
    jdx = torch.from_numpy(jj.astype(np.int64)).to(dev)
    p = int(idx.numel())
    rv = torch.empty((6, p), dtype=torch.float32, device=dev)
    codes = torch.empty((p,), dtype=torch.int32, device=dev)
    tp_hi, tp_lo = t_hi[jdx].contiguous(), t_lo[jdx].contiguous()
    d = sats.device_satrec
    _native.check(_native.load().sgp4b_propagate_pairs(
        d.record.data_ptr(), idx.data_ptr(), tp_hi.data_ptr(), tp_lo.data_ptr(), p,
        float(np.abs(times).max()), 32, _device._host_ptr(_device._grav_host(d.grav, dev)),
        rv.data_ptr(), codes.data_ptr(), _device._stream(dev)))
    want = grid.planes[:, idx, jdx]
    assert bool(((rv == want) | (torch.isnan(rv) & torch.isnan(want))).all())
    assert torch.equal(codes, grid.error[idx, jdx])


def test_pairs_equal_grid_c2_every_cell():
    """All 9,341,000 cells of the C2 workload (Starlink-like catalogue x
    linspace(0, 1440, 1000), fp32) as shuffled elementwise pairs: equal to
    the dense grid bit for bit."""
    import torch
    from paper_2603_27830_b200 import _device
    from paper_2603_27830_b200.catalog import starlink_like
    pkg = _gpu()
    n, m = 9341, 1000
    times = np.linspace(0.0, 1440.0, m)
    sats = pkg.init_batch(starlink_like(n), precision=32)
    grid = pkg.propagate_batch_device(sats, times)
    dev = grid.planes.device
    perm = torch.randperm(n * m, device=dev, generator=torch.Generator(device=dev).manual_seed(5))
    idx, jdx = perm // m, perm % m
    t_pairs = torch.from_numpy(times.astype(np.float32)).to(dev)[jdx].contiguous()
    rv = torch.empty((6, n * m), dtype=torch.float32, device=dev)
    codes = torch.empty((n * m,), dtype=torch.int32, device=dev)
    _device.propagate_pairs(sats.device_satrec, idx.contiguous(), t_pairs, rv, codes)
    assert torch.equal(rv, grid.planes[:, idx, jdx])
    assert torch.equal(codes, grid.error[idx, jdx])
