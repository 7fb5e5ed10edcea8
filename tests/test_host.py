"""Host-side logic that needs no GPU: scheduling helpers, the SGB1 binary
format, gravity constants and API validation (mirrors pkg/tests/test_batch.py
TestPartitionWork / TestTileGrid / TestBinaryFormat and gravity.py)."""

import io
import math

import numpy as np
import pytest

from paper_2603_27830_b200 import (
    WGS72,
    BatchResult,
    ErrorCode,
    epoch_to_julian,
    init_batch,
    partition_work,
    read_grid_binary,
    write_grid_binary,
)
from paper_2603_27830_b200.batch import _tile_grid


@pytest.mark.parametrize("n", range(1, 9))
@pytest.mark.parametrize("m", range(1, 9))
@pytest.mark.parametrize("workers", [1, 2, 3, 5, 8])
def test_partition_work_disjoint_covering_balanced(n, m, workers):
    ranges = partition_work(n, m, workers)
    assert ranges[0][0] == 0 and ranges[-1][1] == n * m
    for (a0, a1), (b0, b1) in zip(ranges, ranges[1:]):
        assert a1 == b0 and a1 > a0
    sizes = [b - a for a, b in ranges]
    assert max(sizes) - min(sizes) <= 1
    assert len(ranges) == min(workers, n * m)


def test_partition_work_rejects_zero_workers():
    with pytest.raises(ValueError):
        partition_work(4, 4, 0)


def test_tile_grid_covers_exactly():
    mask = np.zeros((10, 7), dtype=int)
    for rows, cols in _tile_grid(10, 7, 4, 3):
        mask[rows, cols] += 1
    assert (mask == 1).all()


def _fake_result(precision, n=3, m=5, seed=0):
    rng = np.random.default_rng(seed)
    dt = np.float32 if precision == 32 else np.float64
    planes = rng.normal(size=(6, n, m)).astype(dt)
    error = rng.integers(0, 7, size=(n, m)).astype(np.int32)
    return BatchResult(planes=planes, error=error, n=n, m=m)


@pytest.mark.parametrize("precision", [32, 64])
def test_sgb1_round_trip(precision):
    res = _fake_result(precision)
    buf = io.BytesIO()
    write_grid_binary(res, buf)
    buf.seek(0)
    back = read_grid_binary(buf)
    assert back.n == res.n and back.m == res.m
    assert back.planes.dtype == res.planes.dtype
    assert np.array_equal(back.planes, res.planes) and np.array_equal(back.error, res.error)


def test_sgb1_header_layout():
    res = _fake_result(32, n=2, m=3)
    buf = io.BytesIO()
    write_grid_binary(res, buf)
    raw = buf.getvalue()
    assert raw[:4] == b"SGB1"
    assert int.from_bytes(raw[4:12], "little") == 2
    assert int.from_bytes(raw[12:20], "little") == 3
    assert int.from_bytes(raw[20:24], "little") == 32
    assert raw[24:32] == b"rrrvvve\x00"
    assert len(raw) == 32 + 6 * 2 * 3 * 4 + 2 * 3 * 4
    with pytest.raises(ValueError):
        read_grid_binary(io.BytesIO(b"NOPE" + b"\0" * 28))


def test_wgs72_constants():
    # gravity.py:31-47 of the reference, and the SURVEY §8(a) value of xke
    assert WGS72.mu == 398600.8 and WGS72.radius_earth_km == 6378.135
    assert WGS72.xke == pytest.approx(0.07436691613317342, rel=1e-15)
    assert WGS72.xke == 60.0 / math.sqrt(6378.135 * 6378.135 * 6378.135 / 398600.8)
    assert WGS72.tumin == 1.0 / WGS72.xke
    assert WGS72.j3oj2 == WGS72.j3 / WGS72.j2
    assert WGS72.as_array().shape == (8,)


def test_error_code_values():
    assert [int(c) for c in ErrorCode] == [0, 1, 2, 3, 4, 6, 7]


def test_epoch_to_julian():
    assert epoch_to_julian(2000, 1, 0.5) == 2451545.0
    assert epoch_to_julian(1970, 1, 0.0) == 2440587.5
    assert epoch_to_julian(2020, 366, 0.0) == epoch_to_julian(2021, 1, 0.0) - 1.0
    with pytest.raises(ValueError):
        epoch_to_julian(2021, 366, 0.0)


def test_init_batch_validates_before_touching_the_gpu():
    with pytest.raises(ValueError):
        init_batch([])
    with pytest.raises(ValueError):
        init_batch(np.zeros((7, 0)))
    with pytest.raises(ValueError):
        init_batch(np.zeros((6, 3)))
    with pytest.raises(ValueError):
        init_batch(np.zeros((7, 3)), precision=16)


def test_bench_reference_arm_contract():
    """`bench.py --impl reference` (the reference CPU path on the host cores)
    prints one JSON line with the driver's keys, on a bounded sample."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-rows", "64"],
                         capture_output=True, text=True, timeout=300, cwd=root)
    assert out.returncode == 0, out.stderr
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "dtype", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_bench_reference_arm_nonzero_rank_is_silent():
    """Under torchrun only rank 0 runs the reference arm; other ranks exit 0
    without output."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-rows", "8"],
                         capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode == 0 and out.stdout.strip() == ""


def test_bench_world_size_must_match_gpus():
    """Under a torchrun environment --gpus must equal WORLD_SIZE (a silent
    1-GPU measurement of an N-GPU request is refused)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, RANK="0", WORLD_SIZE="2", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0", "--ref-rows", "8"],
                         capture_output=True, text=True, timeout=300, cwd=root, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_bench_gpus_flag_relaunches_under_torchrun():
    """`bench.py --gpus 2` without torchrun re-executes itself under
    torch.distributed.run with 2 ranks; the reference arm prints one line
    (rank 0) whose config is the same dict the GPU arm prints."""
    import json
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root))
    import bench
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    out = subprocess.run([sys.executable, str(root / "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1", "--warmup", "0", "--ref-rows", "16"],
                         capture_output=True, text=True, timeout=600, cwd=root, env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["impl"] == "reference"
    desc, cols, times, prec, scaling = bench.workload_shape("c2", 2, 0)
    assert d["config"] == bench.bench_config("c2", desc, cols.shape[1], times.size, prec, 2, scaling)
    assert d["cpu_baseline"]["numpy"] and d["cpu_baseline"]["cpu_model"]


def test_time_task_protocol_and_failures():
    """The reference timing protocol (bench.py:48-82): warm-up, doubling
    until the fastest of five trials clears 0.2 s, min per iteration."""
    import time as _t
    from paper_2603_27830_b200 import BenchRecord, TaskFailed, time_task
    calls = []

    def task():
        calls.append(1)
        _t.sleep(0.03)
    rec = time_task(task, label="sleep", n=3, m=4, precision=32)
    assert isinstance(rec, BenchRecord) and rec.trials == 5 and rec.total_cells == 12
    assert rec.iterations & (rec.iterations - 1) == 0            # a power of two
    assert rec.iterations * rec.min_time_s > 0.2
    assert 0.03 <= rec.min_time_s < 0.06
    assert rec.throughput_cells_per_s == 12 / rec.min_time_s

    state = {"k": 0}

    def flaky():
        state["k"] += 1
        if state["k"] == 3:
            raise KeyError("boom")
    with pytest.raises(TaskFailed) as ei:
        time_task(flaky)
    assert ei.value.trial_index == 0 and isinstance(ei.value.__cause__, KeyError)

    def broken():
        raise ValueError("warm-up")
    with pytest.raises(ValueError):                               # warm-up is not wrapped
        time_task(broken)


def test_scaling_sweep_validation():
    from paper_2603_27830_b200 import scaling_sweep
    with pytest.raises(ValueError):
        scaling_sweep("cells", [1, 2], 10, [])
    with pytest.raises(ValueError):
        scaling_sweep("times", [4, 2], 10, [])
    with pytest.raises(ValueError):
        scaling_sweep("times", [2, 2], 10, [])


def test_pack_rejects_init_codes_the_record_cannot_hold():
    """A hand-built SatInit's error_code_at_init travels in the packed
    record's 23-bit code field: codes outside [0, 2^23) are refused before
    any GPU work instead of wrapping to a different (or zero) code."""
    import pytest as _pytest
    from paper_2603_27830_b200 import _device
    from paper_2603_27830_b200.gravity import WGS72
    sr = np.zeros((33, 2))
    for bad in ([-1, 0], [0, 1 << 23]):
        with _pytest.raises(ValueError, match="error_code_at_init"):
            _device.pack_device(sr, np.array(bad), np.zeros(2, np.uint8), WGS72, 64)


# ---- host logic of the transfer and ingest paths (no GPU) -----------------

def test_flag_runs():
    from paper_2603_27830_b200.batch import flag_runs
    f = np.zeros(20, np.uint8)
    assert flag_runs(f, 64) == []
    f[[2, 3, 4, 9, 19]] = 1
    assert flag_runs(f, 64) == [(2, 5), (9, 10), (19, 20)]
    assert flag_runs(f, 2) == [(0, 20)]                      # too many runs
    g = np.ones(20, np.uint8)
    g[:9] = 0
    assert flag_runs(g, 64) == [(0, 20)]                     # more than half flagged
    one = np.array([1], np.uint8)
    assert flag_runs(one, 64) == [(0, 1)]


def test_ingest_host_lines_follow_read_tle_file(tmp_path):
    """The host path of read_catalog_columns pairs lines exactly as
    read_tle_file does (universal newlines, blank and name lines skipped,
    the same 'line 2 missing' error)."""
    from paper_2603_27830_b200.ingest import _as_bytes, _host_lines
    from paper_2603_27830_b200.tle import TleError, read_tle_file
    a = "1 25544U 98067A   24001.50000000  .00016717  00000-0  10270-3 0  9990"
    b = "2 25544  51.6416 247.4627 0006703 130.5360 325.0288 15.49815367 12345"
    for text in (f"ISS\n{a}\n{b}\n", f"{a}\r\n{b}\r\n", f"\n\n{a}\n   \n{b}", f"{a}\r{b}\r",
                 f"X\n{b}\n{a}\n{b}\n"):
        path = tmp_path / "c.tle"
        path.write_bytes(text.encode())
        l1, l2 = _host_lines(_as_bytes(path))
        recs = read_tle_file(path)
        assert len(l1) == len(recs) == 1 and l1[0].rstrip() == a and l2[0].rstrip() == b
    with pytest.raises(TleError, match="line 2 missing"):
        _host_lines(_as_bytes(f"{a}\n{a}\n{b}\n".encode()))
    assert _as_bytes(b"xy").flags.writeable


def test_pinned_pool_keeps_recent_blocks(monkeypatch):
    """The pinned pool (with a fake allocator, no GPU) caches the most
    recently released blocks under its limit, evicting the oldest first, so
    a large grid requested call after call stays cached after smaller tiles
    filled the pool; a block larger than the limit is never cached."""
    import ctypes
    import gc
    from paper_2603_27830_b200 import _hostmem
    libc = ctypes.CDLL(None)
    libc.malloc.restype = ctypes.c_void_p
    libc.malloc.argtypes = [ctypes.c_size_t]
    libc.free.argtypes = [ctypes.c_void_p]
    live = {}

    class FakeLib:
        def sgp4b_host_alloc(self, size, out):
            p = libc.malloc(size)
            live[p] = size
            ctypes.cast(out, ctypes.POINTER(ctypes.c_void_p))[0] = p
            return 0

        def sgp4b_host_free(self, p):
            libc.free(live.pop(p) and p)
            return 0

        def sgp4b_last_error(self):
            return b""

    monkeypatch.setattr(_hostmem._native, "load", lambda: FakeLib())
    _hostmem._free.clear()
    _hostmem._released.clear()
    monkeypatch.setitem(_hostmem._stats, "cached_bytes", 0)
    monkeypatch.setitem(_hostmem._stats, "pinned_bytes", 0)
    mb = 1 << 20
    monkeypatch.setenv("SGP4B_HOST_CACHE_BYTES", str(20 * mb))
    tiles = [_hostmem.alloc(4 * mb) for _ in range(4)]          # 16 MiB of tiles
    del tiles
    gc.collect()
    assert _hostmem.stats()["cached_bytes"] == 16 * mb
    big = _hostmem.alloc(12 * mb)
    del big
    gc.collect()
    st = _hostmem.stats()                                      # oldest tiles evicted
    assert st["cached_bytes"] <= 20 * mb and any(b[0] == 12 * mb for b in _hostmem._free)
    reuses = st["reuses"]
    again = _hostmem.alloc(12 * mb)
    assert _hostmem.stats()["reuses"] == reuses + 1
    del again
    huge = _hostmem.alloc(30 * mb)                              # above the limit
    del huge
    gc.collect()
    assert all(b[0] != 30 * mb for b in _hostmem._free)
    _hostmem.empty_cache()
    assert not live
