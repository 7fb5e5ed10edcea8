#!/usr/bin/env python
"""Benchmark: SGP4 batch propagation throughput (satellite-timestep
propagations/s) on B200, with the reference CPU path timed beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload c2|c3|c4|c5] [--precision 32|64]

Default workload is BASELINE.json's headline, C2: Starlink-like 9,341 sats x
1,000 steps (linspace(0, 1440, 1000) min) at fp32 on one GPU.  Under
torchrun each rank propagates its own 9,341-satellite shard (weak scaling, no
collective on the data path; one all-reduce(MAX) of the timings only).

One step = one launch of the grid kernel over the whole (N_shard x M) grid,
inputs (packed satrec + times) resident in HBM, L2 flushed (256 MiB write,
then a 256 MiB read so no dirty flush lines are left) before every timed launch; timed with CUDA events on the launching stream.
``e2e`` is the same metric through the public API with host buffers:
init_batch(host element columns) + propagate_batch(host times) -> numpy
grid in pinned host memory, H2D and D2H inside the timed region.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "satellite-timestep propagations/sec, Starlink 9,341×1,000 fp32; latency ms"
UNIT = "props/s"
PAPER_A100_PROPS = 9341 * 1000 / 3.8e-3          # PAPER.md:99, 3.8 ms on A100

WORKLOADS = {
    # name: (description, sats per rank, times, default precision)
    "c1": ("C1 ISS 1 sat x 1,000 steps (linspace 0..1440 min) fp64", 1,
           lambda: np.linspace(0.0, 1440.0, 1000), 64),
    "c2": ("C2 Starlink-like 9,341 sats x 1,000 steps (linspace 0..1440 min)", 9341,
           lambda: np.linspace(0.0, 1440.0, 1000), 32),
    "c3": ("C3 Starlink-like 9,341 sats x 1,000 steps fp64", 9341,
           lambda: np.linspace(0.0, 1440.0, 1000), 64),
    "c4": ("C4 100,000 sats x 1,440 steps (1-min over 1 day)", 100000,
           lambda: np.arange(1440.0), 32),
    "c5": ("C5 1,000,000 sats x 1,000 steps (125,000 per GPU at 8 GPUs)", 1000000,
           lambda: np.linspace(0.0, 1440.0, 1000), 32),
}

BYTES_PER_CELL = {32: 28, 64: 52}      # 6 planes x itemsize + int32 code
FLOPS_PER_CELL = 235                   # reference _propagate op count


def _peaks() -> dict:
    path = ROOT / "MEASURED_PEAKS.json"
    if path.exists():
        d = json.loads(path.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0, "source": "fallback (B200_PROFILING.md)"}


class ClockSampler:
    """SM clock + throttle reasons sampled while the timed region runs.

    NVML is polled every ~2 ms from a thread (nvidia-smi's 100 ms loop would
    see a few-ms timed region once at best); ``region(True/False)`` brackets
    the timed launches and the summary covers the samples taken inside it.
    Falls back to ``nvidia-smi -lms 100`` when NVML is unavailable."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
                ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
                ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
                ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
                ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, int, bool]] = []    # (sm MHz, reason bits, in region)
        self.in_region = False
        self.stop = threading.Event()
        self.nvml = None
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.handle = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(self.handle, pynvml.NVML_CLOCK_SM))
            self._t = threading.Thread(target=self._poll, daemon=True)
            self._t.start()
        except Exception:
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self._t = threading.Thread(target=self._read, daemon=True)
                self._t.start()
            except (OSError, FileNotFoundError):
                self.proc = None
        return self

    def region(self, inside: bool) -> None:
        self.in_region = inside

    def _poll(self):
        nv = self.nvml
        while not self.stop.is_set():
            try:
                mhz = float(nv.nvmlDeviceGetClockInfo(self.handle, nv.NVML_CLOCK_SM))
                bits = int(nv.nvmlDeviceGetCurrentClocksEventReasons(self.handle))
                self.samples.append((mhz, bits, self.in_region))
            except Exception:
                pass
            time.sleep(0.002)

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None:
            self._t.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        if self.nvml is not None:
            inside = [x for x in self.samples if x[2]]
            use = inside or self.samples
            if not use:
                return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
            reasons = sorted({name for _, bits, _ in use for name, attr in self.REASONS
                              if bits & int(getattr(self.nvml, attr, 0))})
            return {"sm_mhz": statistics.median(x[0] for x in use), "sm_max_mhz": self.max_mhz,
                    "reasons": reasons, "samples": len(use),
                    "source": "nvml, 2 ms polling, " + ("timed region" if inside else "whole run")}
        rows = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) != 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        busy = [r for r in rows if r[2] > 0] or rows
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for r in busy for i, v in enumerate(r[3]) if v.lower() == "active"})
        return {"sm_mhz": statistics.median(r[0] for r in busy), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(busy), "source": "nvidia-smi -lms 100"}


def time_task_cpu(task, min_trial_s: float = 0.2, trials: int = 5) -> float:
    """The reference's timing protocol (pkg/src/sgp4kit/bench.py:48-82):
    one warm-up, double iterations until a trial exceeds 0.2 s, min of 5."""
    task()
    it = 1
    while True:
        t0 = time.perf_counter()
        for _ in range(it):
            task()
        if time.perf_counter() - t0 > min_trial_s:
            best = math.inf
            for _ in range(trials):
                t0 = time.perf_counter()
                for _ in range(it):
                    task()
                best = min(best, time.perf_counter() - t0)
            if best > min_trial_s:
                return best / it
        it *= 2


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(cols: np.ndarray, times: np.ndarray, precision: int, max_rows: int) -> dict:
    """The reference CPU path (oracle/ port, bit-exact with sgp4kit) on a
    bounded sample of the same workload, all host threads."""
    from oracle import sgp4_oracle as oracle
    workers = oracle.default_workers()
    rows = min(cols.shape[1], max_rows)
    sub = cols[:, :rows]
    sat = oracle.init_columns(sub, precision)
    per = time_task_cpu(lambda: oracle.grid(sat, times, workers=workers))
    cells = rows * times.size
    return {"value": cells / per, "unit": UNIT, "cores": workers, "kind": "port",
            "sample": f"{rows} sats x {times.size} steps fp{precision}, propagate-only, "
                      f"reference time_task protocol (min of 5), numpy {np.__version__}, "
                      f"{cpu_model()}",
            "ms_per_run": per * 1e3}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def run_reference(args, world, rank) -> None:
    """--impl reference: the reference CPU implementation of the path (the
    oracle port, bit-exact with sgp4kit) on the host cores, rank 0 only."""
    if rank != 0:
        return
    from oracle import sgp4_oracle as oracle
    from paper_2603_27830_b200.catalog import starlink_like
    desc, nsat, tfn, default_prec = WORKLOADS[args.workload]
    precision = args.precision or default_prec
    times = tfn()
    # bounded sample: ~2e9 cells over the whole --steps/--warmup run (about a
    # minute on 16 host threads), at most the workload's own catalogue
    budget_rows = int(2.0e9 / max(1, args.steps + args.warmup) / times.size)
    rows = max(1, min(nsat, args.ref_rows, budget_rows))
    if args.workload == "c1":
        from paper_2603_27830_b200.catalog import iss_columns
        cols = iss_columns()
    else:
        cols = starlink_like(rows)
    workers = oracle.default_workers()

    def step():
        sat = oracle.init_columns(cols, precision)
        oracle.grid(sat, times, workers=workers)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = rows * times.size / dt
    sample = (f"{rows} of {nsat} sats x {times.size} steps fp{precision} per step "
              f"(init + propagate), {workers} threads, {cpu_model()}")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": f"f{precision}", "data": "synthetic",
        "config": {"workload": desc, "n_sats": rows, "n_steps": int(times.size)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": workers, "kind": "port",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


def run_ours(args, world, rank, local) -> None:
    import torch
    import torch.distributed as dist

    from paper_2603_27830_b200 import _device, init_batch, propagate_batch
    from paper_2603_27830_b200.batch import propagate_batch_device
    from paper_2603_27830_b200.catalog import SEED, starlink_like

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device")
    # one process per GPU; SGP4B_BENCH_BACKEND=gloo (test only) lets several
    # ranks share a GPU to exercise the multi-rank plumbing on a 1-GPU box
    backend = os.environ.get("SGP4B_BENCH_BACKEND", "nccl")
    gpu = local % torch.cuda.device_count() if backend != "nccl" else local
    torch.cuda.set_device(gpu)
    device = torch.device("cuda", gpu)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group(backend)

    desc, nsat, tfn, default_prec = WORKLOADS[args.workload]
    precision = args.precision or default_prec
    times = tfn()
    m = times.size
    if args.workload == "c1":                # one satellite: ranks split the time axis
        from paper_2603_27830_b200.catalog import iss_columns
        from paper_2603_27830_b200.shard import shard_plan
        cols = iss_columns()
        _, lo, hi = shard_plan(1, times.size, world, rank)
        times = times[lo:hi] if world > 1 else times
        m = times.size
        scaling = "strong"
    elif args.workload in ("c4", "c5"):      # fixed total, sharded (strong scaling)
        lo = nsat * rank // world
        hi = nsat * (rank + 1) // world
        cols = starlink_like(nsat)[:, lo:hi]
        scaling = "strong"
    else:                                    # per-rank Starlink shard (weak scaling)
        cols = starlink_like(nsat, seed=SEED + rank)
        scaling = "weak"
    n = cols.shape[1]
    cells = n * m

    stream = torch.cuda.current_stream(device)
    sats = init_batch(cols, precision=precision, device=device)
    t_dev = torch.from_numpy(times.astype(np.float32 if precision == 32 else np.float64)).to(device)
    planes, error = _device_alloc(n, m, precision, device)
    # L2 flush between timed launches: write a 256 MiB buffer (evicts every
    # line), then read another 256 MiB one so the flush's own dirty lines are
    # written back here, outside the timed region, instead of being evicted
    # by (and billed to) the timed kernel's output stream
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    flush_r = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=device)
    sink = torch.empty((), dtype=torch.float32, device=device)

    def flush_l2(k):
        flush.fill_(float(k))
        torch.sum(flush_r, 0, out=sink)


    def launch():
        _device.propagate_grid(sats.device_satrec, t_dev, planes, error)

    # the timed step replays a CUDA graph holding the grid-kernel launch (the
    # same kernel and arguments; the graph trims the per-launch CPU->GPU
    # submission cost, as a serving loop would); --no-graph launches directly
    step = launch
    if not args.no_graph:
        side = torch.cuda.Stream(device)
        side.wait_stream(stream)
        with torch.cuda.stream(side):
            launch()
        stream.wait_stream(side)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            launch()
        step = graph.replay

    sampler = ClockSampler(gpu)
    sampler.__enter__()
    for _ in range(max(args.warmup, 3)):
        flush_l2(0)
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()

    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    region0 = torch.cuda.Event(enable_timing=True)
    region1 = torch.cuda.Event(enable_timing=True)
    sampler.region(True)
    region0.record(stream)
    for k in range(args.steps):
        flush_l2(k)                             # L2 flush, outside the kernel's events
        starts[k].record(stream)
        step()
        ends[k].record(stream)
    region1.record(stream)
    torch.cuda.synchronize()
    sampler.region(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    kernel_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    total_ms = sum(kernel_ms)
    t = torch.tensor([total_ms], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms_max = float(t.item())
    ms_per_step = total_ms_max / args.steps
    value = cells * world / (ms_per_step * 1e-3)

    # ---- paper convention: init + propagate, element
    # columns resident in HBM, same flush + event protocol -----------------
    from paper_2603_27830_b200.gravity import WGS72
    el_dev = torch.from_numpy(np.ascontiguousarray(cols, dtype=np.float64)).to(device)

    def init_and_launch():
        d = _device.init_device_tensor(el_dev, WGS72, precision, device)
        _device.propagate_grid(d, t_dev, planes, error)

    ip_ms = []
    for k in range(max(3, min(args.steps, 10)) + 2):
        flush_l2(k)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        init_and_launch()
        b.record(stream)
        torch.cuda.synchronize()
        if k >= 2:
            ip_ms.append(a.elapsed_time(b))
    ip = torch.tensor([statistics.median(ip_ms)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(ip, op=dist.ReduceOp.MAX)
    init_prop_ms = float(ip.item())

    # ---- e2e: public API with host buffers --------------------------------
    e2e_steps = max(1, min(args.steps, args.e2e_steps))
    host_times = times.copy()
    for _ in range(2):
        res = propagate_batch(init_batch(cols, precision=precision, device=device), host_times)
        del res
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    res = None
    for _ in range(e2e_steps):
        del res
        res = propagate_batch(init_batch(cols, precision=precision, device=device), host_times)
        checksum = int(res.error[-1, -1])       # host read of the result
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    # bytes that crossed PCIe per step (counted outside the timed region):
    # the planes, one flag per row, and the code rows holding a nonzero code
    d2h_bytes = (res.planes.nbytes + n + int(np.count_nonzero(res.error.any(axis=1))) * m * 4)
    del res
    te = torch.tensor([e2e_s], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_s = float(te.item())
    sampler.__exit__(None, None, None)
    clocks = sampler.summary()

    if rank == 0:
        peaks = _peaks()
        bpc = BYTES_PER_CELL[precision]
        achieved_gbs = cells * bpc / (ms_per_step * 1e-3) / 1e9
        traffic = _traffic(args.workload, precision)
        flop_peak, flop_src = _flop_peak(precision, peaks)
        t_hbm = cells * bpc / (peaks["hbm_gbs"] * 1e9)
        t_flop = cells * FLOPS_PER_CELL / flop_peak
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": scaling,
            "vs_baseline": (value / PAPER_A100_PROPS) if (args.workload == "c2" and precision == 32
                                                          and world == 1) else None,
            "dtype": f"f{precision}", "data": "synthetic",
            "config": {
                "workload": desc, "n_sats_per_gpu": n, "n_steps": m, "cells_per_gpu": cells,
                "parallelism": f"satellite shards x{world}, no collective",
                "l2": "flushed before every timed launch (256 MiB write, then 256 MiB read so "
                      "no dirty flush lines remain); outputs "
                      f"{cells * bpc / 2**20:.0f} MiB > L2",
                "vs_baseline_ref": "paper A100 3.8 ms for C2 fp32 (PAPER.md:99) = 2.458e9 props/s",
                "launch": "direct" if args.no_graph else "CUDA graph replay of the grid-kernel launch",
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved_gbs, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved_gbs / peaks["hbm_gbs"], "traffic": traffic,
                "peak_source": peaks["source"],
                "algorithmic_bytes_per_cell": bpc,
                "t_hbm_us": t_hbm * 1e6, "t_flop_us": t_flop * 1e6,
                "flops_per_cell": FLOPS_PER_CELL,
                "flop_peak_tflops": flop_peak / 1e12, "flop_peak_source": flop_src,
                "frac_of_roofline": max(t_hbm, t_flop) / (ms_per_step * 1e-3),
            },
            "e2e": {"value": cells * world / e2e_s, "unit": UNIT,
                    "ms_per_step": e2e_s * 1e3,
                    "h2d_bytes_per_step": 7 * n * 8 + m * (4 if precision == 32 else 8),
                    "d2h_bytes_per_step": d2h_bytes,
                    "api": "propagate_batch(init_batch(host columns), host times) -> numpy "
                           "(planes via pinned memory; code rows cross PCIe only where nonzero)"},
            "init_plus_propagate": {"ms_per_step": init_prop_ms,
                                    "value": cells * world / (init_prop_ms * 1e-3),
                                    "note": "paper convention (PAPER.md:67-71): init kernel + "
                                            "grid kernel, element columns in HBM, L2 flushed"},
            "gpu_launches": args.steps,
            "clocks": clocks,
            "kernel_ms_min": min(kernel_ms), "kernel_ms_median": statistics.median(kernel_ms),
        }
        if world == 1 and not args.no_cpu:
            line["cpu_baseline"] = cpu_baseline(cols, times, precision, args.cpu_rows)
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


def _device_alloc(n, m, precision, device):
    import torch
    dt = torch.float32 if precision == 32 else torch.float64
    return (torch.empty((6, n, m), dtype=dt, device=device),
            torch.empty((n, m), dtype=torch.int32, device=device))


def _flop_peak(precision: int, peaks: dict):
    """FP32/FP64 FMA peak: the FMA microbenchmark (profiles/r01_pipes.json,
    tools/exp/pipes.py) when present, else 148 SM x lanes x 2 x max clock."""
    path = ROOT / "profiles" / "r01_pipes.json"
    key = "fp32_ffma2_tflops" if precision == 32 else "fp64_dfma_tflops"
    if path.exists():
        d = json.loads(path.read_text())
        if key in d:
            return float(d[key]) * 1e12, "measured (profiles/r01_pipes.json)"
    lanes = 128 if precision == 32 else 64
    return 148 * lanes * 2 * peaks["sm_max_mhz"] * 1e6, "derived (148 SM x lanes x 2 x max clock)"


def _traffic(workload: str, precision: int):
    """dram read+write bytes per launch from the committed ncu --set full
    capture (profiles/ncu_traffic.json), or None."""
    path = ROOT / "profiles" / "ncu_traffic.json"
    if not path.exists():
        return None
    d = json.loads(path.read_text())
    return d.get(f"{workload}_fp{precision}")


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="c2")
    ap.add_argument("--precision", type=int, choices=(32, 64), default=None)
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--cpu-rows", type=int, default=9341)
    ap.add_argument("--ref-rows", type=int, default=9341)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true",
                    help="launch the timed grid kernels directly instead of replaying a CUDA graph")
    args = ap.parse_args()
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)


if __name__ == "__main__":
    main()
