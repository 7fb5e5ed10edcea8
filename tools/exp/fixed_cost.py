"""Decompose the grid kernel's fixed per-launch cost: event-bracketed time of
an empty torch kernel, and of the grid kernel at a tiny and the C2 size with
and without an L2 flush before the launch."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_27830_b200 import _device, init_batch            # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like          # noqa: E402

dev = torch.device("cuda", 0)
times = torch.from_numpy(np.linspace(0.0, 1440.0, 1000).astype(np.float32)).to(dev)
flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)
rd = torch.ones(64 << 20, dtype=torch.float32, device=dev)
sink = torch.empty((), device=dev)
tiny = torch.empty(1, device=dev)


def t_of(fn, do_flush):
    ts = []
    for k in range(30):
        if do_flush:
            flush.fill_(k)
            torch.sum(rd, 0, out=sink)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        if k >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    return round(float(np.median(ts)), 2)


out = {"empty_fill_us": t_of(lambda: tiny.fill_(1.0), False)}
for n in (296, 9341):
    sats = init_batch(starlink_like(n), precision=32, device=dev)
    planes = torch.empty((6, n, 1000), device=dev)
    codes = torch.empty((n, 1000), dtype=torch.int32, device=dev)
    fn = lambda: _device.propagate_grid(sats.device_satrec, times, planes, codes, t_absmax=1440.0)
    out[f"n{n}_flushed_us"] = t_of(fn, True)
    out[f"n{n}_warm_us"] = t_of(fn, False)
    # 1 step only: 1 chunk per row
    t1 = times[:128].clone()
    p1 = torch.empty((6, n, 128), device=dev)
    c1 = torch.empty((n, 128), dtype=torch.int32, device=dev)
    fn1 = lambda: _device.propagate_grid(sats.device_satrec, t1, p1, c1, t_absmax=1440.0)
    out[f"n{n}_m128_flushed_us"] = t_of(fn1, True)
    out[f"n{n}_m128_warm_us"] = t_of(fn1, False)
print(json.dumps(out, indent=1))
