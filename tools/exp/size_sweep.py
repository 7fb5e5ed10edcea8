"""Grid-kernel time vs catalogue size at 1,000 steps (fp32), L2 flushed
before each launch: the intercept of the linear fit is the fixed per-launch
cost (launch, ramp, drain), the slope the steady per-row cost."""
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
out = {}
for n in (296, 1184, 2368, 4736, 9341, 18682, 37364, 74728):
    sats = init_batch(starlink_like(n), precision=32, device=dev)
    planes = torch.empty((6, n, 1000), device=dev)
    codes = torch.empty((n, 1000), dtype=torch.int32, device=dev)
    ts = []
    for k in range(25):
        flush.fill_(k)
        torch.sum(rd, 0, out=sink)
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        _device.propagate_grid(sats.device_satrec, times, planes, codes, t_absmax=1440.0)
        b.record()
        torch.cuda.synchronize()
        if k >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    out[n] = round(float(np.median(ts)), 2)
ns = np.array(list(out.keys()), float)
us = np.array(list(out.values()))
sel = ns >= 2368
slope, icpt = np.polyfit(ns[sel], us[sel], 1)
print(json.dumps({"us_by_n": out, "fit_us_per_1k_rows": slope * 1e3, "fit_intercept_us": icpt}, indent=1))
