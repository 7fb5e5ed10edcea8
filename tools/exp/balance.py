"""Successive direct C2 grid launches (L2 flushed between them): event time
per launch, to see whether the SM-speed balancing converges.  Run with
SGP4B_BALANCE=0 / unset to compare."""
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2603_27830_b200 import _device, init_batch   # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like  # noqa: E402

dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 9341
prec = int(sys.argv[2]) if len(sys.argv) > 2 else 32
launches = int(sys.argv[3]) if len(sys.argv) > 3 else 300
dt = torch.float32 if prec == 32 else torch.float64
times = torch.from_numpy(np.linspace(0.0, 1440.0, 1000)).to(dev, dt)
sats = init_batch(starlink_like(n), precision=prec, device=dev)
planes = torch.empty((6, n, 1000), device=dev, dtype=dt)
codes = torch.empty((n, 1000), dtype=torch.int32, device=dev)
flush = torch.empty(64 << 20, device=dev)
out = []
for k in range(launches):
    flush.fill_(k)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    _device.propagate_grid(sats.device_satrec, times, planes, codes, t_absmax=1440.0)
    b.record()
    torch.cuda.synchronize()
    out.append(a.elapsed_time(b) * 1e3)
o = np.array(out)
print(json.dumps({"balance": os.environ.get("SGP4B_BALANCE", "on"), "n": n, "prec": prec,
                  "first10": [round(x, 1) for x in o[:10]],
                  "median_10_50": round(float(np.median(o[10:50])), 2),
                  "median_last100": round(float(np.median(o[-100:])), 2),
                  "min": round(float(o.min()), 2), "p90_last100": round(float(np.percentile(o[-100:], 90)), 2)}))
