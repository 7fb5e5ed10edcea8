"""Elementwise sgp4_propagate (one time per satellite): device time of the
pairs launch and the end-to-end call, vs the same cells as a dense grid row."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200 import _device
from paper_2603_27830_b200.catalog import starlink_like
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 32
npdt = np.float32 if prec == 32 else np.float64
out = {"precision": prec}
for n in (10_000, 1_000_000):
    cols = starlink_like(n)
    sats = pkg.init_batch(cols, precision=prec)
    init = sats.init
    t = np.random.default_rng(1).uniform(0, 1440, n).astype(npdt)
    pkg.sgp4_propagate(init, t)
    torch.cuda.synchronize()
    e2e = []
    for _ in range(7):
        t0 = time.perf_counter(); s = pkg.sgp4_propagate(init, t); e2e.append(time.perf_counter() - t0)
    dev = sats.device_satrec
    idx = torch.arange(n, device="cuda"); td = torch.from_numpy(t).cuda()
    rv = torch.empty((6, n), device="cuda", dtype=torch.float32 if prec == 32 else torch.float64); c = torch.empty(n, dtype=torch.int32, device="cuda")
    tb = float(np.abs(t).max())      # explicit bound: no device reduction inside the events
    for _ in range(3):
        _device.propagate_pairs(dev, idx, td, rv, c, t_absmax=tb)
    torch.cuda.synchronize()
    ks = []
    for _ in range(20):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _device.propagate_pairs(dev, idx, td, rv, c, t_absmax=tb); b.record()
        torch.cuda.synchronize()
        ks.append(a.elapsed_time(b) * 1e3)
    out[n] = {"e2e_ms_median": round(float(np.median(e2e)) * 1e3, 2),
              "e2e_ms_all": [round(x * 1e3, 2) for x in e2e],
              "pairs_kernel_us_median": round(float(np.median(ks)), 1)}
print(json.dumps(out))
