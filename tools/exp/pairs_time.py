"""Elementwise sgp4_propagate (one time per satellite): device time of the
pairs launch and the end-to-end call, vs the same cells as a dense grid row."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200 import _device
from paper_2603_27830_b200.catalog import starlink_like
out = {}
for n in (10_000, 1_000_000):
    cols = starlink_like(n)
    sats = pkg.init_batch(cols, precision=32)
    init = sats.init
    t = np.random.default_rng(1).uniform(0, 1440, n).astype(np.float32)
    pkg.sgp4_propagate(init, t)
    torch.cuda.synchronize()
    t0 = time.perf_counter(); s = pkg.sgp4_propagate(init, t); t1 = time.perf_counter()
    dev = sats.device_satrec
    idx = torch.arange(n, device="cuda"); td = torch.from_numpy(t).cuda()
    rv = torch.empty((6, n), device="cuda"); c = torch.empty(n, dtype=torch.int32, device="cuda")
    for _ in range(3):
        _device.propagate_pairs(dev, idx, td, rv, c)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); _device.propagate_pairs(dev, idx, td, rv, c); b.record(); torch.cuda.synchronize()
    out[n] = {"e2e_ms": round((t1 - t0) * 1e3, 2), "pairs_kernel_us": round(a.elapsed_time(b) * 1e3, 1)}
print(json.dumps(out))
