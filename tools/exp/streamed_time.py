"""propagate_batch_streamed throughput (C4-like 100k x 1440 fp32) for a few
tile shapes, against propagate_batch (whole grid) and the D2H floor."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200.catalog import starlink_like

cols = starlink_like(100_000); times = np.arange(1440, dtype=np.float64)
sats = pkg.init_batch(cols, precision=32)
out = {}
def sink(rows, cols_, planes, err):
    pass
for tr, tc in ((10_000, 1440), (2_000, 1440), (100_000, 144)):
    pkg.propagate_batch_streamed(sats, times, tr, tc, sink)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    s = pkg.propagate_batch_streamed(sats, times, tr, tc, sink)
    dt = time.perf_counter() - t0
    out[f"streamed_{tr}x{tc}_ms"] = round(dt * 1e3, 1)
for _ in range(2):
    r = pkg.propagate_batch(sats, times); del r
torch.cuda.synchronize(); t0 = time.perf_counter()
r = pkg.propagate_batch(sats, times); x = int(r.error[-1, -1])
out["propagate_batch_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
out["grid_bytes"] = 100_000 * 1440 * 28
print(json.dumps(out, indent=1))
