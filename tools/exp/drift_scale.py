"""drift_report at catalogue scale on the GPU: wall
time and the paper's Fig. 3 statistic (fp32 vs fp64 median drift)."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg                              # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like          # noqa: E402
from paper_2603_27830_b200.tle import MeanElements               # noqa: E402

out = {}
for n in (9341, 100000):
    cols = starlink_like(n)
    els = [MeanElements(*cols[:, i], 2026, 13, 0.0) for i in range(n)]
    pkg.drift_report(els[:64], horizon_days=1.0, step_minutes=90.0)      # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rep = pkg.drift_report(els, horizon_days=14.0, step_minutes=90.0)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    out[n] = {"seconds": round(dt, 3), "steps": int(rep.days.size),
              "epoch_median_m": round(float(rep.p50_km[0]) * 1e3, 3),
              "day14_median_m": round(float(rep.p50_km[-1]) * 1e3, 3),
              "day14_p95_m": round(float(rep.p95_km[-1]) * 1e3, 3)}
print(json.dumps(out, indent=1))
