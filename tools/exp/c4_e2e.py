"""C4 (100k x 1440 fp32) propagate_batch wall time vs the raw planes D2H."""
import json, os, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200 import _hostmem
from paper_2603_27830_b200.catalog import starlink_like
sats = pkg.init_batch(starlink_like(100_000), precision=32)
times = np.arange(1440, dtype=np.float64)
for _ in range(3):
    r = pkg.propagate_batch(sats, times); del r
ts = []
for _ in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    r = pkg.propagate_batch(sats, times); x = int(r.error[-1, -1]); ts.append(time.perf_counter() - t0); del r
nb = 6 * 100_000 * 1440 * 4
src = torch.empty(nb // 4, device="cuda"); dst = torch.from_numpy(np.asarray(_hostmem.alloc(nb))[:nb].view(np.float32))
dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
t0 = time.perf_counter(); dst.copy_(src, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t0
print(json.dumps({"threads": os.environ.get("SGP4B_HOST_THREADS", "default"),
                  "propagate_batch_ms": [round(t * 1e3, 1) for t in ts], "planes_d2h_ms": round(d2h * 1e3, 1)}))
