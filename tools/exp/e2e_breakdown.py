"""Where the C2 end-to-end time goes (host columns in, numpy grid out)."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg                              # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like          # noqa: E402

cols = starlink_like(9341)
times = np.linspace(0.0, 1440.0, 1000)
for _ in range(3):
    pkg.propagate_batch(pkg.init_batch(cols, precision=32), times)
torch.cuda.synchronize()
acc = {}
R = 20
for _ in range(R):
    t0 = time.perf_counter()
    sats = pkg.init_batch(cols, precision=32)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    res = pkg.propagate_batch(sats, times)
    t2 = time.perf_counter()
    _ = int(res.error[-1, -1])
    t3 = time.perf_counter()
    for k, v in (("init_batch", t1 - t0), ("propagate_batch", t2 - t1), ("read", t3 - t2)):
        acc[k] = acc.get(k, 0.0) + v / R
    del res
print(json.dumps({k: round(v * 1e3, 3) for k, v in acc.items()}, indent=1))

# raw DMA floors into the same kind of pinned block
from paper_2603_27830_b200 import _hostmem                         # noqa: E402
dev = torch.device("cuda")
for label, nbytes in (("planes_224MB", 6 * 9341 * 1000 * 4), ("grid_261MB", 7 * 9341 * 1000 * 4)):
    src = torch.empty(nbytes // 4, dtype=torch.float32, device=dev)
    dst = torch.from_numpy(np.asarray(_hostmem.alloc(nbytes))[:nbytes].view(np.float32))
    for _ in range(3):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / R
    print(f"{label}: {dt * 1e3:.3f} ms = {nbytes / dt / 1e9:.1f} GB/s")
