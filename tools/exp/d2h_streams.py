"""D2H rate of a 224 MB grid into pinned memory with 1, 2 and 4 concurrent
copy streams (copy engines), and chunk sizes."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_27830_b200 import _hostmem
nb = 6 * 9341 * 1000 * 4
src = torch.empty(nb // 4, dtype=torch.float32, device="cuda")
dst = torch.from_numpy(np.asarray(_hostmem.alloc(nb))[:nb].view(np.float32))
out = {}
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    per = (nb // 4) // ns
    def once():
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                lo = i * per; hi = (nb // 4) if i == ns - 1 else lo + per
                dst[lo:hi].copy_(src[lo:hi], non_blocking=True)
        for s in streams:
            s.synchronize()
    for _ in range(3):
        once()
    t0 = time.perf_counter()
    for _ in range(10):
        once()
    dt = (time.perf_counter() - t0) / 10
    out[f"streams_{ns}"] = {"ms": round(dt * 1e3, 3), "GBs": round(nb / dt / 1e9, 1)}
print(json.dumps(out))
