"""Device->host bandwidth into pinned memory: one copy vs several
concurrent chunks on separate streams (the e2e path's D2H is ~4.8 ms)."""
import json
import time

import torch

dev = torch.device("cuda", 0)
n = 261_548_000 // 4
src = torch.ones(n, device=dev)
dst = torch.empty(n, pin_memory=True)
out = {}
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    chunks_s = src.chunk(k)
    chunks_d = dst.chunk(k)
    best = 1e9
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for s, a, b in zip(streams, chunks_s, chunks_d):
            with torch.cuda.stream(s):
                b.copy_(a, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    out[f"streams{k}_ms"] = round(best * 1e3, 3)
    out[f"streams{k}_gbs"] = round(src.numel() * 4 / best / 1e9, 1)
h2d = torch.empty(n, device=dev)
best = 1e9
for _ in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    h2d.copy_(dst, non_blocking=True); torch.cuda.synchronize()
    best = min(best, time.perf_counter() - t0)
out["h2d_gbs"] = round(n * 4 / best / 1e9, 1)
print(json.dumps(out, indent=1))
