"""Event-bracketed C2 grid-kernel time launched directly vs replayed from a
CUDA graph, L2 flushed before each launch (bench.py protocol)."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_27830_b200 import _device, init_batch            # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like          # noqa: E402

dev = torch.device("cuda", 0)
n, m = 9341, 1000
sats = init_batch(starlink_like(n), precision=32, device=dev)
t = torch.from_numpy(np.linspace(0.0, 1440.0, m).astype(np.float32)).to(dev)
planes = torch.empty((6, n, m), device=dev)
codes = torch.empty((n, m), dtype=torch.int32, device=dev)
flush = torch.empty(64 << 20, device=dev)
rd = torch.ones(64 << 20, device=dev)
sink = torch.empty((), device=dev)

def launch():
    _device.propagate_grid(sats.device_satrec, t, planes, codes, t_absmax=1440.0)

s = torch.cuda.Stream()
s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    launch()
torch.cuda.current_stream().wait_stream(s)
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    launch()
ref_p = planes.clone()

def timed(fn, reps=60):
    ts = []
    for k in range(reps):
        flush.fill_(k)
        torch.sum(rd, 0, out=sink)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        if k >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    return round(float(np.median(ts)), 2), round(float(np.min(ts)), 2)

out = {"direct_us": timed(launch), "graph_us": timed(g.replay)}
planes.zero_(); g.replay(); torch.cuda.synchronize()
out["graph_output_equal"] = bool(torch.equal(planes, ref_p))
print(json.dumps(out, indent=1))
