"""Per-warp timeline of one C2 launch (SGP4B_TIMELINE build): when warps
start, finish their first row and exit, relative to the earliest start."""
import ctypes
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
os.environ["SGP4B_LIBRARY"] = str(ROOT / "paper_2603_27830_b200" / "libsgp4b_TL.so")
from paper_2603_27830_b200 import _device, _native, init_batch   # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like           # noqa: E402

lib = _native.load()
fn = lib.sgp4b_debug_timeline
fn.argtypes = [ctypes.c_void_p, ctypes.c_int]
dev = torch.device("cuda", 0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 9341
times = torch.from_numpy(np.linspace(0.0, 1440.0, 1000).astype(np.float32)).to(dev)
sats = init_batch(starlink_like(n), precision=32, device=dev)
planes = torch.empty((6, n, 1000), device=dev)
codes = torch.empty((n, 1000), dtype=torch.int32, device=dev)
flush = torch.empty(64 << 20, device=dev)
for k in range(4):
    flush.fill_(k)
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    _device.propagate_grid(sats.device_satrec, times, planes, codes, t_absmax=1440.0)
    b.record()
    torch.cuda.synchronize()
warps = 148 * 16
buf = np.zeros((warps, 4), dtype=np.uint64)
assert fn(buf.ctypes.data, warps) == 0
t0 = buf[:, 0].min()
st = (buf[:, 0] - t0) / 1e3
fr = (buf[:, 1] - t0) / 1e3
en = (buf[:, 2] - t0) / 1e3
q = lambda x: [round(float(v), 2) for v in np.percentile(x, [0, 10, 50, 90, 100])]
print(json.dumps({"event_us": a.elapsed_time(b) * 1e3, "start_us_pct": q(st),
                  "first_row_done_us_pct": q(fr), "end_us_pct": q(en),
                  "sms": int(np.unique(buf[:, 3]).size)}, indent=1))
np.save(str(ROOT / "gpurun_out" / f"timeline_{n}.npy"), buf)
