"""Init kernel time vs catalogue size (fp32 records), element columns in HBM."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_2603_27830_b200 import _device                       # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like         # noqa: E402
from paper_2603_27830_b200.gravity import WGS72                 # noqa: E402

dev = torch.device("cuda", 0)
out = {}
for n in (9341, 100000, 1000000):
    el = torch.from_numpy(starlink_like(n)).to(dev)
    ts = []
    for k in range(8):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        _device.init_device_tensor(el, WGS72, 32, dev)
        b.record()
        torch.cuda.synchronize()
        if k >= 2:
            ts.append(a.elapsed_time(b) * 1e3)
    out[n] = round(float(np.median(ts)), 1)
print(json.dumps({"init_us_by_n": out}, indent=1))
