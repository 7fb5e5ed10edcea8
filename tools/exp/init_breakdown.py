"""init_batch host-side cost split: column copy, H2D (pageable vs pinned),
kernel launch + sync."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg                              # noqa: E402
from paper_2603_27830_b200 import _device                        # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like          # noqa: E402
from paper_2603_27830_b200.gravity import WGS72                  # noqa: E402

dev = torch.device("cuda", 0)
cols = starlink_like(9341)
R = 50
def avg(fn):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(R):
        fn()
        torch.cuda.synchronize()
    return round((time.perf_counter() - t0) / R * 1e6, 1)
el_dev = torch.from_numpy(cols).to(dev)
out = {
    "np_copy_us": avg(lambda: np.array(cols, dtype=np.float64, order="C")),
    "h2d_pageable_us": avg(lambda: torch.from_numpy(cols).to(dev)),
    "h2d_pinned_us": avg(lambda: torch.from_numpy(cols).pin_memory().to(dev, non_blocking=True)),
    "init_device_tensor_us": avg(lambda: _device.init_device_tensor(el_dev, WGS72, 32, dev)),
    "init_batch_us": avg(lambda: pkg.init_batch(cols, precision=32)),
}
print(json.dumps(out, indent=1))
