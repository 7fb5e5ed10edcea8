"""Grid-kernel time for a C2-sized grid (9,341 x 1,000 fp32) per catalogue
mix: Starlink-like (Kepler class 1), the reference's LEO corpus tiled
(mostly class 2, some isimp), and class-2-only eccentricities."""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from paper_2603_27830_b200 import _device, init_batch             # noqa: E402
from paper_2603_27830_b200.catalog import starlink_like           # noqa: E402
from paper_2603_27830_b200.tle import parse_catalog_columns       # noqa: E402

lines = [ln for ln in (ROOT / "tests/golden/leo_corpus.tle").read_text().splitlines() if ln]
corpus = parse_catalog_columns(lines[0::2], lines[1::2])
n, m = 9341, 1000
mixes = {"starlink_class1": starlink_like(n),
         "leo_corpus_tiled": np.tile(corpus, (1, -(-n // corpus.shape[1])))[:, :n]}
c2 = starlink_like(n).copy()
c2[1] = np.random.default_rng(3).uniform(0.005, 0.09, n)
mixes["class2_e_0.005_0.09"] = c2
dev = torch.device("cuda", 0)
t = torch.from_numpy(np.linspace(0.0, 1440.0, m).astype(np.float32)).to(dev)
planes = torch.empty((6, n, m), device=dev)
codes = torch.empty((n, m), dtype=torch.int32, device=dev)
flush = torch.empty(64 << 20, device=dev)
rd = torch.ones(64 << 20, device=dev)
sink = torch.empty((), device=dev)
out = {}
for name, cols in mixes.items():
    sats = init_batch(cols, precision=32, device=dev)
    ts = []
    for k in range(30):
        flush.fill_(k)
        torch.sum(rd, 0, out=sink)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); _device.propagate_grid(sats.device_satrec, t, planes, codes); b.record()
        torch.cuda.synchronize()
        if k >= 5:
            ts.append(a.elapsed_time(b) * 1e3)
    out[name] = round(float(np.median(ts)), 2)
print(json.dumps({"us": out}, indent=1))
