"""Wall time of the first, second and third propagate_batch call for a few
grid sizes (pinning policy: _hostmem.worth_pinning)."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200.catalog import starlink_like
out = {}
for n, m, prec in ((9341, 1000, 32), (9341, 1000, 64), (100_000, 1440, 32)):
    sats = pkg.init_batch(starlink_like(n), precision=prec)
    times = np.linspace(0, 1440, m)
    ts = []
    for k in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = pkg.propagate_batch(sats, times); x = int(r.error[-1, -1])
        ts.append(round((time.perf_counter() - t0) * 1e3, 1))
        del r
    out[f"{n}x{m}_fp{prec}_ms"] = ts
print(json.dumps(out))
