import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200.catalog import starlink_like
for n in (1_000_000,):
    cols = starlink_like(n); times = np.linspace(0, 1440, 1000)
    for k in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        res = pkg.propagate_batch(pkg.init_batch(cols, precision=32), times)
        x = int(res.error[-1, -1]); t1 = time.perf_counter()
        print(n, k, round(t1 - t0, 3), 's', res.planes.nbytes / (t1 - t0) / 1e9, 'GB/s', flush=True)
        del res
