import cProfile, pstats, sys, time, io
import numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200 import _hostmem
from paper_2603_27830_b200.catalog import starlink_like
cols = starlink_like(9341); times = np.linspace(0, 1440, 1000)
hc, ht = _hostmem.empty([(cols.shape, np.float64), (times.shape, np.float32)]); hc[...] = cols; ht[...] = times
for _ in range(5):
    r = pkg.propagate_batch(pkg.init_batch(hc, precision=32), ht); del r
torch.cuda.synchronize()
pr = cProfile.Profile()
t0 = time.perf_counter()
pr.enable()
for _ in range(20):
    r = pkg.propagate_batch(pkg.init_batch(hc, precision=32), ht); x = int(r.error[-1, -1]); del r
pr.disable()
print("per step ms", (time.perf_counter() - t0) / 20 * 1e3)
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(18); print(s.getvalue()[:4000])
