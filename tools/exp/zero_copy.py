"""Grid kernel writing the planes straight into pinned host memory over
PCIe (zero-copy, UVA) vs HBM + one D2H: C2 fp32."""
import json, sys, time
from pathlib import Path
import numpy as np, torch
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_2603_27830_b200 as pkg
from paper_2603_27830_b200 import _device, _hostmem, _native
from paper_2603_27830_b200.catalog import starlink_like

cols = starlink_like(9341); times = np.linspace(0, 1440, 1000)
n, m = cols.shape[1], times.size
sats = pkg.init_batch(cols, precision=32)
dev = sats.device_satrec
t_d = torch.from_numpy(times.astype(np.float32)).cuda()
planes_h, codes_h = _hostmem.empty([((6, n, m), np.float32), ((n, m), np.int32)])
codes_d = torch.empty((n, m), dtype=torch.int32, device="cuda")
planes_d = torch.empty((6, n, m), dtype=torch.float32, device="cuda")
g = _device._grav_host(dev.grav, dev.device)
lib = _native.load()
s = torch.cuda.current_stream().cuda_stream

def zero_copy():
    _native.check(lib.sgp4b_propagate_grid(dev.record.data_ptr(), n, t_d.data_ptr(), None, m, 1440.0,
                                           32, g.ctypes.data, planes_h.ctypes.data, n * m, m,
                                           codes_d.data_ptr(), m, s))

def hbm_then_d2h():
    _native.check(lib.sgp4b_propagate_grid(dev.record.data_ptr(), n, t_d.data_ptr(), None, m, 1440.0,
                                           32, g.ctypes.data, planes_d.data_ptr(), n * m, m,
                                           codes_d.data_ptr(), m, s))
    torch.from_numpy(planes_h).copy_(planes_d, non_blocking=True)

out = {}
for name, fn in (("zero_copy", zero_copy), ("hbm_then_d2h", hbm_then_d2h)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(10):
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
    out[name] = {"ms_median": round(float(np.median(ts)), 3), "GBs": round(planes_h.nbytes / np.median(ts) / 1e6, 1)}
# the zero-copy planes equal the HBM ones
zero_copy(); torch.cuda.synchronize(); zc = planes_h.copy()
hbm_then_d2h(); torch.cuda.synchronize()
out["bitwise_equal"] = bool(np.array_equal(zc.view(np.uint32), planes_h.view(np.uint32)))
print(json.dumps(out))
