"""Init kernel time (C2 catalogue, fp32 records, columns in HBM) for each
library given on the command line (SGP4B_LIBRARY per subprocess)."""
import json
import os
import subprocess
import sys

CODE = r'''
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
from paper_2603_27830_b200 import _device
from paper_2603_27830_b200.catalog import starlink_like
from paper_2603_27830_b200.gravity import WGS72
dev = torch.device("cuda", 0)
el = torch.from_numpy(starlink_like(9341)).to(dev)
ts = []
for k in range(40):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    torch.cuda._sleep(400000)        # GPU busy while the host queues the launch
    a.record()
    d = _device.init_device_tensor(el, WGS72, 32, dev)
    b.record()
    torch.cuda.synchronize()
    if k >= 5:
        ts.append(a.elapsed_time(b) * 1e3)
ref = d.codes.cpu().numpy().copy(), d.record.cpu().numpy().copy()
print(json.dumps({"init_us_median": round(float(np.median(ts)), 2), "init_us_min": round(float(min(ts)), 2),
                  "codes_sum": int(ref[0].sum()), "rec_hash": float(np.nansum(ref[1].astype(np.float64)))}))
'''
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if len(sys.argv) == 1:                  # in-process (under ncu): current SGP4B_LIBRARY
    exec(CODE % root)
for so in sys.argv[1:]:
    env = dict(os.environ, SGP4B_LIBRARY=os.path.abspath(so))
    out = subprocess.run([sys.executable, "-c", CODE % root], env=env, capture_output=True, text=True)
    print(so, out.stdout.strip() or out.stderr[-500:])
