"""Event-bracketed time of trivial kernels launched right behind a busy
kernel (the bench protocol's situation): the launch + completion floor."""
import json

import torch

dev = torch.device("cuda", 0)
flush = torch.empty(64 << 20, device=dev)
one = torch.empty(1, device=dev)
big = torch.empty(148 * 512, device=dev)
out = {}
for name, fn in (("fill_1_elem", lambda: one.fill_(1.0)),
                 ("fill_75776_elem", lambda: big.fill_(1.0)),
                 ("two_back_to_back_fills", lambda: (one.fill_(1.0), one.fill_(2.0)))):
    ts = []
    for k in range(30):
        flush.fill_(k)
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    ts.sort()
    out[name + "_us_median"] = round(ts[len(ts) // 2], 2)
print(json.dumps(out, indent=1))
