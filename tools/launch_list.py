"""Compact an ncu launch list (--metrics gpu__time_duration.sum --csv
--log-file) into kernel,grid,block,duration_ns rows plus per-kernel totals
and the grid kernel's share of the device time.
    python tools/launch_list.py gpurun_out/launches_c2.csv profiles/rNN_launches_c2_fp32.csv"""
import collections
import csv
import sys

src, dst = sys.argv[1], sys.argv[2]
lines = [ln for ln in open(src) if ln.startswith('"')]
rows = list(csv.DictReader(lines))
out = []
tot = collections.defaultdict(float)
for r in rows:
    if r["Metric Name"] != "gpu__time_duration.sum":
        continue
    ns = float(r["Metric Value"].replace(",", ""))
    name = r["Kernel Name"]
    out.append((name[:80], r["Grid Size"], r["Block Size"], int(ns)))
    short = name.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    tot[short] += ns
with open(dst, "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "grid", "block", "duration_ns"])
    w.writerows(out)
    all_ns = sum(tot.values())
    w.writerow([])
    w.writerow(["# kernel (template args elided)", "launches", "total_ns", "share_of_device_time"])
    counts = collections.Counter(n.split("(")[0].replace("void ", "").replace("<unnamed>::", "")
                                 for n, *_ in ((r["Kernel Name"],) for r in rows
                                               if r["Metric Name"] == "gpu__time_duration.sum"))
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        w.writerow([k, counts[k], int(v), f"{v / all_ns:.3f}"])
print(open(dst).read()[-900:])
