#!/bin/bash
# ncu duration of init_kernel (C2 catalogue) for each library argument
mkdir -p gpurun_out
for so in "$@"; do
  SGP4B_LIBRARY=$PWD/$so timeout 300 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:init_kernel -c 12 --csv \
    python tools/exp/init_variants.py > /tmp/ncu_iv.csv 2>/dev/null
  python - "$so" <<'PY'
import csv, sys, statistics
rows = [r for r in csv.reader(l for l in open('/tmp/ncu_iv.csv') if l.startswith('"'))]
h = rows[0]; d = rows[1:]
t = [float(r[h.index('Metric Value')].replace(',', '')) for r in d if r[h.index('Metric Name')] == 'gpu__time_duration.sum']
i = [float(r[h.index('Metric Value')].replace(',', '')) for r in d if r[h.index('Metric Name')] == 'smsp__inst_executed.sum']
print(sys.argv[1], 'init_kernel us median', statistics.median(t) / 1e3 if t else None, 'min', min(t) / 1e3 if t else None, 'inst', i[:1])
PY
done
