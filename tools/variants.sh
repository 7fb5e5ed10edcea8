#!/bin/bash
# time the grid kernel for each prebuilt library variant (BENCH_ARGS adds bench flags)
mkdir -p gpurun_out
for lib in paper_2603_27830_b200/libsgp4b*.so; do
  r=$(SGP4B_LIBRARY=$PWD/$lib timeout 300 python bench.py --no-cpu --e2e-steps 1 --steps 50 $BENCH_ARGS 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step']*1e3, d['kernel_ms_min']*1e3, d['roofline']['frac'])")
  echo "$lib $BENCH_ARGS us_per_step,min_us,frac = $r" >> gpurun_out/variants.txt
done
