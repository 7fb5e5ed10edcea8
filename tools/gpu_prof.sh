#!/bin/bash
# ncu captures for one round: full set of the fp32 and fp64 grid kernels and
# the init kernel (one launch each), plus the C2 launch list.
#   tools/gpu_prof.sh <tag>
tag=${1:-r02}
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu --no-accuracy --e2e-steps 1"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 3 -c 1 -f \
  -o gpurun_out/${tag}_c2_grid $B > gpurun_out/${tag}_ncu_c2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 3 -c 1 -f \
  -o gpurun_out/${tag}_c3_grid $B --precision 64 > gpurun_out/${tag}_ncu_c3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:init_kernel -s 1 -c 1 -f \
  -o gpurun_out/${tag}_c2_init $B > gpurun_out/${tag}_ncu_init.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/${tag}_launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu --e2e-steps 1 \
  > gpurun_out/${tag}_launches_c2.log 2>&1
ls -la gpurun_out
