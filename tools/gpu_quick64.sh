#!/bin/bash
# fp64 iteration: GPU tests, C3 bench, ncu of the fp64 grid kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu -x -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --precision 64 --no-cpu --steps 100 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 3 -c 1 -f -o gpurun_out/prof_c3_fp64 python bench.py --precision 64 --steps 2 --warmup 3 --no-cpu --no-accuracy --e2e-steps 1 > gpurun_out/ncu_full64.log 2>&1
ls -la gpurun_out
