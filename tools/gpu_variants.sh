#!/bin/bash
# Bench every build/<dir>/*.so variant on one workload (SGP4B_LIBRARY swaps
# the library), then the GPU tests against the in-tree library.
#   tools/gpu_variants.sh <dir> <bench args...>
dir=$1; shift
mkdir -p gpurun_out
: > gpurun_out/variants.txt
for so in build/$dir/*.so; do
  echo "== $so" >> gpurun_out/variants.txt
  SGP4B_LIBRARY=$PWD/$so timeout 300 python bench.py --no-cpu --steps 100 "$@" 2>>gpurun_out/variants.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
a=d.get('accuracy',{})
print(round(d['ms_per_step']*1e3,2),'us frac',round(d['roofline']['frac'],4),'ip',round(d['init_plus_propagate']['ms_per_step']*1e3,2),'dr',a.get('dr_max_km'),'dv',a.get('dv_max_kms'),'codes',a.get('code_mismatch_vs_ref_fp64'))" >> gpurun_out/variants.txt 2>&1
done
if [ -n "$RUN_TESTS" ]; then
  timeout 1500 python -m pytest tests -q -m gpu -s -p no:cacheprovider $RUN_TESTS > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
cat gpurun_out/variants.txt
