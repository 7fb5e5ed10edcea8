#!/bin/bash
# C3 (fp64) bench of every prebuilt libsgp4b_*.so variant, with the accuracy check
mkdir -p gpurun_out
: > gpurun_out/variants64.txt
for lib in paper_2603_27830_b200/libsgp4b_*.so; do
  SGP4B_LIBRARY=$PWD/$lib timeout 300 python bench.py --precision 64 --no-cpu --e2e-steps 1 --steps 100 $BENCH_ARGS 2>>gpurun_out/variants64.err | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); a=d.get('accuracy',{})
print('$lib', round(d['ms_per_step']*1e3,2),'us min',round(d['kernel_ms_min']*1e3,2),'frac',round(d['roofline']['frac'],4),'dr',a.get('dr_max_km'),'dv',a.get('dv_max_kms'),'codes',a.get('code_mismatch_vs_ref_fp64'))" >> gpurun_out/variants64.txt 2>&1
done
cat gpurun_out/variants64.txt
