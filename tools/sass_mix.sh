#!/bin/bash
# Static SASS instruction mix of the fp32 grid kernel's (non-isimp, Kepler KCLASS=1|2)
# chunk loop, per cell: builds an analysis cubin where every row runs that
# instance, then counts the loop body's instructions by opcode.
#   tools/sass_mix.sh [extra nvcc flags]
set -e
out=${TMPDIR:-/tmp}/sgp4b_mix
mkdir -p $out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -DSGP4B_ONLY_CLASS_K1=${KCLASS:-1} "$@" \
  -I include -cubin -o $out/k1.cubin paper_2603_27830_b200/csrc/sgp4b.cu -Xptxas -v 2>&1 \
  | grep -A2 "grid_kernelIfLb1ELb0" | grep -E "registers|spill"
cuobjdump -sass $out/k1.cubin | awk '/Function : .*grid_kernelIfLb1ELb0/{f=1} f&&/Function : /&&!/grid_kernelIfLb1ELb0/{f=0} f' > $out/k1.sass
python3 tools/sass_loop_mix.py $out/k1.sass
