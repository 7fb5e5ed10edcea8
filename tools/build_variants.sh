#!/bin/bash
# Build libsgp4b_<name>.so variants in parallel for tools/variants.sh:
#   tools/build_variants.sh "name:-DFLAG=1 -DOTHER=2" ...
cd "$(dirname "$0")/.."
for v in "$@"; do
  name=${v%%:*}; flags=${v#*:}
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
      $flags -I include -o paper_2603_27830_b200/libsgp4b_$name.so paper_2603_27830_b200/csrc/sgp4b.cu \
      -Xptxas -v 2>&1 | grep -A2 "Compiling entry.*grid_kernelIfLb1ELb0" | grep -E "registers|spill" \
      | tr -s ' \n' ' ' | sed "s/^/$name: /"; echo ) &
done
wait
