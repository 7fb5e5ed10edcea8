#!/bin/bash
# Build the microbenchmark libraries used by tools/exp/*.py (sm_100a).
cd "$(dirname "$0")"
for f in pipes store_ceiling; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Xcompiler -fPIC -shared -o $f.so $f.cu || exit 1
done
