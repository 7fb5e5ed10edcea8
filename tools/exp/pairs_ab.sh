# A/B of the elementwise pairs path: one-step grid rows (rows.so, built with
# -DSGP4B_PAIRS_LANE=0) against the lane-per-pair kernels (lane.so)
mkdir -p gpurun_out
for prec in 32 64; do for v in rows lane; do echo "== $v fp$prec"; SGP4B_LIBRARY=$PWD/build/pairs/$v.so timeout 200 python tools/exp/pairs_time.py $prec; done; done > gpurun_out/pairs_ab.txt 2>&1
timeout 600 python -m pytest tests -q -m gpu -p no:cacheprovider -k "pairs or scalar or randomized or kepler_class or hand_built or batch_equals or ref" > gpurun_out/pytest_pairs.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_pairs.log
tail -3 gpurun_out/pytest_pairs.log; cat gpurun_out/pairs_ab.txt
