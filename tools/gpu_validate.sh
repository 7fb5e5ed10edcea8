mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -s > gpurun_out/pytest_gpu_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu_full.log
SGP4B_LIBRARY=$PWD/build/pairs/lane.so timeout 200 python tools/exp/pairs_time.py > gpurun_out/pairs_lane.txt 2>&1
tail -3 gpurun_out/pytest_gpu_full.log; grep -E "passed|failed|Error" gpurun_out/pytest_gpu_full.log | tail -5; cat gpurun_out/pairs_lane.txt
