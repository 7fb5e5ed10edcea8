mkdir -p gpurun_out
bash tools/gpu_variants.sh v64 --precision 64 > /dev/null
cp gpurun_out/variants.txt gpurun_out/variants64.txt
bash tools/gpu_variants.sh v64 > /dev/null
cp gpurun_out/variants.txt gpurun_out/variants32.txt
timeout 1500 python -m pytest tests -q -m gpu -s -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
