mkdir -p gpurun_out
python tools/exp/pipes64.py > gpurun_out/pipes64.json 2>&1
bash tools/gpu_variants.sh v64 --precision 64
