mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:grid_kernel -s 3 -c 1 -f -o gpurun_out/prof_c3_s1 python bench.py --precision 64 --steps 2 --warmup 3 --no-cpu --no-accuracy --e2e-steps 1 > gpurun_out/ncu_full64.log 2>&1
ls -la gpurun_out | head
