mkdir -p gpurun_out
for v in rows lane; do echo "== $v"; SGP4B_LIBRARY=$PWD/build/pairs/$v.so timeout 200 python tools/exp/pairs_time.py; done > gpurun_out/pairs_ab.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum -k regex:pairs_kernel --clock-control none -c 3 python tools/exp/pairs_time.py > gpurun_out/pairs_ncu.txt 2>&1
cat gpurun_out/pairs_ab.txt; grep -E "pairs_kernel32|duration|warps_active|inst_executed|dram" gpurun_out/pairs_ncu.txt | head -20
