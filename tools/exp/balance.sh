mkdir -p gpurun_out; : > gpurun_out/balance.txt
for v in 0 1 0 1; do
  SGP4B_BALANCE=$v timeout 120 python tools/exp/balance.py 9341 32 300 >> gpurun_out/balance.txt 2>&1
done
SGP4B_BALANCE=0 timeout 120 python tools/exp/balance.py 9341 64 200 >> gpurun_out/balance.txt 2>&1
SGP4B_BALANCE=1 timeout 120 python tools/exp/balance.py 9341 64 200 >> gpurun_out/balance.txt 2>&1
SGP4B_BALANCE=0 timeout 120 python tools/exp/balance.py 30000 32 200 >> gpurun_out/balance.txt 2>&1
SGP4B_BALANCE=1 timeout 120 python tools/exp/balance.py 30000 32 200 >> gpurun_out/balance.txt 2>&1
SGP4B_BALANCE=0 timeout 200 python bench.py --no-cpu --steps 200 --no-graph 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/balance.txt
SGP4B_BALANCE=1 timeout 200 python bench.py --no-cpu --steps 200 --no-graph 2>/dev/null | tail -1 | cut -c1-200 >> gpurun_out/balance.txt
cat gpurun_out/balance.txt
