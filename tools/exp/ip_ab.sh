# A/B of the init kernel satellites-per-warp variants (built by tools/build_variants.sh with -DSGP4B_INIT_PER_WARP=32/16/8; the macro was not kept)
set -x
cd $GRAFT_REPO_ROOT
L=paper_2603_27830_b200
for r in 1 2; do
python tools/exp/init_variants.py $L/libsgp4b_ip32.so $L/libsgp4b_ip16.so $L/libsgp4b_ip8.so
done > gpurun_out/ip_init.txt 2>&1
for r in 1 2; do for v in ip32 ip16 ip8; do
SGP4B_LIBRARY=$PWD/$L/libsgp4b_$v.so python bench.py --no-cpu --no-accuracy --e2e-steps 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', d['ms_per_step']*1e3, d['init_plus_propagate']['ms_per_step']*1e3)"
done; done > gpurun_out/ip_bench.txt 2>&1
cat gpurun_out/ip_init.txt gpurun_out/ip_bench.txt
