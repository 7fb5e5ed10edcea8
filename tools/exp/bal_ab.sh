# A/B of the SM-speed balanced partition (SGP4B_SMBAL=0/1 builds from
# tools/build_variants.sh): C2/C3/C4 grid step (graph and direct launches)
cd $GRAFT_REPO_ROOT
L=$PWD/paper_2603_27830_b200
for r in 1 2; do for v in ${VARIANTS:-bal0 bal1}; do
  for args in "--workload c2" "--workload c2 --no-graph" "--workload c2 --precision 64" "--workload c4"; do
    SGP4B_LIBRARY=$L/libsgp4b_$v.so python bench.py --no-cpu --no-accuracy --e2e-steps 3 $args \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', '$args', round(d['ms_per_step']*1e3,2), round(d['init_plus_propagate']['ms_per_step']*1e3,2), round(d['e2e']['ms_per_step'],3))"
  done
done; done
