cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --workload cfg2 > gpurun_out/bench_cfg2.log 2>&1
timeout 900 python bench.py --workload cfg1 > gpurun_out/bench_cfg1.log 2>&1
