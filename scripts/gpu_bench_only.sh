cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench $?" >> gpurun_out/status.txt
