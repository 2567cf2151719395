cd $GRAFT_REPO_ROOT
timeout 2400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_full.csv python bench.py --placements 52 --warmup 3 --steps 1 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "ncul $?" >> gpurun_out/status.txt
