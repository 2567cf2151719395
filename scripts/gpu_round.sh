cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $? >> gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $? >> gpurun_out/status.txt
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench $? >> gpurun_out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo ncul $? >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"attn_f16|tc_gemm|segment_max|des_kernel|attn_kernel" -c 10 -o gpurun_out/prof -f python bench.py --placements 26 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1; echo ncuf $? >> gpurun_out/status.txt
