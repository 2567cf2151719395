# round-end measurement: full GPU tests, headline bench, PPO timings, ncu of the PPO kernels
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final_pytest.log 2>&1; echo "pytest $?" >> gpurun_out/final_status.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench $?" >> gpurun_out/final_status.txt
timeout 600 python scripts/bench_ppo.py 1 cfg4 > gpurun_out/final_ppo_cfg4.json 2>&1; echo "ppo4 $?" >> gpurun_out/final_status.txt
GO_TRAIN_ATTN=simt GO_TRAIN_GEMM=simt timeout 600 python scripts/bench_ppo.py 1 cfg4 > gpurun_out/final_ppo_cfg4_simt.json 2>&1; echo "ppo4s $?" >> gpurun_out/final_status.txt
timeout 600 python scripts/bench_ppo.py > gpurun_out/final_ppo_cfg1.json 2>&1; echo "ppo1 $?" >> gpurun_out/final_status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dkv_kernel|dq_kernel|trunk_mma_kernel" --launch-skip 10 -c 6 -o gpurun_out/ppo_kernels python scripts/bench_ppo.py 1 cfg4 > gpurun_out/ncu_ppo_full.log 2>&1; echo "ncu $?" >> gpurun_out/final_status.txt
