#!/bin/bash
# tcgen05 tape evidence: full GPU tests, ncu --set full of the tape kernels, cfg5 PPO epoch.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2t
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2t/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2t/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"tape_fwd_kernel|tape_dq_kernel|tape_dkv_kernel|wgrad_tc_kernel" -c 4 \
  -o gpurun_out/r2t/tape -f python scripts/bench_ppo.py 1 cfg4 > gpurun_out/r2t/ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/r2t/rc.txt
timeout 2400 python scripts/bench_ppo_cfg5.py 1 > gpurun_out/r2t/ppo_cfg5.json 2> gpurun_out/r2t/ppo_cfg5.err
echo "ppo rc=$?" >> gpurun_out/r2t/rc.txt
