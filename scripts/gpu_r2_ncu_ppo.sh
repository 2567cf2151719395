#!/bin/bash
# Round-2 run: GPU tests, targeted ncu --set full captures of the hot kernels, then the
# cfg5 PPO epoch measurement.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> gpurun_out/r2/rc.txt
for spec in "attn_f16_kernel:1" "ffn_kernel:2" "trunk_mma_kernel:1" "tc_gemm_kernel:3" "segment_max128:1"; do
  name=${spec%%:*}; cnt=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$name -c $cnt \
    -o gpurun_out/r2/k_$name -f python scripts/micro.py tc 2 > gpurun_out/r2/ncu_$name.log 2>&1
  echo "ncu $name rc=$?" >> gpurun_out/r2/rc.txt
done
timeout 2400 python scripts/bench_ppo_cfg5.py 1 > gpurun_out/r2/ppo_cfg5.json 2> gpurun_out/r2/ppo_cfg5.err
echo "ppo rc=$?" >> gpurun_out/r2/rc.txt
