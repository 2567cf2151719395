# PPO tests + per-sample cfg4 PPO timing under the training-attention modes
# usage: MODES="default GO_TRAIN_ATTN=mma GO_TRAIN_ATTN=simt" bash scripts/gpu_ppo_cmp.sh
cd $GRAFT_REPO_ROOT
for mode in ${MODES:-default}; do
  e=""; [ "$mode" != default ] && e="$mode"
  echo "== $mode" >> gpurun_out/ppo_cmp.log
  env $e timeout 600 python -m pytest tests/test_gpu_ppo.py -m gpu -q 2>&1 | grep -E "passed|failed|Error:" | head -5 >> gpurun_out/ppo_cmp.log
  [ -n "$NO_TIMING" ] && continue
  env $e timeout 600 python scripts/bench_ppo.py 1 cfg4 2>&1 | cut -c1-260 >> gpurun_out/ppo_cmp.log
done
