# usage: CONFIGS="GO_ATTN=tf32 GO_POLY16=4 GO_POLYLP=1,GO_POLY16=4" bash scripts/gpu_sweep.sh
# (first config = logits reference; commas separate env assignments within a config)
cd $GRAFT_REPO_ROOT
mkdir -p /tmp/lg
[ -n "$PYTEST_ENV$RUN_PYTEST" ] && env ${PYTEST_ENV:-} timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
i=0
for c in $CONFIGS; do
  echo "$c" >> gpurun_out/sweep.log
  env ${c//,/ } GO_SAVE_LOGITS=/tmp/lg/$i.pt timeout 300 python scripts/micro.py tc 8 2>&1 | grep forward >> gpurun_out/sweep.log
  i=$((i+1))
done
python - >> gpurun_out/sweep.log 2>&1 <<PY
import torch, os
n = $i
r = torch.load('/tmp/lg/0.pt').double()
for k in range(1, n):
    if os.path.exists(f'/tmp/lg/{k}.pt'):
        x = torch.load(f'/tmp/lg/{k}.pt').double()
        print(f"config {k}: logits max|d|/max|ref| vs config 0 = {float((x-r).abs().max()/r.abs().max()):.3e}")
PY
