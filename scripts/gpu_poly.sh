cd $GRAFT_REPO_ROOT
mkdir -p /tmp/lg
./scripts/exp_probe > gpurun_out/exp_probe.json 2>&1
GO_ATTN=tf32 GO_SAVE_LOGITS=/tmp/lg/tf32.pt timeout 300 python scripts/micro.py tc 8 >> gpurun_out/poly.log 2>&1
for k in 0 2 3 4 5 6 8; do
  GO_POLY16=$k GO_SAVE_LOGITS=/tmp/lg/np$k.pt timeout 300 python scripts/micro.py tc 8 >> gpurun_out/poly.log 2>&1
done
python - >> gpurun_out/poly.log 2>&1 <<'PY'
import torch
r = torch.load('/tmp/lg/tf32.pt').double()
for k in (0, 2, 3, 4, 5, 6, 8):
    x = torch.load(f'/tmp/lg/np{k}.pt').double()
    print(f"np={k}: max|d|/max|ref| vs tf32 = {float((x-r).abs().max()/r.abs().max()):.3e}")
PY
GO_POLY16=4 timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_poly4.log 2>&1
