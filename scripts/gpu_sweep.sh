cd $GRAFT_REPO_ROOT
GO_S64=1 timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest.log 2>&1
for s in 0 1; do for k in ${NPS:-2 3 4}; do
  echo "S64=$s NP=$k" >> gpurun_out/sweep.log
  GO_S64=$s GO_POLY16=$k timeout 300 python scripts/micro.py tc 8 2>&1 | grep forward >> gpurun_out/sweep.log
done; done
