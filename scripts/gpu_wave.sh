cd $GRAFT_REPO_ROOT
for w in 2097152 4194304 8388608; do
  echo "GO_WAVE_ROWS=$w" >> gpurun_out/wave.log
  GO_WAVE_ROWS=$w timeout 600 python bench.py --placements 832 --warmup 1 --steps 1 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['kernel_ms'])" >> gpurun_out/wave.log 2>&1
done
