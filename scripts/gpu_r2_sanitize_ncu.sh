#!/bin/bash
# Round-2 evidence run (one GPU): compute-sanitizer on the small end-to-end workload, then
# ncu --set full captures of the hot kernels and the launch list of a short bench step.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r2
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_small.py \
    > gpurun_out/r2/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2/sanitize_rc.txt
done
timeout 900 ncu --set full --clock-control none --import-source on \
  -k regex:"attn_f16_kernel|tc_gemm_kernel|ffn_kernel|segment_max128|trunk_mma_kernel|des_kernel" \
  --launch-skip 0 --launch-count 12 -o gpurun_out/r2/full -f python scripts/micro.py tc 2 \
  > gpurun_out/r2/ncu_full.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
  --log-file gpurun_out/r2/launches.csv python bench.py --steps 1 --warmup 0 --placements 64 \
  --no-cpu-baseline > gpurun_out/r2/ncu_launch.log 2>&1
echo done
