#!/bin/bash
# Round-2 closing measurement: full GPU suite (parity reports refreshed), smoke, the
# headline bench (mode R), the mode-S line, the reference arm, and the bench's launch list.
cd $GRAFT_REPO_ROOT
OUT=gpurun_out/final
mkdir -p $OUT/parity
GO_PARITY_REPORT_DIR=$OUT/parity timeout 2400 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.txt 2>&1
echo "pytest rc=$?" >> $OUT/rc.txt
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $OUT/smoke.txt 2>&1
echo "smoke rc=$?" >> $OUT/rc.txt
timeout 1800 python bench.py --steps 3 --warmup 3 > $OUT/bench_R.json 2> $OUT/bench_R.err
echo "bench R rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --steps 3 --warmup 3 --mode S --no-cpu-baseline > $OUT/bench_S.json 2> $OUT/bench_S.err
echo "bench S rc=$?" >> $OUT/rc.txt
timeout 900 python bench.py --impl reference --steps 1 --warmup 3 > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "bench ref rc=$?" >> $OUT/rc.txt
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file $OUT/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $OUT/ncu_bench.log 2>&1
echo "ncu rc=$?" >> $OUT/rc.txt
