cd $GRAFT_REPO_ROOT
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1; echo "bench $?" >> gpurun_out/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --placements 256 --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1; echo "ncul $?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_f16 -c 1 -o gpurun_out/attn_full -f python scripts/micro.py tc 2 > gpurun_out/ncu_attn.log 2>&1; echo "ncuattn $?" >> gpurun_out/status.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"tc_gemm_kernel|segment_max|trunk_mma|ffn_kernel|features_inproj|neighbor_sample|sample_kernel|repack_kv16|mean_partial" -c 24 -o gpurun_out/others_full -f python scripts/micro.py tc 2 > gpurun_out/ncu_others.log 2>&1; echo "ncuothers $?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none -k regex:"des_kernel" -c 1 -o gpurun_out/des_full -f python scripts/micro.py des 256 > gpurun_out/ncu_des.log 2>&1; echo "ncudes $?" >> gpurun_out/status.txt
