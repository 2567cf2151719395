cd $GRAFT_REPO_ROOT
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ffn_kernel|trunk_mma_kernel|tc_gemm_kernel<144|tc_gemm_kernel<128, 1, 1" -c 8 -o gpurun_out/more_full -f python scripts/micro.py tc 2 > gpurun_out/ncu_more.log 2>&1; echo "more $?" >> gpurun_out/status.txt
timeout 600 ncu --set full --clock-control none -k regex:"des_kernel" -c 1 -o gpurun_out/des_full2 -f python scripts/micro.py des 512 > gpurun_out/ncu_des2.log 2>&1; echo "des $?" >> gpurun_out/status.txt
