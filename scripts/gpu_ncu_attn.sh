cd $GRAFT_REPO_ROOT
GO_POLY16=${NP:-3} timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_f16 -c 1 -o gpurun_out/attn_cur -f python scripts/micro.py tc 2 > gpurun_out/ncu_attn.log 2>&1
