cd $GRAFT_REPO_ROOT
ncu --set full --clock-control none -k regex:spmm_group_kernel -s 6 -c 2 -o gpurun_out/cfg3_group python tests/ncu_one.py cfg3 1 > gpurun_out/ncu_cfg3_full.log 2>&1
