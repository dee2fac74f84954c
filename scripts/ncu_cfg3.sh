cd $GRAFT_REPO_ROOT
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv \
    -k regex:spmm --log-file gpurun_out/launches_cfg3b.csv python tests/ncu_one.py cfg3 1 > gpurun_out/ncu_launch3.log 2>&1
