cd $GRAFT_REPO_ROOT
python tests/bench_one_blockop.py 2097152 0 1 0 0 3 > gpurun_out/one.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/one_ncu.csv python tests/bench_one_blockop.py 2097152 0 1 0 0 3 > /dev/null 2>&1
SPB_TS_BULK=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/one_ncu_old.csv python tests/bench_one_blockop.py 2097152 0 1 0 0 3 > /dev/null 2>&1
