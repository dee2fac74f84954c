cd $GRAFT_REPO_ROOT
python tests/ncu_one.py cfg2 > gpurun_out/ncu_one_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size,launch__shared_mem_per_block_dynamic --clock-control none --csv \
    -k regex:ts_ --log-file gpurun_out/ts_bulk_launches.csv python tests/ncu_one.py cfg2 > /dev/null 2>&1
SPB_TS_BULK=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,launch__grid_size --clock-control none --csv \
    -k regex:ts_ --log-file gpurun_out/ts_old_launches.csv python tests/ncu_one.py cfg2 > /dev/null 2>&1
