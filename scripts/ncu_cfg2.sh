# ncu launch list of one cfg2 partition + full captures of the top kernels (single GPU)
cd $GRAFT_REPO_ROOT
python tests/ncu_one.py cfg2 > gpurun_out/ncu_one_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r01c.csv python tests/ncu_one.py cfg2 > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:spmm_ell_kernel -s 40 -c 1 \
    -o gpurun_out/ell_full_r01c python tests/ncu_one.py cfg2 > gpurun_out/ncu_full1.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:ts_bulk_kernel -s 120 -c 4 \
    -o gpurun_out/ts_full_r01c python tests/ncu_one.py cfg2 > gpurun_out/ncu_full2.log 2>&1
