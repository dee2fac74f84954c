cd $GRAFT_REPO_ROOT
python tests/ncu_one.py cfg2 > gpurun_out/ncu_one_plain.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:ts_bulk_kernel -s 300 -c 6 \
    -o gpurun_out/bulk_full3 python tests/ncu_one.py cfg2 > gpurun_out/ncu_bulk.log 2>&1
