# A/B 2: short-bin lanes-over-columns variant; Laplacian parity with long normalized rows
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -x -q > gpurun_out/vc2_tests.log 2>&1
SPB_VEC_COLS_SHORT=1 timeout 900 python -m pytest tests/test_gpu_solver.py -x -q > gpurun_out/vc2_tests_short.log 2>&1
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vc2_cfg3_def.json 2> gpurun_out/vc2_cfg3_def.err
SPB_VEC_COLS_SHORT=1 timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vc2_cfg3_short.json 2> gpurun_out/vc2_cfg3_short.err
SPB_VEC_COLS_SHORT=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg3_vc2.csv python tests/ncu_one.py cfg3 1 > gpurun_out/ncu_cfg3_vc2.log 2>&1
