# A/B: lanes-over-columns SpMM for long irregular rows vs the per-lane whole-row form
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_kernels.py -x -q > gpurun_out/vc_tests.log 2>&1
timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vc_cfg3_new.json 2> gpurun_out/vc_cfg3_new.err
SPB_VEC_COLS=0 SPB_LONG_COLS=0 timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vc_cfg3_old.json 2> gpurun_out/vc_cfg3_old.err
SPB_VEC_COLS=0 timeout 600 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/vc_cfg3_longonly.json 2> gpurun_out/vc_cfg3_longonly.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg3_vc.csv python tests/ncu_one.py cfg3 1 > gpurun_out/ncu_cfg3_vc.log 2>&1
timeout 900 python bench.py --config cfg5 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/vc_cfg5_new.json 2> gpurun_out/vc_cfg5_new.err
