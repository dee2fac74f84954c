# Round-end check of HEAD: GPU tests, default bench, reference arm, smoke, cfg2 launch list
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/f_gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/f_gpu_tests.log
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/f_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/f_smoke.log
timeout 900 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f_bench_ref.json 2> gpurun_out/f_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/f_launches_cfg2.csv python tests/ncu_one.py cfg2 1 > gpurun_out/f_ncu_launch.log 2>&1
