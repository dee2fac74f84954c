# Round-end style check: GPU tests, default bench, reference arm, smoke; then cfg3 vector-SpMM profiles
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cfg3_b.json 2> gpurun_out/cfg3_b.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_cfg3.csv python tests/ncu_one.py cfg3 1 > gpurun_out/ncu_cfg3_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_vec_kernel -s 20 -c 3 \
    -o gpurun_out/cfg3_vec python tests/ncu_one.py cfg3 1 > gpurun_out/ncu_cfg3_vec.log 2>&1
