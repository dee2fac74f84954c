# Re-entry check of HEAD: GPU tests, default bench, reference arm, smoke, cfg4 and cfg5 numbers
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gpu_tests.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/cfg4_b.json 2> gpurun_out/cfg4_b.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_ell -s 60 -c 2 \
    -o gpurun_out/cfg4_ell python tests/ncu_one.py cfg4 1 > gpurun_out/ncu_cfg4_ell.log 2>&1
