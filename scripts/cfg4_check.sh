cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
for v in 0 1 2; do
SPB_ELL_VARIANT=$v timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/big_cfg4_v$v.json 2> gpurun_out/big_cfg4.err
done
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg2_check.json 2>/dev/null
