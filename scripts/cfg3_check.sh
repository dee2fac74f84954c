cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 1200 python bench.py --config cfg3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/big_cfg3.json 2> gpurun_out/big_cfg3.err
SPB_PROFILE=1 timeout 600 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/big_cfg3_prof.err
