cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bulk_on.json 2>gpurun_out/bulk_on.err
SPB_TS_STAGE_KB=12 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bulk_12.json 2>/dev/null
SPB_TS_STAGE_KB=48 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bulk_48.json 2>/dev/null
SPB_TS_BULK=0 timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bulk_off.json 2>/dev/null
SPB_PROFILE=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/bulk_prof.err
