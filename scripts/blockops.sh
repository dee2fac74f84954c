cd $GRAFT_REPO_ROOT
echo "== bulk" ; python tests/bench_blockops.py 2097152 6 micro 2>&1 | grep -v BLOCKOPS; python tests/bench_blockops.py 2097152 6 2>&1 | grep -v BLOCKOPS
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bulk_on.json 2>gpurun_out/bulk_on.err
SPB_PROFILE=1 timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/bulk_prof.err
