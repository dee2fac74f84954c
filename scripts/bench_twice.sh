cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b1.json 2>/dev/null
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2.json 2>/dev/null
