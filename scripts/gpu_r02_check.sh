set -x
nproc; lscpu | grep "Model name"
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_t1.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/r02_t1.log
timeout 900 python scripts/cpu_thread_sweep.py cfg2 > gpurun_out/r02_sweep.log 2>&1; echo "sweep rc=$?"
cp profiles/cpu_thread_sweep.json gpurun_out/ 2>/dev/null
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench1.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench1.log
