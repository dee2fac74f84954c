# focused parity + bench + profile after a change (edit the -k filter as needed)
timeout 2000 python -m pytest tests/test_gpu_guard.py tests/test_gpu_solver.py tests/test_gpu_recurrence.py tests/test_gpu_precond.py tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider -k "not cfg3 and not cfg5 and not cfg4" > gpurun_out/w_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/w_t.log; grep -E "^(FAILED|ERROR|E  )" gpurun_out/w_t.log | head -20
bash scripts/gpu_bench.sh cfg2
bash scripts/gpu_profile.sh cfg2
