# focused parity + bench + profile after a change (edit the -k filter as needed)
timeout 2000 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline.py tests/test_gpu_solver.py -m gpu -q -p no:cacheprovider -k "mj or cfg4 or cfg1 or partition or initial" > gpurun_out/w_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/w_t.log; grep -E "^(FAILED|ERROR|E  )" gpurun_out/w_t.log | head -20
bash scripts/gpu_bench.sh cfg4
