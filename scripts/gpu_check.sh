# focused parity + bench after a change (edit the -k filter as needed)
timeout 1500 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_precond.py -m gpu -q -p no:cacheprovider -k "spmm or mesh or poly or precond" > gpurun_out/w_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/w_t.log; grep -E "^(FAILED|ERROR|E  )" gpurun_out/w_t.log | head -20
bash scripts/gpu_bench.sh cfg4
