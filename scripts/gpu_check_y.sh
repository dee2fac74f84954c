# pipelined two-step kernel: bit-exact poly parity on meshes + A/B on cfg2
timeout 1500 python -m pytest tests/test_gpu_precond.py tests/test_gpu_solver.py tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider -k "not cfg3 and not cfg5 and not cfg4" > gpurun_out/y_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/y_t.log; grep -E "^(FAILED|ERROR|E  )" gpurun_out/y_t.log | head -20
bash scripts/gpu_ab.sh cfg2 head pipe
