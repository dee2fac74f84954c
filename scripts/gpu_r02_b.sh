# preconditioner seams, AMG, shim caller and CLI parity; then ncu of the structured-mesh SpMM
timeout 1200 python -m pytest tests/test_gpu_precond.py tests/test_gpu_amg.py tests/test_gpu_solver.py tests/test_cli.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_b_t.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r02_b_t.log | tail -3; grep -E "^(FAILED|E  )" gpurun_out/r02_b_t.log | head -40
bash scripts/gpu_ncu_mesh.sh
