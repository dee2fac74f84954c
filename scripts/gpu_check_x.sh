# register-resident mt19937_64 twist: bit-exact initial blocks + cfg2/cfg3 bench
timeout 2000 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline.py tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider -k "initial or cfg1 or cfg2 or poly" > gpurun_out/x_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/x_t.log; grep -E "^(FAILED|ERROR|E  )" gpurun_out/x_t.log | head -20
bash scripts/gpu_bench.sh cfg2
bash scripts/gpu_profile.sh cfg2
