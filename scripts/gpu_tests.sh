# The full -m gpu suite on one GPU, then the default bench line (driver-equivalent round-end check).
# usage: gpurun --timeout 3600 -- 'bash scripts/gpu_tests.sh'
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/gpu_tests.log; grep -E "^(FAILED|E  )" gpurun_out/gpu_tests.log | head -20
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"; tail -c 400 gpurun_out/bench.json
