# full -m gpu suite on one GPU + the default bench line
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/r02_p_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_p_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_p_t.log | head -20
timeout 900 python bench.py > gpurun_out/r02_p_bench.json 2> gpurun_out/r02_p_bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/r02_p_bench.json
