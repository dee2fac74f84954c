# ELL shuffle path: parity (bit-identical to the gather path), GPU test suite, A/B on cfg2 / cfg4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ell_shfl.py -x -q > gpurun_out/shfl_tests.log 2>&1; echo rc=$? >> gpurun_out/shfl_tests.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests2.log 2>&1; echo rc=$? >> gpurun_out/gpu_tests2.log
for S in 0 1; do
  SPB_ELL_SHFL=$S timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_cfg2_s$S.json 2> gpurun_out/ab_cfg2_s$S.err
  SPB_ELL_SHFL=$S timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ab_cfg4_s$S.json 2> gpurun_out/ab_cfg4_s$S.err
done
