# cfg3 A/B: previous build (diag/ab/libprev.so) vs HEAD, phase profile of both
for lib in prev head; do
  if [ $lib = prev ]; then export SPECPART_B200_LIB=$PWD/diag/ab/libprev.so; else unset SPECPART_B200_LIB; fi
  SPB_PROFILE=1 timeout 600 python diag/profile_run.py cfg3 > gpurun_out/r02_i_prof_cfg3_$lib.log 2>&1; echo "== $lib"; tail -22 gpurun_out/r02_i_prof_cfg3_$lib.log
done
unset SPECPART_B200_LIB
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -p no:cacheprovider -k "guard or combine or shim or cpp" > gpurun_out/r02_i_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_i_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_i_t.log | head -20
