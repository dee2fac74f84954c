# cfg3 profile of the previous build (diag/ab/libprev.so); guard-band test; combine seam tests
SPECPART_B200_LIB=$PWD/diag/ab/libprev.so SPB_PROFILE=1 timeout 600 python diag/profile_run.py cfg3 > gpurun_out/r02_j_prof_cfg3_prev.log 2>&1; echo "== prev"; tail -14 gpurun_out/r02_j_prof_cfg3_prev.log
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "guard or combine" > gpurun_out/r02_j_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_j_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_j_t.log | head -20
