# piecewise initial block on the device: parity; cfg3 profile; then ncu --set full of the cfg3 irregular SpMM
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider -k "initial or cfg3 or cfg5" > gpurun_out/r02_l_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_l_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_l_t.log | head
SPB_PROFILE=1 timeout 600 python diag/profile_run.py cfg3 > gpurun_out/r02_l_prof_cfg3.log 2>&1; tail -18 gpurun_out/r02_l_prof_cfg3.log
python diag/ncu_one.py cfg3 1 > gpurun_out/r02_l_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_rowcols -s 20 -c 3 \
    -o gpurun_out/r02_cfg3_vec python diag/ncu_one.py cfg3 1 > gpurun_out/r02_l_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/r02_l_ncu.log
