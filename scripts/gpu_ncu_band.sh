# ncu --set full of the band-staged mesh SpMM on cfg2 (one partition after a warm-up)
python diag/ncu_one.py cfg2 2 > gpurun_out/r02_ncu_band_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_band_kernel -s 200 -c 3 \
    -o gpurun_out/r02_band_cfg2 python diag/ncu_one.py cfg2 2 > gpurun_out/r02_ncu_band.log 2>&1
echo "rc=$?"; tail -5 gpurun_out/r02_ncu_band.log
