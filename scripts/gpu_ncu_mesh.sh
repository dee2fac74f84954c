# ncu --set full of the structured-mesh SpMM on cfg2 (one partition after a warm-up)
python diag/ncu_one.py cfg2 2 > gpurun_out/r02_ncu_mesh_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:spmm_mesh_kernel -s 200 -c 2 \
    -o gpurun_out/r02_mesh2_cfg2 python diag/ncu_one.py cfg2 2 > gpurun_out/r02_ncu_mesh.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/r02_ncu_mesh.log
