# ncu --set full of the cfg2 polynomial-step SpMM (pattern ELL), two launches (with / without H terms)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:spmm_ell -s 40 -c 2 \
    -o gpurun_out/cfg2_ell python tests/ncu_one.py cfg2 1 > gpurun_out/ncu_cfg2_ell.log 2>&1
