# cfg2: pattern-ELL 7-point SpMM variants (0: CB2/MINB4, 1: CB2/MINB5, 2: CB1/MINB6, 3: CB4/MINB3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1 2 3 0; do
  SPB_ELL_VARIANT=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/pv_cfg2_v$v.json 2> gpurun_out/pv_cfg2_v$v.err
done
