# cfg4: pattern-ELL 27-point SpMM variants (0: CB1/MINB4, 1: CB1/MINB3, 2: CB2/MINB3)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in 0 1 2; do
  SPB_ELL_VARIANT=$v timeout 900 python bench.py --config cfg4 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/pv_cfg4_v$v.json 2> gpurun_out/pv_cfg4_v$v.err
done
