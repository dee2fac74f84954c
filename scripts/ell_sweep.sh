cd $GRAFT_REPO_ROOT
for v in 0 1 2 3; do
  SPB_ELL_VARIANT=$v timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ell_v$v.json 2>/dev/null
done
