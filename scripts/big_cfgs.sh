cd $GRAFT_REPO_ROOT
for c in cfg1 cfg3 cfg4; do
  timeout 1200 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/big_$c.json 2> gpurun_out/big_$c.err
done
SPB_PROFILE=1 timeout 600 python bench.py --config cfg3 --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/big_cfg3_prof.err
