cd $GRAFT_REPO_ROOT
for c in cfg2q cfg2e; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sc_$c.json 2> /dev/null
  SPB_PROFILE=1 timeout 600 python bench.py --config $c --steps 1 --warmup 2 --no-cpu-baseline > /dev/null 2> gpurun_out/prof_$c.err
done
