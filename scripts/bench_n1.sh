cd $GRAFT_REPO_ROOT
nproc > gpurun_out/n1_nproc.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/n1.json 2> gpurun_out/n1.err
SPB_PROFILE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/n1_prof.err
