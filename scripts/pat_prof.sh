cd $GRAFT_REPO_ROOT
SPB_PROFILE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/pat_on_prof.err
SPB_NO_ELL_PAT=1 SPB_PROFILE=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2> gpurun_out/pat_off_prof.err
