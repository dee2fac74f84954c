# cfg3 / cfg2 phase profiles with the initial-block phase split
for c in cfg3 cfg2; do SPB_PROFILE=1 timeout 600 python diag/profile_run.py $c > gpurun_out/r02_k_prof_$c.log 2>&1; echo "== $c"; tail -19 gpurun_out/r02_k_prof_$c.log; done
