# X reorthonormalized every 16 iterations + [H | P] merged orthonormalization: parity, cfg2/cfg4 bench, cfg2 profile
run() { timeout 900 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_h_$1_$2.json 2> gpurun_out/r02_h_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_h_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], d['e2e']['value'], r['ms_per_launch'], r['launches_per_step'], r['frac'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_h_$1_$2.err; }
timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_recurrence.py tests/test_gpu_amg.py tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_h_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_h_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_h_t.log | head -20
run cfg2 h
run cfg4 h
run cfg3 h
SPB_PROFILE=1 timeout 300 python diag/profile_run.py cfg2 > gpurun_out/r02_h_prof_cfg2.log 2>&1; tail -30 gpurun_out/r02_h_prof_cfg2.log
