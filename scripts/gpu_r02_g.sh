# padded row-major blocks (irregular graphs): parity + cfg3 A/B; cfg2 phase profile
run() { timeout 900 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_g_$1_$2.json 2> gpurun_out/r02_g_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_g_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['launches_per_step'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_g_$1_$2.err; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_recurrence.py tests/test_gpu_amg.py tests/test_gpu_precond.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_g_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_g_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_g_t.log | head
timeout 900 python -m pytest tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider -k "cfg3" > gpurun_out/r02_g_tb.log 2>&1; echo "pytest-cfg3 rc=$?"; tail -2 gpurun_out/r02_g_tb.log
run cfg3 pad
SPB_RECURRENCE=1 run cfg3 pad_recur
SPB_PROFILE=1 timeout 300 python diag/profile_run.py cfg2 > gpurun_out/r02_g_prof_cfg2.log 2>&1; tail -40 gpurun_out/r02_g_prof_cfg2.log
