# two-step polynomial kernel: parity (kernels, precond, solver, baseline cfg2) + cfg2 bench + profile
timeout 1500 python -m pytest tests/test_gpu_precond.py tests/test_gpu_solver.py tests/test_gpu_kernels.py tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider -x -k "not cfg3 and not cfg5 and not cfg4" > gpurun_out/r02_r_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_r_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_r_t.log | head -20
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_r_bench.json 2> gpurun_out/r02_r_bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r02_r_bench.json').read().strip().splitlines()[-1]); r=d['roofline']
print(d['ms_per_step'], d['e2e']['value'], r['ms_per_launch'], r['launches_per_step'], r['frac'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_r_bench.err
SPB_PROFILE=1 timeout 300 python diag/profile_run.py cfg2 > gpurun_out/r02_r_prof.log 2>&1; tail -16 gpurun_out/r02_r_prof.log
