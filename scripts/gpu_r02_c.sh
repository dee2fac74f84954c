# re-check: structured-mesh SpMM (compile-time stencil), preconditioner seams, AMG; mesh A/B
run() { timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_c_$1_$2.json 2> gpurun_out/r02_c_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_c_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['launches_per_step'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_c_$1_$2.err; }
timeout 1200 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_precond.py tests/test_gpu_amg.py tests/test_gpu_solver.py tests/test_cli.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_c_t.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r02_c_t.log | tail -3; grep -E "^(FAILED|E  )" gpurun_out/r02_c_t.log | head -30
for cfg in cfg2 cfg4; do
  SPB_MESH=0 run $cfg ell
  run $cfg mesh
done
