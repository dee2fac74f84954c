# recurrence tests, preconditioner seams; recurrence A/B on cfg3 and cfg2
run() { timeout 900 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline $3 > gpurun_out/r02_d_$1_$2.json 2> gpurun_out/r02_d_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_d_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['launches_per_step'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_d_$1_$2.err; }
timeout 1200 python -m pytest tests/test_gpu_recurrence.py tests/test_gpu_precond.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_d_t.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r02_d_t.log | tail -3; grep -E "^(FAILED|E  )" gpurun_out/r02_d_t.log | head -30
for cfg in cfg3 cfg2 cfg1; do
  run $cfg off ""
  SPB_RECURRENCE=1 run $cfg on ""
done
timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -q -p no:cacheprovider -k "mesh or spmm_bit_exact" > gpurun_out/r02_d_t2.log 2>&1; echo "pytest-mesh rc=$?"; tail -2 gpurun_out/r02_d_t2.log
for cfg in cfg2 cfg4; do
  SPB_MESH_CTAS=2 run $cfg mesh2 ""
  SPB_MESH_CTAS=3 run $cfg mesh3 ""
done
