# 27-point register-tiled mesh SpMM: parity, cfg4 A/B; cfg2 bench line (default settings)
run() { timeout 900 python bench.py --config $1 --steps $3 --warmup 3 $4 > gpurun_out/r02_f_$1_$2.json 2> gpurun_out/r02_f_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_f_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], d['e2e'], r['ms_per_launch'], r['launches_per_step'], r['frac'], d['result']['cut'], d['result']['iterations'], d.get('cpu_baseline'))" || tail -5 gpurun_out/r02_f_$1_$2.err; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_f_t.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_f_t.log
timeout 900 python -m pytest tests/test_gpu_baseline.py -m gpu -q -p no:cacheprovider -k "cfg4" > gpurun_out/r02_f_tb.log 2>&1; echo "pytest-cfg4 rc=$?"; tail -2 gpurun_out/r02_f_tb.log
SPB_MESH=0 run cfg4 ell 5 --no-cpu-baseline
run cfg4 mesh 5 --no-cpu-baseline
run cfg2 default 20 ""
