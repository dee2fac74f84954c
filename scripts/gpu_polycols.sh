# A/B: GMRES-polynomial apply column by column (L2-resident sweeps) vs all columns per root
run() { timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_pc_$1_$2.json 2> gpurun_out/r02_pc_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_pc_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['launches_per_step'], r['frac'], d['result']['cut'], d['result']['iterations'])"; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_pc_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pc_t.log
SPB_POLY_COLS=1 timeout 900 python -m pytest tests/test_gpu_solver.py tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider -k "poly or cfg2" > gpurun_out/r02_pc_t2.log 2>&1; echo "pytest-cols rc=$?"; tail -3 gpurun_out/r02_pc_t2.log
for cfg in cfg2 cfg4; do
  SPB_BAND=0 run $cfg rows
  SPB_BAND=0 SPB_POLY_COLS=1 run $cfg cols
  SPB_POLY_COLS=1 run $cfg cols_band
done
timeout 900 python -m pytest tests/test_gpu_amg.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_amg_t.log 2>&1; echo "pytest-amg rc=$?"; tail -30 gpurun_out/r02_amg_t.log
