# A/B of the band-staged mesh SpMM (spmm_band.cu) against the pattern-ELL kernel
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider > gpurun_out/r02_band_t.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/r02_band_t.log
timeout 900 python -m pytest tests/test_gpu_baseline.py -m gpu -q -x -p no:cacheprovider -k "cfg1 or cfg2" > gpurun_out/r02_band_tb.log 2>&1; echo "pytest-baseline rc=$?"; tail -5 gpurun_out/r02_band_tb.log
for cfg in cfg2 cfg4; do
  SPB_BAND=0 timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ab_${cfg}_old.json 2> gpurun_out/r02_ab_${cfg}_old.err
  timeout 600 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ab_${cfg}_band.json 2> gpurun_out/r02_ab_${cfg}_band.err
  for v in old band; do python -c "
import json,sys; d=json.loads(open('gpurun_out/r02_ab_${cfg}_'+'$v'+'.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$cfg', '$v', d['ms_per_step'], r['ms_per_launch'], r['frac'], d['result']['cut'], d['result']['iterations'])"; done
done
