# A/B of the band-staged mesh SpMM: ring sized for 2 or 3 CTAs/SM vs the pattern-ELL kernel
set -x
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider -k "spmm or lobpcg or poly" > gpurun_out/r02_band2_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_band2_t.log
run() { timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ab2_$1_$2.json 2> gpurun_out/r02_ab2_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_ab2_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])"; }
for cfg in cfg2 cfg4 cfg1; do
  SPB_BAND=0 run $cfg old
  SPB_BAND_CTAS=2 run $cfg b2
  SPB_BAND_CTAS=3 run $cfg b3
done
