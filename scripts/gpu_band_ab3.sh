# A/B of the band-staged mesh SpMM variants (L2 prefetch, rows per thread, ring sizing) vs pattern ELL
run() { timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ab3_$1_$2.json 2> gpurun_out/r02_ab3_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_ab3_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])"; }
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py -m gpu -q -x -p no:cacheprovider -k "spmm or lobpcg or poly" > gpurun_out/r02_band3_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_band3_t.log
for cfg in cfg2 cfg4; do
  SPB_BAND=0 run $cfg old
  SPB_BAND_CTAS=3 run $cfg b3r2
  SPB_BAND_CTAS=2 run $cfg b2r2
  SPB_BAND_CTAS=3 SPB_BAND_RPT=1 run $cfg b3r1
  SPB_BAND_CTAS=4 SPB_BAND_RPT=1 run $cfg b4r1
done
