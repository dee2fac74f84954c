# irregular SpMM A/B: loads in flight per lane (U = 4 / 6 / 8, int32 ids) vs the committed build
for lib in base u4 u6 u8; do
  SPECPART_B200_LIB=$PWD/diag/ab/lib$lib.so timeout 900 python bench.py --config cfg3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_n_$lib.json 2> gpurun_out/r02_n_$lib.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02_n_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib', d['ms_per_step'], r['ms_per_launch'], r['frac'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_n_$lib.err
done
