# A/B of library builds on one configuration: bash scripts/gpu_ab.sh cfg2 v1 h2  (diag/ab/lib<name>.so)
cfg=$1; shift
for lib in "$@"; do
  SPECPART_B200_LIB=$PWD/diag/ab/lib$lib.so timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ab_$lib.json 2> gpurun_out/ab_$lib.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$lib.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$lib', d['ms_per_step'], r['ms_per_launch'], r['frac'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/ab_$lib.err
done
