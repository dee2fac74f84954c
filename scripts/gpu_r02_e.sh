# relabel A/B on the R-MAT configs, then the full GPU suite (baseline parity incl. cfg3-cfg5)
run() { timeout 900 python bench.py --config $1 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02_e_$1_$2.json 2> gpurun_out/r02_e_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_e_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['launches_per_step'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_e_$1_$2.err; }
SPB_RELABEL=0 run cfg3 plain
run cfg3 relabel
SPB_RECURRENCE=1 run cfg3 relabel_recur
SPB_RELABEL=0 run cfg5 plain
run cfg5 relabel
SPB_RECURRENCE=1 run cfg5 relabel_recur
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02_e_t.log 2>&1; echo "pytest rc=$?"
grep -E "passed|failed" gpurun_out/r02_e_t.log | tail -3; grep -E "^(FAILED|E  )" gpurun_out/r02_e_t.log | head -30
