# bench lines of one configuration ($1, default cfg2) at N = every visible GPU (torchrun when N > 1)
# usage: gpurun [--gpus N] -- 'bash scripts/gpu_bench.sh cfg4'
cfg=${1:-cfg2}; N=$(nvidia-smi -L | wc -l)
if [ "$N" -gt 1 ]; then
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_n$N.json 2> gpurun_out/bench_${cfg}_n$N.err
else
  timeout 1500 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${cfg}_n1.json 2> gpurun_out/bench_${cfg}_n1.err
fi
python -c "
import json; d=json.loads(open('gpurun_out/bench_${cfg}_n$N.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$cfg', d['n_gpus'], d['ms_per_step'], d['e2e']['value'], r['ms_per_launch'], r['frac'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/bench_${cfg}_n$N.err
