# multi-GPU: row-partitioned parity (ce / fused / nccl paths) and the bench at N = GPUs
N=$(nvidia-smi -L | wc -l); echo "gpus=$N"
timeout 1500 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_dist_t.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_dist_t.log; grep -E "^(FAILED|E  )" gpurun_out/r02_dist_t.log | head -20
for cfg in cfg2 cfg4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus $N --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_dist_$cfg.json 2> gpurun_out/r02_dist_$cfg.err
  python -c "
import json; d=json.loads(open('gpurun_out/r02_dist_$cfg.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$cfg', d['n_gpus'], d['ms_per_step'], r['ms_per_launch'], r['frac'], d['result']['cut'], d['result']['iterations'], d.get('halo'))" || tail -5 gpurun_out/r02_dist_$cfg.err
done
