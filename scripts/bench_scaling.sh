# multi-GPU bench sweep (run under gpurun --gpus N): N=1.. available, P2P default; dist tests first
cd $GRAFT_REPO_ROOT
NG=$(nvidia-smi -L | wc -l)
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/dist_tests.log 2>&1
for CFG in ${CFGS:-cfg2}; do
  timeout 600 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sc_${CFG}_n1.json 2> /dev/null
  for N in 2 4 8; do
    [ $N -le $NG ] || continue
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2954$N bench.py --config $CFG --gpus $N --steps 3 --warmup 3 2>gpurun_out/sc_${CFG}_n$N.err | grep '^{' > gpurun_out/sc_${CFG}_n$N.json
  done
done
SPB_PROFILE=1 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29552 bench.py --gpus $NG --steps 1 --warmup 3 > /dev/null 2> gpurun_out/sc_prof.err
