# multi-GPU bench sweep (run under gpurun --gpus N): cfg2 at N=1, 2 (P2P and NCCL halo), profile at N=2
cd $GRAFT_REPO_ROOT
NG=$(nvidia-smi -L | wc -l)
CFG=${CFG:-cfg2}
timeout 300 python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg_n1.json 2> gpurun_out/mg_n1.err
for N in 2 4 8; do
  [ $N -le $NG ] || continue
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2954$N bench.py --config $CFG --gpus $N --steps 3 --warmup 3 2>gpurun_out/mg_n$N.err | grep '^{' > gpurun_out/mg_n$N.json
done
SPB_P2P=0 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29551 bench.py --config $CFG --gpus 2 --steps 3 --warmup 3 2>/dev/null | grep '^{' > gpurun_out/mg_n2_nccl.json
SPB_PROFILE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29552 bench.py --config $CFG --gpus 2 --steps 1 --warmup 3 > /dev/null 2> gpurun_out/mg_n2_prof.err
