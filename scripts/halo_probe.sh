cd $GRAFT_REPO_ROOT
NG=$(nvidia-smi -L | wc -l)
SPB_HALO_PROBE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$NG --master-addr=127.0.0.1 --master-port=29561 bench.py --gpus $NG --steps 2 --warmup 3 > gpurun_out/probe.json 2> gpurun_out/probe.err
