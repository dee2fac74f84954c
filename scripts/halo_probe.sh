cd $GRAFT_REPO_ROOT
SPB_HALO_PROBE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29561 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/probe.json 2> gpurun_out/probe.err
