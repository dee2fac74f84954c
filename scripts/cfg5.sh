cd $GRAFT_REPO_ROOT
timeout 1500 python bench.py --config cfg5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/cfg5_n1.json 2> gpurun_out/cfg5_n1.err
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29580 bench.py --config cfg5 --gpus 2 --steps 1 --warmup 3 2>gpurun_out/cfg5_n2.err | grep '^{' > gpurun_out/cfg5_n2.json
