cd $GRAFT_REPO_ROOT
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg_n1.json 2> gpurun_out/mg_n1.err
timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29541 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/mg_n2.json 2> gpurun_out/mg_n2.err
SPB_PROFILE=1 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29542 bench.py --gpus 2 --steps 1 --warmup 3 > /dev/null 2> gpurun_out/mg_n2_prof.err
