# 4-GPU check (gpurun --gpus 4): CLI tests, dist tests, cfg2/cfg3/cfg5 at N=4, cfg4 at N=4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_cli.py -q -s -m gpu > gpurun_out/cli_gpu.log 2>&1; echo rc=$? >> gpurun_out/cli_gpu.log
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/mg_dist_tests.log 2>&1; echo rc=$? >> gpurun_out/mg_dist_tests.log
for CFG in cfg2 cfg3 cfg4 cfg5; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29571 bench.py --config $CFG --gpus 4 --steps 3 --warmup 3 2>gpurun_out/mg_${CFG}_n4.err | grep '^{' > gpurun_out/mg_${CFG}_n4.json
done
