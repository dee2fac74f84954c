# multi-GPU irregular graphs (run under gpurun --gpus 4): dist tests, cfg3 at 1/2/4, cfg5 at 2/4
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_dist.py -x -q > gpurun_out/isc_dist_tests.log 2>&1
for N in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2964$N bench.py --config cfg3 --gpus $N --steps 3 --warmup 3 2>gpurun_out/isc_cfg3_n$N.err | grep '^{' > gpurun_out/isc_cfg3_n$N.json
done
for N in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2966$N bench.py --config cfg5 --gpus $N --steps 2 --warmup 3 2>gpurun_out/isc_cfg5_n$N.err | grep '^{' > gpurun_out/isc_cfg5_n$N.json
done
