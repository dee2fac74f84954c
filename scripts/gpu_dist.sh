# multi-GPU: row-partitioned parity (copy-engine / fused / NCCL halo paths), then cfg2 and cfg4 bench lines
# usage: gpurun --gpus 2 -- 'bash scripts/gpu_dist.sh'
timeout 1500 python -m pytest tests/test_gpu_dist.py -m gpu -q -p no:cacheprovider > gpurun_out/dist_tests.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/dist_tests.log
for cfg in cfg2 cfg4; do bash scripts/gpu_bench.sh $cfg; done
