# phase profile (SPB_PROFILE) of one partition of $1 (default cfg2): one GPU, or rank 0 of N under torchrun
cfg=${1:-cfg2}; N=$(nvidia-smi -L | wc -l)
if [ "$N" -gt 1 ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
    diag/profile_dist.py $cfg > gpurun_out/profile_${cfg}_n$N.log 2>&1
else
  SPB_PROFILE=1 timeout 600 python diag/profile_run.py $cfg > gpurun_out/profile_${cfg}_n1.log 2>&1
fi
tail -20 gpurun_out/profile_${cfg}_n$N.log
