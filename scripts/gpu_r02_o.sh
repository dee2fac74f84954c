# rank-0 phase profile of cfg2 at N = GPUs
N=$(nvidia-smi -L | wc -l)
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 \
  diag/profile_dist.py cfg2 > gpurun_out/r02_o_prof_n$N.log 2>&1; tail -22 gpurun_out/r02_o_prof_n$N.log
