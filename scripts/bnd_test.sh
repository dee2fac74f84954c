cd $GRAFT_REPO_ROOT
for pct in 40 60 80; do
 for N in 2 4; do
  SPB_HALO_BND_PCT=$pct timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2957$N bench.py --gpus $N --steps 3 --warmup 3 2>/dev/null | grep '^{' > gpurun_out/sc_b${pct}_n$N.json
 done
done
