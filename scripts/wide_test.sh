cd $GRAFT_REPO_ROOT
for W in 0 1; do
  SPB_ELL_WIDE=$W timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sc_w${W}_n1.json 2> /dev/null
  for N in 2 4; do
    SPB_ELL_WIDE=$W timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2954$N bench.py --gpus $N --steps 3 --warmup 3 2>/dev/null | grep '^{' > gpurun_out/sc_w${W}_n$N.json
  done
done
