cd $GRAFT_REPO_ROOT
for mode in "SPB_HALO_CE_SPLIT=1" "SPB_HALO_CE=1" "SPB_HALO_CE=0 SPB_HALO_FUSE=0"; do
  env $mode timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29567 bench.py --gpus 2 --steps 3 --warmup 3 2>/dev/null | grep '^{' > "gpurun_out/hf_$(echo $mode | tr ' =' '__').json"
done
