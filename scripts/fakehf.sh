cd $GRAFT_REPO_ROOT
python bench.py --config cfg2h --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fh0.json 2>/dev/null
SPB_FAKE_HF=1 python bench.py --config cfg2h --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fh1.json 2>/dev/null
