# bench lines of the irregular BASELINE configurations (R-MAT s22 / s24), one GPU
bash scripts/gpu_bench.sh cfg3
bash scripts/gpu_bench.sh cfg5
