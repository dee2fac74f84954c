# structured-mesh SpMM (spmm_mesh.cu): parity tests, then A/B against the pattern-ELL kernel
run() { timeout 600 python bench.py --config $1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r02_mesh_$1_$2.json 2> gpurun_out/r02_mesh_$1_$2.err;
  python -c "
import json; d=json.loads(open('gpurun_out/r02_mesh_$1_$2.json').read().strip().splitlines()[-1]); r=d['roofline']
print('$1', '$2', d['ms_per_step'], r['ms_per_launch'], r['launches_per_step'], r['frac'], r['all_spmm'], d['result']['cut'], d['result']['iterations'])" || tail -5 gpurun_out/r02_mesh_$1_$2.err; }
timeout 120 ./build/tma_probe 36 0 -2; timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_solver.py tests/test_gpu_amg.py -m gpu -q -p no:cacheprovider > gpurun_out/r02_mesh_t.log 2>&1; echo "pytest rc=$?"; tail -30 gpurun_out/r02_mesh_t.log | grep -v "^\s*$" | tail -25
for cfg in cfg2 cfg4 cfg1; do
  SPB_MESH=0 run $cfg ell
  run $cfg mesh
done
