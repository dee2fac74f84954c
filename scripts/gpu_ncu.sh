# ncu evidence for one configuration ($1, default cfg2), each only after a clean plain run:
#   launches  -> the launch list (gpu__time_duration, DRAM bytes) of one partition after a warm-up
#   full RE   -> ncu --set full of the first launch matching the kernel regex RE after SKIP ($3) launches
# usage: gpurun -- 'bash scripts/gpu_ncu.sh cfg2 launches'  |  'bash scripts/gpu_ncu.sh cfg2 full spmm_mesh_poly2 30'
cfg=${1:-cfg2}; mode=${2:-launches}
python diag/ncu_one.py $cfg 1 > gpurun_out/ncu_${cfg}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/ncu_${cfg}_plain.log; exit 1; }
if [ "$mode" = launches ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv \
      --log-file gpurun_out/ncu_${cfg}_launches.csv python diag/ncu_one.py $cfg 2 > gpurun_out/ncu_${cfg}.log 2>&1
else
  ncu --set full --clock-control none --import-source on -k regex:$3 -s ${4:-30} -c 1 \
      -o gpurun_out/ncu_${cfg}_$3 python diag/ncu_one.py $cfg 1 > gpurun_out/ncu_${cfg}.log 2>&1
fi
echo "ncu rc=$?"; tail -2 gpurun_out/ncu_${cfg}.log
