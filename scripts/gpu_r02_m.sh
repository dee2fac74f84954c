# ncu launch list of one cfg3 partition (after a clean plain run)
python diag/ncu_one.py cfg3 1 > gpurun_out/r02_m_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 2000 --csv \
    --log-file gpurun_out/r02_m_launches_cfg3.csv python diag/ncu_one.py cfg3 1 > gpurun_out/r02_m_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/r02_m_ncu.log
