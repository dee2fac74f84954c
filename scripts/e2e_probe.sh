cd $GRAFT_REPO_ROOT
nvidia-smi -i 0 --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > /dev/null 2>&1 &
SMI=$!
sleep 2
SPB_PROFILE=1 python tests/e2e_probe2.py > gpurun_out/e2e_probe2.log 2>&1
SPB_POOL_RESERVE_GB=0 SPB_PROFILE=1 python tests/e2e_probe2.py > gpurun_out/e2e_probe3.log 2>&1
kill $SMI
