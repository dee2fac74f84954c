# one compute-sanitizer tool per call ($1 = memcheck | racecheck | synccheck | initcheck), after a clean plain run
timeout 600 python diag/sanitize_run.py > gpurun_out/r02_sanitize_plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool $1 --error-exitcode 9 --print-limit 40 python diag/sanitize_run.py \
    > gpurun_out/r02_sanitize_$1.log 2>&1
echo "rc=$?"; tail -25 gpurun_out/r02_sanitize_$1.log
