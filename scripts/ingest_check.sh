# device ingestion: parity tests + timing vs the reference on raw R-MAT
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_ingest.py -x -q > gpurun_out/ingest_tests.log 2>&1
timeout 1500 python tests/ingest_bench.py 18 22 24 > gpurun_out/ingest_bench.json 2> gpurun_out/ingest_bench.err
