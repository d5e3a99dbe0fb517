timeout 900 python -m pytest tests/test_tick_gpu.py tests/test_integration_gpu.py -x -q 2>&1 | tail -1 > gpurun_out/r2s3_cov.txt
bash tools/ab_tickprof.sh build_variants/tick_base.so >> gpurun_out/r2s3_cov.txt 2>&1
