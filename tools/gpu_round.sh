timeout 900 python -m pytest tests/test_tick_gpu.py tests/test_integration_gpu.py tests/test_slo.py -x -q 2>&1 | tail -1 > gpurun_out/r2s3_ff.txt
bash tools/ab_tickprof.sh build_variants/tick_base.so >> gpurun_out/r2s3_ff.txt 2>&1
