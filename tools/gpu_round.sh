timeout 900 python -m pytest tests/test_tick_gpu.py tests/test_integration_gpu.py tests/test_slo.py tests/test_limits_gpu.py -x -q 2>&1 | tail -1 > gpurun_out/r2s3_lazy.txt
RAPP_TICK_MASK_NONE=1 timeout 900 python -m pytest tests/test_tick_gpu.py -x -q -k "bracket or config4 or random" 2>&1 | tail -1 >> gpurun_out/r2s3_lazy.txt
bash tools/ab_tickprof.sh build_variants/tick_base.so >> gpurun_out/r2s3_lazy.txt 2>&1
