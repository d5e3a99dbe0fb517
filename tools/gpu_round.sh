timeout 900 python -m pytest tests/test_tick_gpu.py tests/test_integration_gpu.py tests/test_slo.py tests/test_limits_gpu.py -x -q 2>&1 | tail -2 > gpurun_out/r2s3_spec.txt
RAPP_LIB=build_variants/prof.so timeout 300 python tools/tick_commit_breakdown.py --full-grid > gpurun_out/r2s3_commit_breakdown3.txt 2>&1
bash tools/ab_tickprof.sh build_variants/tick_base.so >> gpurun_out/r2s3_spec.txt 2>&1
