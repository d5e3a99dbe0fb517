timeout 600 python -m pytest tests/test_limits_gpu.py -x -q > gpurun_out/r2s3_limits.log 2>&1
timeout 600 python tools/tick_e2e_split.py --full-grid > gpurun_out/r2s3_tick_split.txt 2>&1
TICKS=40 timeout 600 python tools/tick_profile.py --full-grid > gpurun_out/r2s3_tickprof_full.txt 2>&1
