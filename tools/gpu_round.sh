timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
TICKS=12 timeout 600 python tools/tick_profile.py > gpurun_out/tick_profile.log 2>&1
TICKS=12 timeout 600 python tools/tick_profile.py --full-grid > gpurun_out/tick_profile_full.log 2>&1
cat gpurun_out/tick_profile.log gpurun_out/tick_profile_full.log
