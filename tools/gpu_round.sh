timeout 900 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -2
echo "== full"; TICKS=8 timeout 300 python tools/tick_profile.py --full-grid 2>&1 | awk '{print $6}' | tr '\n' ' '; echo
echo "== cfg4"; TICKS=8 timeout 300 python tools/tick_profile.py 2>&1 | awk '{print $6}' | tr '\n' ' '; echo
TICKS=2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tick -c 20 --csv --log-file gpurun_out/ncu_tick_side.csv python tools/tick_profile.py > gpurun_out/ncu_tick_side.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/ncu_tick_side.log
