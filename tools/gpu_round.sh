timeout 900 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -2
timeout 600 python -c "
import sys, argparse; sys.path.insert(0,'.')
import bench
a = argparse.Namespace(ticks=20, steps=20)
r = bench.run_replay(a, 0); print('replay', r['e2e_us_median'], r['e2e_us_max'])
t = bench.run_tick(a, 0, ticks=20); print('cfg4', t['device_us_median'], t['e2e_us_median'])
"
