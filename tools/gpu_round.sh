timeout 600 python -m pytest tests/test_tick_gpu.py -x -q -k "replay or golden" 2>&1 | tail -30
