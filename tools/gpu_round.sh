timeout 900 python -m pytest tests/test_tick_gpu.py -q -x -k "many_gpus" 2>&1 | tail -15
