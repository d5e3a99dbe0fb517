timeout 600 python -m pytest tests/test_config1.py tests/test_tick_gpu.py -x -q 2>&1 | tail -3
