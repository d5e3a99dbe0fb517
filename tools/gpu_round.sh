timeout 600 python -m pytest tests/test_metrics.py -x -q 2>&1 | tail -25
