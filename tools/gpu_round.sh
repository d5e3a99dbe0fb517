timeout 300 python -m pytest tests/test_learned.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --workload mlp --steps 30 2>&1 | tail -1 | cut -c 1-900
