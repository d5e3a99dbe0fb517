timeout 600 python -m pytest tests/test_learned.py tests/test_interp_gpu.py -x -q 2>&1 | tail -2
timeout 600 python bench.py --workload mlp --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['e2e'])"
