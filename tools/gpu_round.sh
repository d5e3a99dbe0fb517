timeout 300 python tools/mlp_debug.py 2>&1 | grep -v Exception | head -12
timeout 300 python -m pytest tests/test_learned.py -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload mlp --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['search'])"
