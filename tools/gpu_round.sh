for v in paper_2505_01968_b200/librapp_b200.so build_variants/l3cuda.so; do
echo "== $v"
RAPP_LIB=$v timeout 300 python -m pytest tests/test_learned.py -x -q 2>&1 | tail -1
RAPP_LIB=$v timeout 600 python bench.py --workload mlp --steps 30 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['search']['points_per_s'])"
done
