for v in paper_2505_01968_b200/librapp_b200.so build_variants/u2.so build_variants/u8.so; do
echo "== $v"; RAPP_LIB=$v timeout 300 python bench.py --workload lattice --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['kernel_ms_per_launch'], d['roofline']['frac'])"
done
