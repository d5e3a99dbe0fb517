# A/B of K3 library variants on the config-5 lattice bench: bash tools/ab_lattice.sh v1 v2 ...
# (variants are build_variants/<v>.so; the in-tree library runs the parity tests first)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_search_gpu.py tests/test_config1.py -x -q 2>&1 | tail -1
for i in 1 2; do
for v in "$@"; do
echo -n "$v: "; RAPP_LIB=build_variants/$v.so timeout 300 python bench.py --workload lattice --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['value']/1e12,4), d['roofline']['kernel_ms_per_launch'], d['clocks']['sm_mhz'])"
done; done
