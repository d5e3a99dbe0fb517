# A/B of the host tick path: bash tools/ab_tick_e2e.sh v1 v2 ... (build_variants/<v>.so)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -1
for i in 1 2; do for v in "$@"; do
echo "== $v"; RAPP_LIB=build_variants/$v.so timeout 300 python tools/tick_e2e_split.py 2>/dev/null | grep call
RAPP_LIB=build_variants/$v.so timeout 300 python tools/tick_e2e_split.py --full-grid 2>/dev/null | grep call
done; done
