# A/B of tick library variants: bash tools/ab_tick.sh v1 v2 ... (build_variants/<v>.so);
# the in-tree library runs the tick parity tests first
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -1
for i in 1 2; do
for v in "$@"; do
echo -n "$v full: "; RAPP_LIB=build_variants/$v.so TICKS=40 timeout 300 python tools/tick_profile.py --full-grid 2>&1 | python tools/tick_summary.py
echo -n "$v cfg4: "; RAPP_LIB=build_variants/$v.so TICKS=40 timeout 300 python tools/tick_profile.py 2>&1 | python tools/tick_summary.py
done; done
