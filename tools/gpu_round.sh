timeout 900 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -2
for v in build_variants/prev.so paper_2505_01968_b200/librapp_b200.so; do
echo "== $v full"; RAPP_LIB=$v TICKS=8 timeout 600 python tools/tick_profile.py --full-grid 2>&1 | awk '{print $6}' | tr '\n' ' '; echo
echo "== $v cfg4"; RAPP_LIB=$v TICKS=8 timeout 600 python tools/tick_profile.py 2>&1 | awk '{print $6}' | tr '\n' ' '; echo
done
