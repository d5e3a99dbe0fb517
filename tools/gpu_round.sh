timeout 900 python -m pytest tests/test_tick_gpu.py -q -x 2>&1 | tail -2
RAPP_LIB=build_variants/prof.so timeout 300 python tools/tick_commit_breakdown.py --full-grid 2>&1 | tail -12 | head -4
for i in 1 2; do
echo "== new full"; TICKS=40 timeout 300 python tools/tick_profile.py --full-grid 2>&1 | python tools/tick_summary.py
echo "== prev full"; RAPP_LIB=build_variants/prev.so TICKS=40 timeout 300 python tools/tick_profile.py --full-grid 2>&1 | python tools/tick_summary.py
done
