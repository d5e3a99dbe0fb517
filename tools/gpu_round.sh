nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/glds tools/micro/generic_lds.cu >/dev/null 2>&1 || true
timeout 900 python -m pytest tests/test_tick_gpu.py -q -x 2>&1 | tail -2
for i in 1 2; do
echo "== new full"; TICKS=40 timeout 300 python tools/tick_profile.py --full-grid 2>&1 | python tools/tick_summary.py
echo "== prev full"; RAPP_LIB=build_variants/prev.so TICKS=40 timeout 300 python tools/tick_profile.py --full-grid 2>&1 | python tools/tick_summary.py
done
echo "== new cfg4"; TICKS=40 timeout 300 python tools/tick_profile.py 2>&1 | python tools/tick_summary.py
echo "== prev cfg4"; RAPP_LIB=build_variants/prev.so TICKS=40 timeout 300 python tools/tick_profile.py 2>&1 | python tools/tick_summary.py
