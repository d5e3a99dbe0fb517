for r in 1 2; do
for v in build_variants/prev.so paper_2505_01968_b200/librapp_b200.so; do
echo "== $v full"; RAPP_LIB=$v TICKS=8 timeout 600 python tools/tick_profile.py --full-grid 2>&1 | awk '{print $6}' | tr '\n' ' '; echo
done; done
