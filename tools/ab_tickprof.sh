#!/usr/bin/env bash
# A/B of tick library variants: heavy full-grid and config-4 ticks (tools/tick_profile.py),
# interleaved runs.  bash tools/ab_tickprof.sh VARIANT.so ...  (in-tree library = "main")
for rep in 1 2; do
  for v in main "$@"; do
    lib=paper_2505_01968_b200/librapp_b200.so; [ "$v" != main ] && lib=$v
    for fg in --full-grid ""; do
      echo "== $v $fg rep $rep"
      RAPP_LIB=$lib TICKS=9 timeout 300 python tools/tick_profile.py $fg 2>&1 | awk '{print $2, $6}' | tr '\n' ' '; echo
    done
  done
done
