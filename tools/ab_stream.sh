#!/usr/bin/env bash
# A/B of K2 library variants (build_variants/<v>.so): k2_probe parity + timing on one
# config-2 table, then the default bench line's device value.  bash tools/ab_stream.sh v1 v2 ...
for rep in 1 2; do
  for v in "$@"; do
    echo "== $v rep $rep"
    RAPP_LIB=build_variants/$v.so timeout 300 python tools/k2_probe.py 50000000 10 2>&1 | tail -2
    RAPP_LIB=build_variants/$v.so timeout 300 python bench.py --steps 30 --no-e2e --no-cpu-baseline --no-extra 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('bench', round(d['value']/1e9,2), 'e9/s frac', d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
