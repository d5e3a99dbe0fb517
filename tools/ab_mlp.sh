#!/usr/bin/env bash
# A/B of learned-MLP library variants: parity tests, then the MLP bench line.
for v in "$@"; do echo "$v: $(RAPP_LIB=build_variants/$v.so timeout 600 python -m pytest tests/test_learned.py -x -q 2>&1 | tail -1)"; done
for rep in 1 2 3; do
  for v in "$@"; do
    echo -n "$v: "; RAPP_LIB=build_variants/$v.so timeout 600 python bench.py --workload mlp --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value']/1e9,3), 'e9/s frac', d['roofline']['frac'], d['clocks']['sm_mhz'])"
  done
done
