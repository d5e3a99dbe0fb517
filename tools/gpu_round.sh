timeout 600 python bench.py --workload tick > gpurun_out/bench_tick.log 2>&1
timeout 900 python bench.py --workload tick --full-grid --ticks 20 > gpurun_out/bench_tick_full.log 2>&1
for f in bench_tick bench_tick_full; do tail -1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); t=d['tick']; print(t['grid'], t['device_us_median'], t['device_us_max'], t['e2e_us_median'], d['clocks'])"; done
