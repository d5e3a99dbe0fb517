#!/usr/bin/env bash
# Round-2 session-4 measurement set: GPU tests, smoke, default bench line (all extras),
# launch list, ncu --set full of K2, compute-sanitizer over K2 and the tick.
mkdir -p gpurun_out
P=gpurun_out/s5
python -m pytest tests -m gpu -q > ${P}_gputest.log 2>&1; echo "tests rc=$?" >> ${P}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc=$?" >> ${P}_smoke.log
python bench.py --steps 30 --warmup 5 > ${P}_bench_default.log 2>&1; echo "rc=$?" >> ${P}_bench_default.log
python bench.py --workload lattice --steps 20 --warmup 3 > ${P}_bench_lattice.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file ${P}_launches.csv python bench.py --steps 2 --warmup 3 --no-extra --no-cpu-baseline > ${P}_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_interp_fast -c 1 -f \
  -o ${P}_k2 python tools/k2_probe.py 20000000 1 > ${P}_ncu_k2.log 2>&1
CASES="k2 tick" bash tools/sanitize.sh > /dev/null 2>&1; cp gpurun_out/sanitize_summary.txt ${P}_sanitize_summary.txt
