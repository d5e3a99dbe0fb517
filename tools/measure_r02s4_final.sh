#!/usr/bin/env bash
# Round-2 session-4 closing measurement set (1 x B200): GPU tests, smoke, every bench line,
# the reference arm, and the lattice workload's launch list.
mkdir -p gpurun_out
P=gpurun_out/s8
python -m pytest tests -m gpu -q > ${P}_gputest.log 2>&1; echo "tests rc=$?" >> ${P}_gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > ${P}_smoke.log 2>&1; echo "smoke rc=$?" >> ${P}_smoke.log
python bench.py > ${P}_bench_default_100.log 2>&1
python bench.py --steps 20 --warmup 5 > ${P}_bench_default_20.log 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > ${P}_bench_reference.log 2>&1
python bench.py --workload lattice --steps 20 --warmup 3 > ${P}_bench_lattice.log 2>&1
python bench.py --workload mlp > ${P}_bench_mlp.log 2>&1
for r in 1 2; do python bench.py --workload tick --full-grid --ticks 50 --warmup 5 > ${P}_tick_full_$r.log 2>&1; done
python bench.py --workload tick --ticks 50 --warmup 5 > ${P}_tick_c4.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
  --log-file ${P}_lattice_launches.csv python bench.py --workload lattice --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > ${P}_ncu_lattice.log 2>&1
