set -x
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/bench_reference.log 2>&1
timeout 600 python bench.py --workload lattice > gpurun_out/bench_lattice.log 2>&1
timeout 600 python bench.py --workload tick > gpurun_out/bench_tick.log 2>&1
timeout 900 python bench.py --workload tick --full-grid --ticks 20 > gpurun_out/bench_tick_full.log 2>&1
timeout 600 python bench.py --workload mlp > gpurun_out/bench_mlp.log 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_default.csv python bench.py --steps 2 --warmup 3 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mec_lattice -c 1 -o gpurun_out/prof_k3_final python bench.py --workload lattice --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls gpurun_out
