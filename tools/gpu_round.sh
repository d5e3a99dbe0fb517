# round-2 final measurement set, results under gpurun_out/r2i_*
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2i_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2i_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2i_smoke.log 2>&1
timeout 900 python bench.py --detail gpurun_out/r2i_default_detail.json > gpurun_out/r2i_default.log 2>&1
timeout 600 python bench.py --workload lattice > gpurun_out/r2i_lattice.log 2>&1
timeout 600 python bench.py --workload tick --full-grid > gpurun_out/r2i_tick_full.log 2>&1
timeout 600 python bench.py --workload tick > gpurun_out/r2i_tick_c4.log 2>&1
timeout 600 python bench.py --workload mlp > gpurun_out/r2i_mlp.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2i_reference.log 2>&1
TICKS=40 timeout 600 python tools/tick_profile.py --full-grid > gpurun_out/r2i_tickprof_full.txt 2>&1
TICKS=40 timeout 600 python tools/tick_profile.py > gpurun_out/r2i_tickprof_c4.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i_launches_default.csv python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > /dev/null 2>&1
