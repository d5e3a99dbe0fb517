mkdir -p gpurun_out
timeout 900 python bench.py --detail gpurun_out/r2j_default_detail.json > gpurun_out/r2j_default.log 2>&1
timeout 600 python bench.py --workload tick --full-grid > gpurun_out/r2j_tick_full.log 2>&1
timeout 600 python bench.py --workload tick > gpurun_out/r2j_tick_c4.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r2j_gputest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2j_gputest.log
