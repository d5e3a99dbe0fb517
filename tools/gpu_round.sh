timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1
tail -c 3000 gpurun_out/bench_default.log
