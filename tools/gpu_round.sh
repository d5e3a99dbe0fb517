timeout 600 python bench.py --workload mlp --steps 30 > gpurun_out/bench_mlp.log 2>&1; tail -c 600 gpurun_out/bench_mlp.log
