timeout 300 python -m pytest tests/test_learned.py -x -q 2>&1 | tail -5
timeout 600 python bench.py --workload mlp --steps 30 > gpurun_out/bench_mlp.log 2>&1
cat gpurun_out/bench_mlp.log | tail -3
