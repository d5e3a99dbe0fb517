timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mlp -s 2 -c 1 -o gpurun_out/r2h_mlp python bench.py --workload mlp --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 600 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -1 > gpurun_out/r2h_tick_nvtx.txt
