timeout 900 python -m pytest tests/test_tick_gpu.py tests/test_integration_gpu.py tests/test_boundary.py -x -q 2>&1 | tail -2 > gpurun_out/r2s3_book.txt
timeout 600 python bench.py --workload tick --full-grid --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r2s3_book.txt
timeout 600 python bench.py --workload tick --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/r2s3_book.txt
timeout 600 python tools/tick_e2e_split.py --full-grid >> gpurun_out/r2s3_book.txt 2>&1
