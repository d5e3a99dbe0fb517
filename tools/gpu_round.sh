timeout 900 python -m pytest tests/test_tick_gpu.py tests/test_integration_gpu.py tests/test_boundary.py tests/test_limits_gpu.py -x -q 2>&1 | tail -1 > gpurun_out/r2s3_pyopt.txt
timeout 900 python tools/tick_py_profile.py --full-grid >> gpurun_out/r2s3_pyopt.txt 2>&1
timeout 600 python bench.py --workload tick --full-grid --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['tick'])" >> gpurun_out/r2s3_pyopt.txt
