for sp in 0 1 0 1; do echo "RAPP_TICK_SPIN=$sp"; RAPP_TICK_SPIN=$sp timeout 600 python bench.py --workload tick --full-grid --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['tick'])"; RAPP_TICK_SPIN=$sp timeout 600 python bench.py --workload tick --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['tick'])"; done > gpurun_out/r2s3_spin.txt 2>&1
RAPP_TICK_SPIN=1 timeout 600 python -m pytest tests/test_tick_gpu.py -x -q 2>&1 | tail -1 >> gpurun_out/r2s3_spin.txt
