timeout 600 python -m pytest tests/test_interp_gpu.py tests/test_config1.py -x -q 2>&1 | tail -2 > gpurun_out/r2s3_ab_k2.txt
bash tools/ab_stream.sh k2_r1 k2_r2 k2_r2_sus k2_r1_sus k2_r2_s3 >> gpurun_out/r2s3_ab_k2.txt 2>&1
