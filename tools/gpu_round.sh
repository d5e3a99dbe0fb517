bash tools/ab_stream.sh k2_base k2_dual > gpurun_out/r2s3_ab_k2dual.txt 2>&1
RAPP_LIB=build_variants/k2_dual.so timeout 600 python -m pytest tests/test_interp_gpu.py tests/test_config1.py -x -q 2>&1 | tail -2 >> gpurun_out/r2s3_ab_k2dual.txt
