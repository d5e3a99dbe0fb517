echo "k3_duff parity: $(RAPP_LIB=build_variants/k3_duff.so timeout 300 python -m pytest tests/test_search_gpu.py tests/test_config1.py tests/test_slo.py -x -q 2>&1 | tail -1)" > gpurun_out/r2s3_ab_k3h.txt
bash tools/ab_lattice.sh k3_cur k3_duff >> gpurun_out/r2s3_ab_k3h.txt 2>&1
