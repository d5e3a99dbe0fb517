for v in k3_consec k3_consec_ru2; do echo "$v parity: $(RAPP_LIB=build_variants/$v.so timeout 300 python -m pytest tests/test_search_gpu.py tests/test_config1.py tests/test_slo.py -x -q 2>&1 | tail -1)"; done > gpurun_out/r2s3_ab_k3g.txt
bash tools/ab_lattice.sh k3_sv k3_consec k3_consec_ru2 >> gpurun_out/r2s3_ab_k3g.txt 2>&1
