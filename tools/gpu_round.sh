RAPP_LIB=build_variants/prof.so timeout 300 python tools/tick_commit_breakdown.py --full-grid > gpurun_out/r2s3_commit_breakdown4.txt 2>&1
