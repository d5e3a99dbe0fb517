CASES="mlp" bash tools/sanitize.sh > /dev/null 2>&1; cp gpurun_out/sanitize_summary.txt gpurun_out/r2s3_sanitize_mlp.txt
