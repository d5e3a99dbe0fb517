timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_gputest3.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2s3_gputest3.log
