bash tools/ab_mlp.sh mlp_l3 mlp_ffma2 mlp_ffma2_db2 > gpurun_out/r2s3_ab_mlp5.txt 2>&1
