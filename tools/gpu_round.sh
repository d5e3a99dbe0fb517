bash tools/ab_mlp.sh mlp_ff mlp_ff_l3 > gpurun_out/r2s3_ab_mlp2.txt 2>&1
