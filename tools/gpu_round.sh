bash tools/ab_lattice.sh k3_c4 k3_c32 k3_c64 > gpurun_out/r2s3_ab_k3c.txt 2>&1
