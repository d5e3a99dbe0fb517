bash tools/ab_lattice.sh k3_base k3_runbr > gpurun_out/r2s3_ab_k3d.txt 2>&1
