bash tools/ab_lattice.sh k3_runbr k3_ru2 k3_sv > gpurun_out/r2s3_ab_k3e.txt 2>&1
