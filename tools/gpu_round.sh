set -x
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_tick_commit -c 1 -o gpurun_out/prof_commit python tools/tick_profile.py > gpurun_out/ncu_commit.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_mec_lattice -c 1 -o gpurun_out/prof_lattice_r01b python bench.py --workload lattice --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/ncu_lattice.log 2>&1
ls -la gpurun_out
