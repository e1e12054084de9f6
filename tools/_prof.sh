set -e
ncu --set full --clock-control none --import-source on -k regex:"k_lanczos|k_bisect" -c 3 -o gpurun_out/prof_c2b python tools/prof_step.py C2 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_bisect" -c 2 -o gpurun_out/prof_c3b python tools/prof_step.py C3 > gpurun_out/ncu_full3.log 2>&1
