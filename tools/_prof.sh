set -e
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-guided > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_lanczos|k_bisect" -c 3 -o gpurun_out/prof_c2 python tools/prof_step.py C2 > gpurun_out/ncu_full.log 2>&1
python bench.py --config C4 --no-cpu-baseline --no-guided --steps 3 > gpurun_out/bench_c4.json 2>&1
python bench.py --config C3 --no-cpu-baseline --no-guided --steps 3 > gpurun_out/bench_c3.json 2>&1
