#!/bin/bash
# Round profiling recipe (run under gpurun): tests, smoke, bench lines for C1-C5, the reference arm,
# the ncu launch list of the bench command and ncu --set full captures of both engines on C2 and C4.
# Summarise with: python tools/ncu_report.py gpurun_out/prof_c2.ncu-rep gpurun_out/launches_c2.csv profiles/rNN_c2_ncu.md /tmp/x.json
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
for c in C1 C3 C4 C5; do python bench.py --config $c --no-cpu-baseline --no-guided --steps 3 > gpurun_out/bench_$c.json 2>&1 || true; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2>&1 || true
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-guided > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_lanczos|k_bisect" -c 3 -o gpurun_out/prof_c2 -f python tools/prof_step.py C2 > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_lanczos|k_bisect" -c 3 -o gpurun_out/prof_c4 -f python tools/prof_step.py C4 > gpurun_out/ncu_full_c4.log 2>&1
tail -c 600 gpurun_out/bench_c2.json
