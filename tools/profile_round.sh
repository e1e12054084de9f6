#!/bin/bash
# Round profiling recipe (run under gpurun): GPU tests, smoke, bench lines (C5 headline + C1-C4), the reference
# arm, the ncu launch list of the default bench command, and ncu --set full captures of both engines on C2,
# C4 and C5. Summarise here with tools/ncu_report.py (see profiles/rNN_*_ncu.md).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -rs > gpurun_out/gputest.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_C5.log 2>&1
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C5.log 2>&1
timeout 300 python bench.py --impl reference --config C2 > gpurun_out/bench_ref_C2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
for c in C2 C4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lanczos|k_bisect" -c 3 \
    -o gpurun_out/prof_$c -f python tools/prof_c5.py $c 0 > gpurun_out/ncu_full_$c.log 2>&1
done
