#!/bin/bash
# Round profiling recipe (run under gpurun): GPU tests, smoke, bench lines (C5 headline + C1-C4), the reference
# arm, the ncu launch list of the default bench command, and ncu --set full captures of the engines on C2,
# C4 and C5 (matrix 0). Each ncu pass runs only after the same command exited 0 without ncu.
# Summarise here with tools/ncu_report.py (see profiles/rNN_*_ncu.md).
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -s -rs > gpurun_out/gputest.log 2>&1; echo "gputest rc=$?"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/bench_C5.log 2>&1; echo "bench C5 rc=$?"
for c in C1 C2 C3 C4; do timeout 600 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo "bench $c rc=$?"; done
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_C5.log 2>&1; echo "ref C5 rc=$?"
timeout 300 python bench.py --impl reference --config C2 > gpurun_out/bench_ref_C2.log 2>&1; echo "ref C2 rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C5.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1; echo "launch list rc=$?"
for c in C2 C4; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_lanczos|k_bisect" -c 3 \
    -o gpurun_out/prof_$c -f python tools/prof_c5.py $c 0 > gpurun_out/ncu_full_$c.log 2>&1; echo "ncu $c rc=$?"
done
# C5 matrix 0: the bisection kernel (launch 1 of k_bisect; launch 0 is the classification) and engine L
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_bisect --launch-skip 1 --launch-count 1 \
  -o gpurun_out/prof_C5_bisect -f python tools/prof_c5.py C5 0 > gpurun_out/ncu_full_C5_bisect.log 2>&1; echo "ncu C5 bisect rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_lanczos -c 1 \
  -o gpurun_out/prof_C5_lanczos -f python tools/prof_c5.py C5 0 > gpurun_out/ncu_full_C5_lanczos.log 2>&1; echo "ncu C5 lanczos rc=$?"
