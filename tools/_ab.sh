timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C2 C3 C4 C5; do timeout 300 python tools/overlap.py $c > /tmp/o.txt 2>&1; head -2 /tmp/o.txt; done
