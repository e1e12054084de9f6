timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in C2 C3 C4; do timeout 200 python tools/overlap.py $c > /tmp/o.txt 2>&1; cat /tmp/o.txt; done
