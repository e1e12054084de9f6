for c in C2 C3 C4; do timeout 300 python tools/overlap.py $c > /tmp/o.txt 2>&1; head -3 /tmp/o.txt; done
