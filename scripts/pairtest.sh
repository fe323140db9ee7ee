for n in 1 4 8 16 64; do timeout 300 python scripts/fill_bench.py $n 2>&1 | tail -1; done
for c in C3 C4; do timeout 300 python scripts/fill_single.py $c 2>&1 | tail -1; done
