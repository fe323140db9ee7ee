for c in C3 C4; do for p in 1 2; do NI_FILL_PAIR=$p timeout 300 python scripts/fill_single.py $c 2>&1 | tail -1 | sed "s/^/pair$p /"; done; done
for n in 4 16 64; do for p in 1 2; do NI_FILL_PAIR=$p timeout 300 python scripts/fill_bench.py $n 2>&1 | tail -1 | sed "s/^/pair$p /"; done; done
