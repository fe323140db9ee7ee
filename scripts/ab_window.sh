for n in 64 16; do for w in 0 2 3 4 6; do NI_FILL_WINDOW=$w timeout 300 python scripts/fill_bench.py $n 2>&1 | tail -1 | sed "s|^|win=$w |"; done; done
NI_FILL_WINDOW=3 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
