#!/bin/bash
# Scheduler/worker statistics of the fill (stats build in exp/lib_stats.so).
for n in 64 8; do NI_LIB=exp/lib_stats.so timeout 300 python scripts/fill_bench.py $n 2>&1 | grep -E "fill stats|maps=" | tail -2; done
NI_LIB=exp/lib_stats.so timeout 300 python scripts/fill_single.py C4 2>&1 | grep -E "fill stats|C4" | tail -2
