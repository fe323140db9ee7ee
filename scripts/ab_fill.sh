#!/bin/bash
# A/B the fill kernel builds in exp/ (NI_LIB) against the in-tree library on C5-like batches.
# Usage: bash scripts/ab_fill.sh "lib1 lib2 ..." "nmaps1 nmaps2 ..."
libs=${1:-"paper_2510_11508_b200/libnormint_b200.so"}
sizes=${2:-"64 8"}
mkdir -p gpurun_out
for n in $sizes; do
  for rep in 1 2; do
    for l in $libs; do
      NI_LIB=$l timeout 300 python scripts/fill_bench.py $n 2>&1 | tail -1 | sed "s|^|$(basename $l) |"
    done
  done
done
