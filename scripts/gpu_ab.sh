#!/bin/bash
# A/B of library variants on the C5 bench: bash scripts/gpu_ab.sh TAG lib1.so lib2.so ...
tag=$1; shift
mkdir -p gpurun_out
for lib in "$@"; do
  n=$(basename $lib .so)
  NI_LIB=$lib timeout 600 python bench.py --no-cpu-baseline > gpurun_out/${tag}_ab_$n.log 2>&1
done
