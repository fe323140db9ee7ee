#!/bin/bash
# Bench lines of every config + the 8-maps-per-rank share of C5 (one rank of --gpus 8).
tag=$1
mkdir -p gpurun_out
for c in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg_$c.log 2>&1
done
timeout 600 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg_maps8.log 2>&1
