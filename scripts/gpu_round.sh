#!/bin/bash
# One GPU call: parity tests, smoke, bench line, launch list, ncu capture of the fill.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [tag]
tag=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
timeout 900 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${tag}_bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/${tag}_ncu_launch.log
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fill_cg -s 1 -c 1 \
  -o gpurun_out/${tag}_fill_full -f python scripts/profile_fill.py 32 \
  > gpurun_out/${tag}_ncu_full.log 2>&1
echo "ncu full exit $?" >> gpurun_out/${tag}_ncu_full.log
