#!/bin/bash
# One GPU call: parity tests, smoke, bench line, per-config step times,
# launch list, ncu --set full captures of the two fine multigrid passes.
# Usage (from the repo root, under gpurun): bash scripts/gpu_round.sh [tag] [skip-tests]
tag=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${tag}_smi.txt 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${tag}_pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${tag}_bench.log
for c in C1 C2 C3 C4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$c.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
  --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/${tag}_ncu_launch.log
for k in pass_a pass_b; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 \
    -o gpurun_out/${tag}_${k}_full -f python scripts/profile_mg.py 64 \
    > gpurun_out/${tag}_ncu_full_$k.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/${tag}_ncu_full_$k.log
done
