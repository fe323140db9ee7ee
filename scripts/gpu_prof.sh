#!/bin/bash
# Profiling pass: launch lists of C5 and C4 steps, ncu --set full of chosen kernels.
# Usage: bash scripts/gpu_prof.sh TAG "kernel regex" COUNT
tag=$1; kre=$2; cnt=${3:-4}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || true
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/${tag}_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_c5.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/${tag}_launches_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_c4.log 2>&1
if [ -n "$kre" ]; then
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$kre" -c $cnt \
    -o gpurun_out/${tag}_kernels_full -f python scripts/profile_mg.py 64 \
    > gpurun_out/${tag}_ncu_full.log 2>&1
  echo "ncu full exit $?" >> gpurun_out/${tag}_ncu_full.log
fi
