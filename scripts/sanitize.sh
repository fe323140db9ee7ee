#!/bin/bash
# compute-sanitizer over the small workloads of scripts/sanitize_case.py.
# Usage (under gpurun): bash scripts/sanitize.sh TAG
tag=${1:-r02}
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python scripts/sanitize_case.py > gpurun_out/${tag}_sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/${tag}_sanitizer_$tool.txt
done
