#!/bin/bash
# Quick GPU iteration: selected tests, the C5 bench line, optional ncu captures.
# Usage: bash scripts/gpu_quick.sh TAG "pytest args" [ncu]
tag=$1; tests=$2; mode=$3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || true
if [ -n "$tests" ]; then
  timeout 1200 python -m pytest $tests -x -q --timeout 300 > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
fi
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${tag}_bench.log
for c in C1 C4; do
  timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_bench_$c.log 2>&1
done
if [ "$mode" = "ncu" ]; then
  for k in pass_a pass_b; do
    timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 \
      -o gpurun_out/${tag}_${k}_full -f python scripts/profile_mg.py 64 \
      > gpurun_out/${tag}_ncu_full_$k.log 2>&1
    echo "ncu full exit $?" >> gpurun_out/${tag}_ncu_full_$k.log
  done
fi
