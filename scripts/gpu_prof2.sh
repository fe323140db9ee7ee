#!/bin/bash
# ncu --set full of the two fine passes + the C5 launch list; optional tests first.
tag=$1; tests=$2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1 || true
if [ -n "$tests" ]; then
  timeout 1200 python -m pytest $tests -x -q > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
fi
for k in pass_a pass_b; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 20 -c 1 \
    -o gpurun_out/${tag}_${k}_full -f python scripts/profile_mg.py 64 \
    > gpurun_out/${tag}_ncu_full_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/${tag}_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_c5.log 2>&1
