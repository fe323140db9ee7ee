#!/bin/bash
# One GPU call: build, GPU parity tests, smoke, C5 bench line, C1-C4 step times,
# stage times, launch lists, ncu --set full of the fine passes.
# Usage (repo root, under gpurun): bash scripts/gpu_check.sh TAG [skip-tests]
mkdir -p gpurun_out
tag=${1:-chk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${tag}_build.log 2>&1
if [ "$2" != "skip-tests" ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/${tag}_pytest.log 2>&1
  echo "pytest exit $?" >> gpurun_out/${tag}_pytest.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/${tag}_smoke.log
fi
timeout 600 python bench.py > gpurun_out/${tag}_bench.log 2>&1
echo "bench exit $?" >> gpurun_out/${tag}_bench.log
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/${tag}_bench_reference.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg_$c.log 2>&1
done
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${tag}_cfg_maps8.log 2>&1
for c in C1 C3 C4; do timeout 300 python scripts/stage_times.py $c 3 > gpurun_out/${tag}_stages_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/${tag}_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_c5.log 2>&1
echo "ncu launch exit $?" >> gpurun_out/${tag}_ncu_launch_c5.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/${tag}_launches_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/${tag}_ncu_launch_c4.log 2>&1
for k in pass_a2 pass_b; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 15 -c 1 \
    -o gpurun_out/${tag}_${k}_full -f python scripts/profile_mg.py 64 > gpurun_out/${tag}_ncu_full_$k.log 2>&1
done
