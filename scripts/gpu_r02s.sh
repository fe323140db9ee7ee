mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r02s_build.log 2>&1
for c in C1 C2 C3; do timeout 300 python scripts/stage_times.py $c 4 > gpurun_out/r02s_stages_$c.log 2>&1; done
timeout 600 python bench.py > gpurun_out/r02s_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02s_launches_c1.csv python scripts/stage_times.py C1 1 > gpurun_out/r02s_ncu_c1.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv --log-file gpurun_out/r02s_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r02s_ncu_c5.log 2>&1
