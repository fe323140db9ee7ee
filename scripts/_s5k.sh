mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s5k_build.log 2>&1
for k in pass_a2 pass_b; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 16 -c 1 \
    -o gpurun_out/s5k_${k}_full -f python scripts/profile_mg.py 64 > gpurun_out/s5k_ncu_full_$k.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/s5k_launches_c5.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/s5k_ncu_launch_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 8000 --csv \
  --log-file gpurun_out/s5k_launches_c4.csv python bench.py --config C4 --steps 1 --warmup 0 --no-cpu-baseline \
  > gpurun_out/s5k_ncu_launch_c4.log 2>&1
timeout 300 python scripts/gaps.py 64 > gpurun_out/s5k_gaps.log 2>&1
