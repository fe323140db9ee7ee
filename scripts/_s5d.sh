mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5d_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5d_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5d_bench.log 2>&1
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5d_cfg_C1.log 2>&1
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5d_cfg_maps8.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/s5d_launches_C1.csv python scripts/profile_cfg.py C1 > gpurun_out/s5d_ncu_C1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:scale_fused -s 3 -c 1 -o gpurun_out/s5d_fused_full -f python scripts/profile_cfg.py C1 > gpurun_out/s5d_ncu_fused.log 2>&1
