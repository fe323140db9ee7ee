mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5e_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5e_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s5e_smoke.log 2>&1
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5e_cfg_C1.log 2>&1
timeout 300 python bench.py --config C2 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5e_cfg_C2.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5e_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"down_kernel|up_kernel" -s 360 -c 20 \
    -o gpurun_out/s5e_coarse_full -f python scripts/profile_mg.py 64 > gpurun_out/s5e_ncu_coarse.log 2>&1
