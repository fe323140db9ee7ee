mkdir -p gpurun_out
rm -f gpurun_out/s5h_check.log
for c in C4 C3 C5_00 C1; do
  timeout 300 python scripts/fill_vs_golden.py $c >> gpurun_out/s5h_check.log 2>&1
done
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5h_bench.log 2>&1
for c in C1 C3 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5h_cfg_$c.log 2>&1
done
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5h_cfg_maps8.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5h_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5h_pytest.log
