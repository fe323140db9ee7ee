mkdir -p gpurun_out
rm -f gpurun_out/s5i_check.log
for c in C4 C3 C5_00 C1; do
  timeout 300 python scripts/fill_vs_golden.py $c >> gpurun_out/s5i_check.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5i_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5i_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5i_bench.log 2>&1
for c in C1 C2 C3 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5i_cfg_$c.log 2>&1
done
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5i_cfg_maps8.log 2>&1
NI_MG_TAIL=0 timeout 300 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5i_cfg_C3_notail.log 2>&1
