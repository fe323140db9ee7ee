mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5f_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5f_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5f_bench.log 2>&1
NI_MG_W_HI=1 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5f_bench_v.log 2>&1
NI_MG_W_HI=2 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5f_bench_w2.log 2>&1
NI_MG_W_HI=4 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5f_bench_w4.log 2>&1
for c in C1 C3 C4; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5f_cfg_$c.log 2>&1
  NI_MG_W_HI=1 timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5f_cfg_${c}_v.log 2>&1
done
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5f_cfg_maps8.log 2>&1
