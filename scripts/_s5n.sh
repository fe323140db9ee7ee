mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/s5n_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/s5n_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5n_bench.log 2>&1
NI_LIB=exp/libni_fullmask.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5n_bench_fullmask.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5n_bench_b.log 2>&1
NI_LIB=exp/libni_fullmask.so timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5n_bench_fullmask_b.log 2>&1
timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5n_cfg_maps8.log 2>&1
timeout 300 python scripts/gaps.py 64 > gpurun_out/s5n_gaps.log 2>&1
