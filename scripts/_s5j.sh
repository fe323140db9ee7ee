mkdir -p gpurun_out
NI_FUSED_MAX_EDGES=65536 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5j_bench_f64k.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5j_bench.log 2>&1
NI_FUSED_MAX_EDGES=65536 timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5j_bench_f64k_b.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s5j_bench_b.log 2>&1
NI_FUSED_MAX_EDGES=65536 timeout 300 python bench.py --maps 8 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s5j_cfg_maps8_f64k.log 2>&1
NI_FUSED_MAX_EDGES=65536 timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q --timeout 300 > gpurun_out/s5j_pytest.log 2>&1
