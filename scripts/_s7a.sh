mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s7a_bench.log 2>&1
timeout 300 python bench.py --config C1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/s7a_cfg_C1.log 2>&1
