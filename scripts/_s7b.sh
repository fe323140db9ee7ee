mkdir -p gpurun_out
timeout 600 python scripts/e2e_outlier.py 14 > gpurun_out/s7b_outlier.log 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s7b_bench.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --steps 20 --warmup 5 > gpurun_out/s7b_bench20.log 2>&1
