mkdir -p gpurun_out
timeout 600 python scripts/e2e_outlier.py 12 > gpurun_out/s7c_outlier.log 2>&1
timeout 600 python scripts/e2e_outlier.py 12 nogc > gpurun_out/s7c_outlier_nogc.log 2>&1
